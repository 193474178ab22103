#!/bin/bash
# windowed spmv refill order: z windows + blob before the previous stage's tile stores drain
# (CGW_ZFIRST=1) vs everything after (0); cfg 5 / cfg 3 step times, bitwise comparison
mkdir -p gpurun_out
for v in 0 1 0 1; do
  echo "=== CGW_ZFIRST=$v"
  REXI_NVCC_EXTRA="-DCGW_ZFIRST=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  [ -f gpurun_out/snap_zf$v.npz ] || timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_zf$v.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
python scripts/cocg_compare.py gpurun_out/snap_zf0.npz gpurun_out/snap_zf1.npz
REXI_NVCC_EXTRA="-DCGW_ZFIRST=1" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_hygiene.py tests/test_gpu_stiff.py -x -q 2>&1 | tail -3
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
