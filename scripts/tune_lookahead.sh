#!/bin/bash
# windowed spmv producer: unit claim and directory entry one stage ahead (CGW_LOOKAHEAD=1) vs
# inside the refill (0); cfg 5 / cfg 3 / cfg 4 step times, bitwise comparison
mkdir -p gpurun_out
for v in 0 1 0 1; do
  echo "=== CGW_LOOKAHEAD=$v"
  REXI_NVCC_EXTRA="-DCGW_LOOKAHEAD=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  [ -f gpurun_out/snap_la$v.npz ] || timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_la$v.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
python scripts/cocg_compare.py gpurun_out/snap_la0.npz gpurun_out/snap_la1.npz
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
timeout 600 python scripts/cocg_steps.py 4 2 2>&1 | grep "^step"
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 5 2 2>&1 | grep "cg_spmv"
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_spmv"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_hygiene.py tests/test_gpu_stiff.py -x -q 2>&1 | tail -3
