#!/bin/bash
# finish kernels at 1-2 lanes: a whole level-2 group per CTA (CG_FL_NARROW=1) vs the
# wide-layout split (0); bitwise comparison, cfg 3 / cfg 5 step times
mkdir -p gpurun_out
for v in 0 1 0 1; do
  echo "=== CG_FL_NARROW=$v"
  REXI_NVCC_EXTRA="-DCG_FL_NARROW=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  [ -f gpurun_out/snap_fl$v.npz ] || timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_fl$v.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
python scripts/cocg_compare.py gpurun_out/snap_fl0.npz gpurun_out/snap_fl1.npz
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "@2 \|@1 \|total"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_hygiene.py tests/test_gpu_stiff.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
