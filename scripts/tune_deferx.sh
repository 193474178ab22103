#!/bin/bash
# COCG x update: in the update kernel (CG_DEFER_X=0, 96 + 80 B per live row-shift
# and iteration) vs deferred to the next spmv (CG_DEFER_X=1, 48 + 112 B = SURVEY
# 8(d)'s 160 B); bitwise comparison of the two and cfg 3 / cfg 5 step times
mkdir -p gpurun_out
for v in 0 1 0 1; do
  echo "=== CG_DEFER_X=$v"
  REXI_NVCC_EXTRA="-DCG_DEFER_X=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python scripts/cocg_snapshot.py gpurun_out/snap_defer$v.npz 2>&1 | tail -1
  python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
python scripts/cocg_compare.py gpurun_out/snap_defer0.npz gpurun_out/snap_defer1.npz
REXI_COCG_TRACE=1 python scripts/cocg_widths.py 3 2 2>&1 | tail -40
python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
