#!/bin/bash
# COCG iteration kernels launched with programmatic stream serialization (default) vs plain
# stream order (REXI_COCG_NOPDL=1); bitwise comparison, cfg 3 / cfg 5 / cfg 4 step times
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
for v in 1 0 1 0; do
  if [ $v = 1 ]; then export REXI_COCG_NOPDL=1; echo "=== plain launches"; else unset REXI_COCG_NOPDL; echo "=== PDL"; fi
  [ -f gpurun_out/snap_pdl$v.npz ] || timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_pdl$v.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
unset REXI_COCG_NOPDL
python scripts/cocg_compare.py gpurun_out/snap_pdl1.npz gpurun_out/snap_pdl0.npz
timeout 600 python scripts/cocg_steps.py 4 2 2>&1 | grep "^step"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_hygiene.py tests/test_gpu_stiff.py tests/test_gpu_distributed.py tests/test_gpu_complex.py -x -q 2>&1 | tail -3
