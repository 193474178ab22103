#!/bin/bash
# COCG narrow layouts (kp <= 2): launch-per-phase kernels (REXI_COCG_NONARROW=1) vs whole
# iterations in one cooperative launch; bitwise comparison, cfg 3 / cfg 5 step times
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== NONARROW"; REXI_COCG_NONARROW=1 timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_nonarrow.npz 2>&1 | tail -1
REXI_COCG_NONARROW=1 timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== narrow"; timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_narrow.npz 2>&1 | tail -1
timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
python scripts/cocg_compare.py gpurun_out/snap_nonarrow.npz gpurun_out/snap_narrow.npz
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_"
echo "=== cfg5 NONARROW"; REXI_COCG_NONARROW=1 timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
echo "=== cfg5 narrow"; timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
