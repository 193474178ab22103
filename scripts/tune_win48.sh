#!/bin/bash
# COCG windowed spmv for the 8- and 4-lane layouts (REXI_COCG_WINMIN=16: off); bitwise comparison, cfg 3 step times
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== win >= 16"; REXI_COCG_WINMIN=16 timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_w16.npz 2>&1 | tail -1
REXI_COCG_WINMIN=16 timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== win >= 8"; REXI_COCG_WINMIN=8 timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== win >= 4"; timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_w4.npz 2>&1 | tail -1
timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
python scripts/cocg_compare.py gpurun_out/snap_w16.npz gpurun_out/snap_w4.npz
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
