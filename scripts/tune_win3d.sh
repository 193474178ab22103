#!/bin/bash
# COCG windowed spmv on 3D patterns (one row-lane per thread, seven windows) vs the staged
# gather kernel (REXI_COCG_NOWIN=1); bitwise comparison, cfg 5 / cfg 3 step times
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== NOWIN"; REXI_COCG_NOWIN=1 timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_nowin3.npz 2>&1 | tail -1
REXI_COCG_NOWIN=1 timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
echo "=== windowed"; timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_win3.npz 2>&1 | tail -1
timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
python scripts/cocg_compare.py gpurun_out/snap_nowin3.npz gpurun_out/snap_win3.npz
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 5 2 2>&1 | grep "cg_"
echo "=== cfg3"; timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
