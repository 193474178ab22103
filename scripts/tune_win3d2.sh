#!/bin/bash
# 3D patterns: windowed spmv at 16 and 8 lanes (one row-lane per thread) vs the gather kernels
# there (REXI_COCG_WINMIN=64); bitwise comparison, cfg 5 step times and per-width profile
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== win >= 64"; REXI_COCG_WINMIN=64 timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_3a.npz 2>&1 | tail -1
REXI_COCG_WINMIN=64 timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== default"; timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_3b.npz 2>&1 | tail -1
timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
python scripts/cocg_compare.py gpurun_out/snap_3a.npz gpurun_out/snap_3b.npz
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 5 2 2>&1 | grep "cg_"
timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
