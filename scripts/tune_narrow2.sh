#!/bin/bash
# COCG: TMA update at every width (REXI_COCG_UTMAMIN=64: the wide ones only) and the windowed
# spmv at 2 / 1 lanes (REXI_COCG_WINMIN=4: off); bitwise comparison, cfg 3 / 5 step times
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== base (utma >= 64, win >= 4)"; REXI_COCG_UTMAMIN=64 REXI_COCG_WINMIN=4 timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_nb.npz 2>&1 | tail -1
REXI_COCG_UTMAMIN=64 REXI_COCG_WINMIN=4 timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== utma all, win >= 4"; REXI_COCG_WINMIN=4 timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== utma all, win >= 2"; REXI_COCG_WINMIN=2 timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
echo "=== utma all, win >= 1"; timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_na.npz 2>&1 | tail -1
timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
python scripts/cocg_compare.py gpurun_out/snap_nb.npz gpurun_out/snap_na.npz
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_"
echo "=== cfg5 base"; REXI_COCG_UTMAMIN=64 REXI_COCG_WINMIN=4 timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
echo "=== cfg5 all"; timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py tests/test_gpu_distributed.py tests/test_gpu_band.py -x -q 2>&1 | tail -3
