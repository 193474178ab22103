#!/bin/bash
# COCG widest-layout spmv: TMA tiles + register gathers (REXI_COCG_NOWIN=1) vs the
# windowed all-TMA kernel; bitwise comparison, cfg 3 / cfg 4 step times, per-width profile
mkdir -p gpurun_out
run() {
  timeout 300 python scripts/cocg_snapshot.py gpurun_out/snap_$1.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
}
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== TMA tiles + gathers (NOWIN)"; REXI_COCG_NOWIN=1 run nowin
echo "=== windowed"; run win
python scripts/cocg_compare.py gpurun_out/snap_nowin.npz gpurun_out/snap_win.npz
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_"
echo "=== cfg4 NOWIN"; REXI_COCG_NOWIN=1 timeout 600 python scripts/cocg_steps.py 4 2 2>&1 | grep "^step"
echo "=== cfg4 windowed"; timeout 600 python scripts/cocg_steps.py 4 2 2>&1 | grep "^step"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
