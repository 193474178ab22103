#!/bin/bash
# COCG row stride = live prefix (ld) on/off x TMA spmv on/off; bitwise comparison, cfg 3 / cfg 5 step times
mkdir -p gpurun_out
run() {
  python scripts/cocg_snapshot.py gpurun_out/snap_$1.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
}
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
echo "=== staged, no ld"; REXI_COCG_NOTMA=1 REXI_COCG_NOLD=1 run st_nold
echo "=== staged, ld"; REXI_COCG_NOTMA=1 run st_ld
echo "=== TMA, no ld"; REXI_COCG_NOLD=1 run tma_nold
echo "=== TMA, ld"; run tma_ld
for v in st_ld tma_nold tma_ld; do python scripts/cocg_compare.py gpurun_out/snap_st_nold.npz gpurun_out/snap_$v.npz; done
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_" 
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 5 2 2>&1 | grep "cg_" 
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
