#!/bin/bash
# COCG wide-layout spmv: staged CSR kernel (REXI_COCG_NOTMA=1) vs the persistent
# TMA-pipelined kernel at several gather shapes; bitwise comparison, cfg 3 / cfg 5 step times
mkdir -p gpurun_out
run() {
  python scripts/cocg_snapshot.py gpurun_out/snap_$1.npz 2>&1 | tail -1
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
}
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
echo "=== staged (NOTMA)"; REXI_COCG_NOTMA=1 run notma
for v in "2 4" "1 8" "4 2"; do
  set -- $v
  echo "=== TMA RP=$1 STB=$2"
  REXI_NVCC_EXTRA="-DCGT_ROWS_PAR=$1 -DCGT_STB=$2" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  run tma$1$2
  python scripts/cocg_compare.py gpurun_out/snap_notma.npz gpurun_out/snap_tma$1$2.npz
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 3 2 2>&1 | grep "cg_" 
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_stiff.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
