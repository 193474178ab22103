#!/bin/bash
# windowed spmv: L2 eviction-priority hints on the bulk copies (tiles evict_first, z windows
# evict_last) vs none (-DCGW_L2HINT=0); cfg 5 / cfg 3 step times; threaded table build time
mkdir -p gpurun_out
for v in 0 1 0 1; do
  echo "=== CGW_L2HINT=$v"
  REXI_NVCC_EXTRA="-DCGW_L2HINT=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
python scripts/prepare_time.py 3 5 2>&1 | grep "screen=True"
REXI_COCG_TRACE=1 timeout 300 python scripts/cocg_widths.py 5 2 2>&1 | grep "cg_spmv"
timeout 900 python -m pytest tests/test_gpu_cocg_layout.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
