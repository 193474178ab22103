#!/bin/bash
# COCG repack policy with the TMA kernels (which move whole rows): row-stride granularity
# (REXI_COCG_LDGRAN lanes) x repack threshold (kp / REXI_COCG_REPACK_DIV frozen lanes); cfg 3 / 4 / 5
mkdir -p gpurun_out
python paper_1912_03312_b200/build_native.py > /dev/null 2>&1
for v in "8 8" "2 8" "2 16" "4 16" "1 16" "8 8"; do
  set -- $v
  echo "=== LDGRAN=$1 REPACK_DIV=$2"
  export REXI_COCG_LDGRAN=$1 REXI_COCG_REPACK_DIV=$2
  timeout 300 python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  timeout 300 python scripts/cocg_steps.py 5 3 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
unset REXI_COCG_LDGRAN REXI_COCG_REPACK_DIV
