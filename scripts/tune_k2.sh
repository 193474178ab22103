#!/bin/bash
# K2 residual-loop unroll x CTAs/SM sweep on cfg2 (refined)
for v in "1 3" "2 3" "3 3" "5 3" "2 2"; do
  set -- $v
  echo "=== K2_RES_UNROLL=$1 K2_MINB=$2"
  REXI_NVCC_EXTRA="-DK2_RES_UNROLL=$1 -DK2_MINB=$2" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  PROBE_PROF=1 python scripts/probe_1d.py 2 2>&1 | grep -E "device-resident|l0_k2|gpu-truth" | tail -3
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
