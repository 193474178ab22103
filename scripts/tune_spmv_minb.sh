#!/bin/bash
# global-CSR spmv (widths < 16) CTAs/SM (register cap) sweep on cfg3/cfg5 step times
for mb in 1 2 3 4; do
  echo "=== CG_SPMV_MINB=$mb"
  REXI_NVCC_EXTRA="-DCG_SPMV_MINB=$mb" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python scripts/cocg_steps.py 3 3 2>&1 | grep "^step"
  python scripts/cocg_steps.py 5 2 2>&1 | grep "^step"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
