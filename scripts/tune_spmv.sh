#!/bin/bash
# WIDE spmv variants: gather batch x CTAs/SM, cfg 3 and 5 per-width profiles
for v in "4 3" "8 2" "4 2" "16 1"; do
  set -- $v
  echo "=== CG_GB=$1 CG_WIDE_MINB=$2"
  REXI_NVCC_EXTRA="-DCG_GB=$1 -DCG_WIDE_MINB=$2" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for c in 3 5; do python scripts/cocg_widths.py $c 2>/dev/null | grep -E "spmv@64|spmv@32|total"; done
done
