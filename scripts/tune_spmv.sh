#!/bin/bash
# global-CSR spmv (narrow widths): z gathers in flight (CG_GB)
for b in 4 8; do
  echo "=== CG_GB=$b"
  REXI_NVCC_EXTRA="-DCG_GB=$b" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for c in 3 5; do REXI_COCG_TRACE=1 python scripts/cocg_widths.py $c 2>/dev/null | grep -E "spmv@(8|4|2|1) |total"; done
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
