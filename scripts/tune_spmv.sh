#!/bin/bash
# staged spmv: z gathers in flight per thread (CG_STB)
for b in 4 8 16; do
  echo "=== CG_STB=$b"
  REXI_NVCC_EXTRA="-DCG_STB=$b" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  for c in 3 5; do python scripts/cocg_widths.py $c 2>/dev/null | grep -E "spmv@64|spmv@32|spmv@16|total"; done
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
