#!/bin/bash
# staged spmv: atomic claim counter vs static striding (cfg3 step 3 width profile)
for v in 0 1; do
  echo "=== CG_STATIC=$v"
  REXI_NVCC_EXTRA="-DCG_STATIC=$v" python -c "from paper_1912_03312_b200 import build_native as b; b.build(force=True)" > /dev/null 2>&1
  python scripts/cocg_widths.py 3 2 2>/dev/null | grep -E "spmv@(64|32)|update@64|total"
done
python -c "from paper_1912_03312_b200 import build_native as b; b.build(force=True)" > /dev/null 2>&1
