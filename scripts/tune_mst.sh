#!/bin/bash
# band solver: rows per block of the staged path (M)
for v in 64 32 16; do
  echo "=== MST=$v"
  REXI_NVCC_EXTRA="-DBAND_MST=$v" python -c "from paper_1912_03312_b200 import build_native as b; b.build(force=True)" > /dev/null 2>&1
  python scripts/band_profile.py 2>/dev/null | grep -E "graph|s1|s3|red"
done
python -c "from paper_1912_03312_b200 import build_native as b; b.build(force=True)" > /dev/null 2>&1
