#!/bin/bash
# band solver: shifts per CTA of the staged interior sweeps (BLG)
for v in 16 8 4; do
  echo "=== BLG=$v"
  REXI_NVCC_EXTRA="-DBAND_BLG=$v" python -c "from paper_1912_03312_b200 import build_native as b; b.build(force=True)" > /dev/null 2>&1
  python scripts/band_profile.py 2>/dev/null | grep -E "graph|s1|s3"
done
python -c "from paper_1912_03312_b200 import build_native as b; b.build(force=True)" > /dev/null 2>&1
