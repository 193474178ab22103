#!/bin/bash
# K2 residual: full double-double vs mixed (exact products for Re(entry) only)
for v in "" "-DK2_MIXED"; do
  echo "=== flags: '$v'"
  REXI_NVCC_EXTRA="$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  PROBE_PROF=1 python scripts/probe_1d.py 2 2>&1 | grep -E "refine=1|gpu-truth|device-resident|l0_k2" | tail -4
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
