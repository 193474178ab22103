#!/bin/bash
for pair in "1e-8 1e-4" "1e-9 1e-5" "1e-9 1e-4" "1e-10 1e-5" "1e-10 1e-6"; do
  set -- $pair
  echo "=== cap1=$1 cap2=$2"
  REXI_COCG_CAP1=$1 REXI_COCG_CAP2=$2 timeout 600 python scripts/probe_cocg.py 3 5 2>&1 | grep -v build
done
