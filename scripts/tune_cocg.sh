#!/bin/bash
# sweep the COCG tolerance pair on the small probes and cfg3/cfg5 timing
for pair in "1e-10 1e-6" "1e-10 1e-4" "1e-11 1e-5" "1e-12 1e-8" "1e-9 1e-7"; do
  set -- $pair
  echo "=== tol1=$1 tol2=$2"
  REXI_COCG_TOL1=$1 REXI_COCG_TOL2=$2 timeout 600 python scripts/probe_cocg.py 3 2>&1 | grep -v build
done
