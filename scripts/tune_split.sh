#!/bin/bash
# tol1/tol2 split sweep (caps = 10x the base) on the small probes and cfg3/cfg5 timing
for pair in "1e-10 1e-6" "1e-11 1e-4" "1e-11 1e-3" "1e-12 1e-3" "1e-12 1e-2" "1e-11 1e-2"; do
  set -- $pair
  c1=$(python -c "print($1*10)"); c2=$(python -c "print(min($2*100, 0.1))")
  echo "=== tol1=$1 tol2=$2 cap1=$c1 cap2=$c2"
  REXI_COCG_TOL1=$1 REXI_COCG_TOL2=$2 REXI_COCG_CAP1=$c1 REXI_COCG_CAP2=$c2 timeout 600 python scripts/probe_cocg.py 3 5 2>&1 | grep -v build
done
