#!/bin/bash
# COCG tolerance split at BASELINE conditioning: accuracy (scripts/tol_check.py,
# north_star: <= 1e-8 vs truth every step, per-shift residual <= 1e-12) and
# full-size cfg3 / cfg5 step times
for v in "1e-10 1e-9 1e-6 1e-4" "1e-10 1e-9 1e-5 1e-3" "3e-10 1e-9 1e-5 1e-3" "1e-10 1e-9 3e-6 3e-4" "1e-9 1e-8 1e-6 1e-4" "1e-10 1e-9 1e-4 1e-3"; do
  set -- $v
  echo "=== tol1=$1 cap1=$2 tol2=$3 cap2=$4"
  export REXI_COCG_TOL1=$1 REXI_COCG_CAP1=$2 REXI_COCG_TOL2=$3 REXI_COCG_CAP2=$4
  timeout 600 python scripts/tol_check.py 2>&1 | tail -1
  python scripts/cocg_steps.py 3 4 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
  python scripts/cocg_steps.py 5 2 2>&1 | grep "^step" | awk '{print $3}' | tr '\n' ' '; echo
done
