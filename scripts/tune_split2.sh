#!/bin/bash
# first-solve / correction split: accuracy (scripts/split_check.py) and cfg3/cfg5 step times
for v in "1e-10 1e-9 1e-6 1e-4" "1e-12 1e-11 1e-4 1e-2" "1e-12 1e-11 1e-5 1e-3" "1e-11 1e-10 1e-5 1e-3" "3e-12 3e-11 1e-4 1e-2"; do
  set -- $v
  echo "=== tol1=$1 cap1=$2 tol2=$3 cap2=$4"
  export REXI_COCG_TOL1=$1 REXI_COCG_CAP1=$2 REXI_COCG_TOL2=$3 REXI_COCG_CAP2=$4
  timeout 600 python scripts/split_check.py 2>&1 | tail -1
  python scripts/cocg_steps.py 3 3 2>&1 | grep "^step" | tr '\n' ' '; echo
  python scripts/cocg_steps.py 5 2 2>&1 | grep "^step" | tr '\n' ' '; echo
done
