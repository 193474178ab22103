#!/bin/bash
# staged spmv gathers-in-flight x CTAs/SM for 3D rows (15 nnz): cfg5 and cfg3 step times
for v in "8 3" "16 2" "16 3" "12 3"; do
  set -- $v
  echo "=== CG_STB=$1 CG_ST_MINB=$2"
  REXI_NVCC_EXTRA="-DCG_STB=$1 -DCG_ST_MINB=$2" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  python scripts/cocg_steps.py 5 2 2>&1 | grep "^step" | tr '\n' ' '; echo
  python scripts/cocg_steps.py 3 1 2>&1 | grep "^step" | tr '\n' ' '; echo
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
