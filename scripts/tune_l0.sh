#!/bin/bash
# level-0 kernels: CTAs/SM (launch bounds) sweep on cfg2, refine 0 and 1
for v in "3 4 4" "4 5 5" "5 5 6" "4 4 5"; do
  set -- $v
  echo "=== S1_MINB=$1 S3_MINB=$2 K3_MINB=$3"
  REXI_NVCC_EXTRA="-DS1_MINB=$1 -DS3_MINB=$2 -DK3_MINB=$3" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  PROBE_PROF=1 python scripts/probe_1d.py 2 2>&1 | grep -E "device-resident|l0_|gpu-truth"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cfg or golden or 1d or tridiag" 2>&1 | tail -2
