#!/bin/bash
# K2's residual: Dot2 (error-free hi parts, K2_ALIGNED=0) vs the aligned-quantum
# form (exact plain-fp64 row sums, K2_ALIGNED=1), at 4 and 5 CTAs/SM (cfg2 refined)
for v in "-DK2_ALIGNED=0" "-DK2_ALIGNED=1" "-DK2_ALIGNED=1 -DK2_MINB=5" "-DK2_ALIGNED=0" "-DK2_ALIGNED=1"; do
  echo "=== $v"
  REXI_NVCC_EXTRA="$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline --secondary 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_s1','l0_k3')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
