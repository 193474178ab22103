#!/bin/bash
# K2 with one shared-memory tile (x overwrites the pivots; the correction reads
# complex64 pivots from HBM) vs two tiles, at 3-5 CTAs/SM (cfg2 refined)
for v in "-DK2_ONE_TILE=1 -DK2_MINB=4" "-DK2_ONE_TILE=1 -DK2_MINB=3" "-DK2_ONE_TILE=1 -DK2_MINB=5" "-DK2_ONE_TILE=0 -DK2_MINB=3"; do
  echo "=== $v"
  REXI_NVCC_EXTRA="$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_s1','l0_k3')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
