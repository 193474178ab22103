#!/bin/bash
# K3 (dd lane sum): lane/block indices by division or by shift, at 7 / 8 CTAs/SM (cfg2 refined)
for v in "-DK3_DIV=1" "-DK3_DIV=0" "-DK3_DIV=1 -DK3_MINB=8" "-DK3_DIV=0 -DK3_MINB=8" "-DK3_DIV=0 -DK3_MINB=6"; do
  echo "=== $v"
  REXI_NVCC_EXTRA="$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_k3')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
