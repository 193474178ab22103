#!/bin/bash
# K2 L2-prefetch distance (in residency waves; 0 = off) on cfg2 (refined)
for d in 0 1 2 0.5; do
  echo "=== REXI_K2_PF=$d"
  REXI_K2_PF=$d timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k.startswith('l0')})"
done
