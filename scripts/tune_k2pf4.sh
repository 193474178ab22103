#!/bin/bash
# K2 at 4 CTAs/SM: L2-prefetch distance, alternating runs (REXI_K2_PF residency waves; cfg2 refined)
for i in 1 2 3; do
  for pf in 1 0.5 0.25; do
    echo -n "REXI_K2_PF=$pf  "
    REXI_K2_PF=$pf timeout 300 python bench.py --steps 200 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/d['steps'],4) for k,v in d['kernels'].items() if k in ('l0_k2',)})"
  done
done
