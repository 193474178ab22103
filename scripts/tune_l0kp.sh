#!/bin/bash
# level-0 kernels with k_pad = 64 at compile time (REXI_L0_KP mask: 1 S1, 2 K2, 4 K3) vs runtime k_pad (cfg2 refined)
for m in 0 7 2 6 3 0 7; do
  echo "=== REXI_L0_KP=$m"
  REXI_L0_KP=$m timeout 300 python bench.py --steps 100 --no-cpu-baseline --secondary 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_s1','l0_k3')})"
done
