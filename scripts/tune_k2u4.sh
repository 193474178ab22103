#!/bin/bash
# K2 at 4 CTAs/SM: residual-loop unroll and L2-prefetch distance (cfg2 refined)
run() { timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_k3')})"; }
for u in 3 7; do
  echo "=== -DK2_RES_UNROLL=$u"
  REXI_NVCC_EXTRA="-DK2_RES_UNROLL=$u" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  run
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
for pf in 0 0.5 1 2; do echo "=== REXI_K2_PF=$pf"; REXI_K2_PF=$pf run; done
