#!/bin/bash
# K2 residual-loop unroll (after the complex64 correction freed registers), cfg2 refined
for u in 3 5 15; do
  echo "=== K2_RES_UNROLL=$u"
  REXI_NVCC_EXTRA="-DK2_RES_UNROLL=$u" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k.startswith('l0')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
