#!/bin/bash
# K3 (complex64 correction) CTAs/SM sweep on cfg2 (refined)
for mb in 5 6 8; do
  echo "=== K3_MINB=$mb"
  REXI_NVCC_EXTRA="-DK3_MINB=$mb" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value'],1), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k.startswith('l0')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
