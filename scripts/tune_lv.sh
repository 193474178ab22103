#!/bin/bash
# reduced-level kernel CTAs/SM (register cap vs spills), cfg2 refined
for mb in 3 2; do
  echo "=== LV_MINB=$mb"
  REXI_NVCC_EXTRA="-DLV_MINB=$mb" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if 'lv' in k})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
