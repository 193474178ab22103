#!/bin/bash
# K2: L2-prefetch of the next wave's complex64 pivot tile (K2_PF32) on/off; cfg2 refined
for v in 0 1 0 1; do
  echo "=== K2_PF32=$v"
  REXI_NVCC_EXTRA="-DK2_PF32=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline --secondary 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_s1','l0_k3')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
