#!/bin/bash
# K2: the correction sweep's complex64 pivots staged by the CTA's bulk copies (K2_I32=1, +16 KB
# shared memory) vs loaded from HBM inside the sweep (K2_I32=0); cfg2 refined
for v in 0 1 0 1; do
  echo "=== K2_I32=$v"
  REXI_NVCC_EXTRA="-DK2_I32=$v" python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1 || { echo build failed; continue; }
  timeout 300 python bench.py --steps 100 --no-cpu-baseline --secondary 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_s1','l0_k3')})"
done
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persist.py tests/test_gpu_edges.py tests/test_gpu_chain.py tests/test_gpu_hygiene.py -x -q 2>&1 | tail -3
