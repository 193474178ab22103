#!/bin/bash
# K3: the dd partial's four words loaded before the lane loop (HEAD) -- cfg2 refined, three runs
python paper_1912_03312_b200/build_native.py --force > /dev/null 2>&1
for v in 1 2 3; do
  timeout 300 python bench.py --steps 100 --no-cpu-baseline --secondary 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(round(d['value'],1), round(d['ms_per_step'],4), {k:round(v['total_ms']/100,4) for k,v in d['kernels'].items() if k in ('l0_k2','l0_s1','l0_k3')})"
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_persist.py tests/test_gpu_edges.py tests/test_gpu_chain.py tests/test_gpu_distributed.py -x -q 2>&1 | tail -3
