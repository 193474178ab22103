#!/bin/bash
# All configs through bench.py (1 GPU) + the reference arm for cfg 1/2 + smoke.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
python bench.py --config 1 --steps 2000 --warmup 10 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1 rc=$?"
python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_cfg2_ref.json 2>&1; echo "ref2 rc=$?"
python bench.py --impl reference --config 1 --steps 200 --warmup 3 > gpurun_out/bench_cfg1_ref.json 2>&1; echo "ref1 rc=$?"
for f in gpurun_out/bench_cfg*.json; do
  python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "unreadable", e); sys.exit()
r = d.get("roofline") or {}
print(f.split("/")[-1], "value=%.4g" % d["value"], "ms/step=%.4g" % d["ms_per_step"],
      "e2e=%s" % ((d.get("e2e") or {}).get("value")), "roof=%s %.3g" % (r.get("kernel"), r.get("frac") or 0),
      "cpu=%s" % ((d.get("cpu_baseline") or {}).get("value")), "clocks=%s" % d.get("clocks"))
PY
done
