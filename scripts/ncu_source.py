"""Per-opcode warp-stall samples and executed warp instructions of one kernel, from
`ncu -i X.ncu-rep --page source --csv --print-source sass > X_sass.csv`:
python scripts/ncu_source.py X_sass.csv [top_n_instructions]"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
src = hdr.index("Source")
samp = next(i for i, h in enumerate(hdr) if h.startswith("# Samples") or h.startswith("Warp Stall Sampling (All"))
inst = next(i for i, h in enumerate(hdr) if h.startswith("Instructions Executed") or h == "# Instructions Executed")
def num(s):
    try: return float(s.replace(",", ""))
    except ValueError: return 0.0
ops = collections.defaultdict(lambda: [0.0, 0.0])
lines = []
for r in rows[hi + 1:]:
    if len(r) <= max(src, samp, inst): continue
    toks = r[src].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    s, n = num(r[samp]), num(r[inst])
    ops[op][0] += s; ops[op][1] += n
    lines.append((s, n, r[src]))
tot = sum(v[0] for v in ops.values()) or 1.0
totn = sum(v[1] for v in ops.values())
print(f"total stall samples {tot:.0f}, warp instructions {totn:.0f}")
for op, (s, n) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:16]:
    print(f"  {op:8s} stall samples {100 * s / tot:5.1f} %   warp instructions {n:12.0f}")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for i, (s, n, t) in enumerate(lines):
    pass
if top:
    print(f"top {top} instructions by stall samples (index in kernel, samples %, text):")
    for s, n, t, i in sorted(((s, n, t, i) for i, (s, n, t) in enumerate(lines)), reverse=True)[:top]:
        print(f"  [{i:5d}] {100 * s / tot:5.2f} %  {t.strip()[:110]}")
