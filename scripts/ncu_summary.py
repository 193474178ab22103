"""Summarise ncu captures: python scripts/ncu_summary.py raw <rep>  |  launches <csv> [first last n]"""
import csv, collections, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_op_read_hit_rate.pct", "sm__warps_active.avg.per_cycle_active",
            "launch__registers_per_thread", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "launch__grid_size"]
    st = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        t = float(r[hdr.index("gpu__time_duration.sum")]) * (1e-3 if units[hdr.index("gpu__time_duration.sum")] == "usecond" else 1.0)
        rd = float(r[hdr.index("dram__bytes_read.sum")]); wr = float(r[hdr.index("dram__bytes_write.sum")])
        print(f"{name}: " + " | ".join(f"{w.split('__')[-1]}={r[hdr.index(w)]} {units[hdr.index(w)]}" for w in want if w in hdr))
        vals = sorted(((float(r[i]) if r[i] else 0.0, hdr[i][34:-23]) for i in st), reverse=True)[:5]
        print("   stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in vals))

def launches(path, first=None, last=None, nlast=1):
    """Per-kernel totals of a launch list; optionally only the launches from
    the first one whose name contains `first` through the `nlast`-th one whose
    name contains `last` (e.g. the device-resident steps of a run)."""
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr = r; start = i + 1; break
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    on, seen = first is None, 0
    for r in rows[start:]:
        if len(r) <= vi: continue
        name = r[ki].split("(")[0]
        if not on and first in name: on = True
        if not on: continue
        v = float(r[vi].replace(",", "")); u = r[ui]
        v = v / 1e6 if u in ("nsecond", "ns") else (v / 1e3 if u in ("usecond", "us") else (v if u in ("msecond", "ms") else v * 1e3))
        a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += v
        if last is not None and last in name:
            seen += 1
            if seen >= nlast: break
    tot = sum(t for _, t in agg.values())
    for k, (c, t) in agg.items():
        print(f"{k:28s} {c:6d} launches {t:10.3f} ms  ({100*t/tot:5.1f}%)  avg {1e3*t/c:9.1f} us")

if __name__ == "__main__":
    if sys.argv[1] == "launches" and len(sys.argv) > 3:
        launches(sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]))
    else:
        {"raw": raw, "launches": launches}[sys.argv[1]](sys.argv[2])
