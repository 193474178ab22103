"""Fold a profile_round.sh run (gpurun_out/) into profiles/: per-kernel raw summaries,
FP64 instruction counts, SASS-level stall summaries, and profiles/ncu_traffic.json
(what bench.py reads for roofline.traffic / fp64): python scripts/update_profiles.py TAG"""
import collections, csv, json, os, re, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
N2, K2 = 1048574, 64

shutil.copy(os.path.join(G, "ncu_raw_summaries.txt"), os.path.join(P, f"{tag}_ncu_raw_summaries.txt"))
shutil.copy(os.path.join(G, "l0_fp64_counts.csv"), os.path.join(P, f"{tag}_l0_fp64_counts.csv"))
shutil.copy(os.path.join(G, "launches_cfg2.csv"), os.path.join(P, f"{tag}_launches_cfg2.csv"))
with open(os.path.join(P, f"{tag}_launches_cfg2_summary.txt"), "w") as fh:
    fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 2 --warmup 1 (cfg 2)\n")
    fh.write(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), "launches",
                             os.path.join(G, "launches_cfg2.csv")], capture_output=True, text=True).stdout)
for k in ("k2", "k3", "s1"):
    src = os.path.join(G, f"cfg2_k_l0_{k}_sass.csv")
    if os.path.exists(src):
        out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_source.py"), src, "12"],
                             capture_output=True, text=True).stdout
        with open(os.path.join(P, f"{tag}_l0_{k}_sass_summary.txt"), "w") as fh:
            fh.write(f"# ncu --set full --import-source on, scripts/cfg_step.py 2, one k_l0_{k} launch: warp-stall samples "
                     "and executed warp instructions by SASS opcode, top instructions\n" + out)
for f in os.listdir(G):
    if f.endswith("_details.csv"):
        shutil.copy(os.path.join(G, f), os.path.join(P, f"{tag}_{f}"))

# FP64 thread-instruction counts per level-0 kernel
rows = list(csv.reader(open(os.path.join(G, "l0_fp64_counts.csv"))))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
kn, mn, mv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
cnt = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) > mv:
        cnt[r[kn]][r[mn]] = float(r[mv].replace(",", ""))
# raw summaries: name -> (us, read, write, fp64 pct)
raw = {}
for line in open(os.path.join(G, "ncu_raw_summaries.txt")):
    m = re.match(r"(?:void )?(\S+?)(?:<.*?>)?: time_duration.sum=([\d.]+) (\w+) \| bytes_read.sum=([\d.]+) (\w+) \| bytes_write.sum=([\d.]+) (\w+)", line)
    if not m:
        continue
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    us = float(m.group(2)) * (1e3 if m.group(3) == "ms" else 1.0)
    pct = re.search(r"pipe_fp64_cycles_active[^=]*=([\d.]+)", line)
    raw.setdefault(m.group(1), (us, float(m.group(4)) * scale[m.group(5)], float(m.group(6)) * scale[m.group(7)],
                                float(pct.group(1)) if pct else None))
path = os.path.join(P, "ncu_traffic.json")
tr = json.load(open(path))
def put(key, kname, config, note):
    if kname not in raw:
        print("missing capture:", kname); return
    us, rd, wr, pct = raw[kname]
    e = tr.setdefault(key, {})
    e.update({"dram_bytes": int(rd + wr), "fp64_pipe_pct": pct, "config": config,
              "capture": f"profiles/{tag}_ncu_raw_summaries.txt ({note}: {us:.0f} us, dram read {rd/1e9:.3f} GB + write {wr/1e9:.3f} GB)"})
put("l0_k2", "k_l0_k2", 2, "ncu --set full, cfg2 refine=1, one k_l0_k2 launch")
put("l0_k3", "k_l0_k3", 2, "ncu --set full, cfg2 refine=1, one k_l0_k3 launch")
put("l0_s1", "k_l0_s1", 2, "ncu --set full, cfg2 refine=1, one k_l0_s1 launch")
put("cg_spmv", "k_cg_spmv_win", 3, "ncu --set full, cfg3, one width-64 launch of the windowed spmv (first capture in the file)")
put("cg_update", "k_cg_update_tma", 3, "ncu --set full, cfg3, one width-64 launch of the TMA update")
for key, pat in (("l0_k2", "k_l0_k2"), ("l0_k3", "k_l0_k3"), ("l0_s1", "k_l0_s1")):
    for name, mm in cnt.items():
        if pat in name:
            f = sum(v for k, v in mm.items() if "inst_executed_op_d" in k)
            tr[key]["fp64_inst"] = int(f)
            tr[key]["fp64_inst_per_row_shift"] = round(f / (N2 * K2), 2)
            tr[key]["fp64_inst_src"] = (f"profiles/{tag}_l0_fp64_counts.csv (smsp__sass_thread_inst_executed_op_"
                                        "{dadd,dfma,dmul}_pred_on.sum, one cfg2 launch)")
json.dump(tr, open(path, "w"), indent=2)
print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "capture"} for k, v in tr.items()}, indent=1))
