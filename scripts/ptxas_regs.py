"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills (stdin)."""
import re, sys
fn = None
rows = []
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and fn:
        rows.append((fn, int(m.group(1)), spill))
        fn, spill = None, ""
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for fn, r, sp in rows:
    if pat in fn:
        print(f"{r:4d} {sp:16s} {fn}")
