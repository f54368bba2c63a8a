"""Hot address windows of a kernel from an ncu report's SASS source page:
    python scripts/sass_hot.py report.ncu-rep [window_bytes] [top]"""
import collections, csv, subprocess, sys
rep = sys.argv[1]
W = int(sys.argv[2], 0) if len(sys.argv) > 2 else 0x400
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; idx = {n: i for i, n in enumerate(h)}
data = []
for r in rows[2:]:
    if len(r) < len(h): continue
    data.append((int(r[0], 16), r[1].strip(), int(r[idx["Instructions Executed"]] or 0),
                 int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)))
base = data[0][0]
tot = sum(d[2] for d in data); tots = max(1, sum(d[3] for d in data))
print("warp instructions", tot)
w = collections.Counter(); ws = collections.Counter()
for a, t, i, s in data:
    w[(a - base) // W] += i; ws[(a - base) // W] += s
for k in sorted(w, key=lambda k: -w[k])[:top]:
    print(f"{k * W:#07x}: {w[k] / tot * 100:5.1f}% inst {ws[k] / tots * 100:5.1f}% smp")
