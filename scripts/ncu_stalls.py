"""Where the warps of one kernel stall, per SASS instruction and per source
line: python scripts/ncu_stalls.py report.ncu-rep [top]
Prints the source page's column names once (the per-reason columns differ
between ncu versions), then the top instructions by samples with their
stall-reason columns, then per CUDA line the barrier/wait samples."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
print("columns:", h)
idx = {n: i for i, n in enumerate(h)}
reason_cols = [n for n in h if n.startswith("stall_") or "Stall" in n or "stall" in n]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
def num(r, c):
    try: return float(r[idx[c]] or 0)
    except (ValueError, KeyError): return 0.0
samp = "Warp Stall Sampling (All Samples)"
data.sort(key=lambda r: -num(r, samp))
tot = sum(num(r, samp) for r in data) or 1
for r in data[:top]:
    rs = sorted(((num(r, c), c) for c in reason_cols if c != samp and num(r, c) > 0), reverse=True)[:4]
    print(f"{r[0]} {num(r, samp)/tot*100:5.2f}%  {r[1][:60]:60s} " + " ".join(f"{c}={v:.0f}" for v, c in rs))
# opcode totals of samples
ops = collections.Counter()
for r in data:
    p = r[1].split()
    if p: ops[(p[1] if p[0].startswith("@") else p[0]).split(".")[0]] += num(r, samp)
print("samples by opcode:", " ".join(f"{o}:{v/tot*100:.1f}%" for o, v in ops.most_common(15)))
