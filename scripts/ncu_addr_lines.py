"""Map SASS addresses to CUDA source lines from an ncu 'cuda,sass' source
CSV (ncu -i R --page source --csv --print-source cuda,sass > x.csv), and sum
the stall samples of one reason per source line:
    python scripts/ncu_addr_lines.py x.csv[.gz] [reason=stall_barrier] [top]"""
import csv, collections, gzip, sys
path = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_barrier"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
cur_file = None; hdr = None; cur = None
per_line = collections.Counter(); tot = 0.0; src = {}
for r in csv.reader(f):
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = {n: i for i, n in enumerate(r)}; ri = len(r) - 1 - r[::-1].index(reason) if reason in r else None; continue
    if hdr is None or ri is None: continue
    if r[0] != "":
        cur = (cur_file, r[0]); src[cur] = r[1][:90]; continue
    if r[2].startswith("0x"):
        try: v = float(r[ri] or 0)
        except ValueError: continue
        per_line[cur] += v; tot += v
print(f"{reason}: total {tot:.0f}")
for k, v in per_line.most_common(top):
    print(f"{v/max(tot,1)*100:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')}")
