"""Per-source-line instruction and stall-sample shares from an ncu report."""
import csv, collections, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = collections.defaultdict(lambda: [0, 0]); cur_file = None; hdr = None; cur = None; tot = 0; tots = 0
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None: continue
    if r[0] != '': cur = (cur_file, r[0], r[1][:80])
    if len(r) > 7 and r[2] != '':
        try: ins = int(r[7] or 0); smp = int(r[4] or 0)
        except ValueError: continue
        res[cur][0] += ins; res[cur][1] += smp; tot += ins; tots += smp
for k, v in sorted(res.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]/tot*100:5.1f}% inst {v[1]/max(tots,1)*100:5.1f}% smp  {k[0]}:{k[1]}  {k[2]}")
