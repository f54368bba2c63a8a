"""Every source line of an ncu report with its executed warp instructions and
stall samples (CSV: file,line,inst,samples,source), for phase attribution:
python scripts/ncu_linedump.py report.ncu-rep > lines.csv"""
import csv, collections, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res = collections.defaultdict(lambda: [0, 0]); cur_file = None; hdr = None; cur = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None: continue
    if r[0] != '': cur = (cur_file, int(r[0]) if r[0].isdigit() else -1, r[1][:100])
    if len(r) > 7 and r[2] != '':
        try: ins = int(r[7] or 0); smp = int(r[4] or 0)
        except ValueError: continue
        res[cur][0] += ins; res[cur][1] += smp
w = csv.writer(sys.stdout)
w.writerow(["file", "line", "inst", "samples", "source"])
for k, v in sorted(res.items(), key=lambda kv: (kv[0][0] or "", kv[0][1])):
    if v[0] or v[1]:
        w.writerow([k[0], k[1], v[0], v[1], k[2]])
