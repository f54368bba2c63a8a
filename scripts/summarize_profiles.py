"""Write profiles/<tag>_launches.txt, <tag>_ncu_full_solve_small.txt and
profiles/ncu_summary.json from gpurun_out captures:
python scripts/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep>"""
import csv, json, subprocess, sys
from collections import defaultdict
tag, lcsv, rep = sys.argv[1:4]
lines = [l for l in open(lcsv) if not l.startswith("==")]
rows = list(csv.reader(lines))
h = rows[0]; ix = {n: i for i, n in enumerate(h)}
out = []
for r in rows[1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    u = r[ix["Metric Unit"]]
    ms = v / 1e6 if u == "ns" else (v / 1e3 if u == "us" else v)
    out.append((r[ix["Kernel Name"]], r[ix["Grid Size"]], r[ix["Block Size"]], ms))
tot = sum(o[3] for o in out)
agg = defaultdict(lambda: [0, 0.0])
for k, g, b, ms in out:
    agg[k][0] += 1; agg[k][1] += ms
with open(f"profiles/{tag}_launches.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 1 --no-cpu-baseline\n")
    f.write("# (cold, serialised per-launch times; shares matter, not absolutes)\n")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{ms:10.3f} ms  {ms/tot*100:5.1f}%  x{n:3d}  {k[:120]}\n")
    f.write("\n# launch list\n")
    for k, g, b, ms in out:
        f.write(f"{ms:10.3f} ms grid {g} block {b} {k[:120]}\n")
summ = subprocess.run(["bash", "scripts/ncu_summary.sh", rep], capture_output=True, text=True).stdout
lines_ = subprocess.run([sys.executable, "scripts/ncu_lines.py", rep, "40"], capture_output=True, text=True).stdout
with open(f"profiles/{tag}_ncu_full_solve_small.txt", "w") as f:
    f.write("# ncu --set full --clock-control none -k regex:solve_small -c 1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline\n")
    f.write("# one launch = 1,000,000 C3 instances (IP-SSA + OG), N=4, M=50\n")
    f.write(summ + lines_)
d = {}
for l in summ.splitlines():
    p = l.split()
    if len(p) >= 2:
        try: d[p[0]] = float(p[1])
        except ValueError: pass
js = {"kernel": "cfb::solve_small_kernel<4>", "launch": "1,000,000 C3 instances (IP-SSA+OG), M=50, N=4",
      "gpu_time_ms": d["gpu__time_duration.sum"],
      "dram_bytes_read": d["dram__bytes_read.sum"] * 1e9, "dram_bytes_write": d["dram__bytes_write.sum"] * 1e9,
      "dram_bytes_per_launch_at_1M": (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) * 1e9,
      "algorithmic_io_bytes_at_1M": 2.8e9,
      "fp64_pipe_active_pct": d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed"],
      "issue_active_pct": d["smsp__issue_active.avg.pct_of_peak_sustained_active"],
      "registers": int(d["launch__registers_per_thread"]),
      "occupancy_warps_pct": d["sm__warps_active.avg.pct_of_peak_sustained_active"],
      "source": f"profiles/{tag}_ncu_full_solve_small.txt"}
json.dump(js, open("profiles/ncu_summary.json", "w"), indent=1)
print(open(f"profiles/{tag}_launches.txt").read()[:600]); print(js)
