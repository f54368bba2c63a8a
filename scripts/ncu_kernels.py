"""Key counters of every kernel in an ncu raw CSV export (one row per launch):
python scripts/ncu_kernels.py raw.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
ix = {n: i for i, n in enumerate(h)}
for r in rows[2:]:
    print("kernel", r[ix["Kernel Name"]][:100])
    for w in want:
        if w in ix:
            print(f"  {w} {r[ix[w]]} {units[ix[w]]}")
    stalls = []
    for n, i in ix.items():
        if "average_warps_issue_stalled" in n and "per_issue_active" in n:
            try:
                v = float(r[i])
            except ValueError:
                continue
            if v > 0.1:
                stalls.append((v, n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
    print("  stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))
