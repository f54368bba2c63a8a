#!/bin/bash
# usage: scripts/ncu_summary.sh <report.ncu-rep>  — key counters + opcode mix + stall reasons
R=$1
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=csv.reader(sys.stdin); h=next(r); units=next(r); vals=next(r)
want=['gpu__time_duration.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__warps_issue_stalled_wait_per_warp_active.pct']
d=dict(zip(h,vals)); u=dict(zip(h,units))
for w in want:
    if w in d: print(w, d[w], u[w])
for n,v in zip(h,vals):
    if 'average_warps_issue_stalled' in n and 'per_issue_active' in n:
        try:
            if float(v)>0.1: print(n.replace('smsp__average_warps_issue_stalled_','stall:'), v)
        except: pass
"
ncu -i $R --page source --csv --print-source sass 2>/dev/null > /tmp/sass_$$.csv
python3 - /tmp/sass_$$.csv <<'PY'
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; idx={n:i for i,n in enumerate(h)}
ops=collections.Counter(); tot=0
for r in rows[2:]:
    if len(r)<len(h): continue
    ins=int(r[idx['Instructions Executed']] or 0)
    p=r[1].split()
    if not p: continue
    op=p[1] if p[0].startswith('@') else p[0]
    ops[op.split('.')[0]]+=ins; tot+=ins
print('warp instructions', tot)
print(' '.join(f"{o}:{c/tot*100:.1f}%" for o,c in ops.most_common(24)))
PY
rm -f /tmp/sass_$$.csv
