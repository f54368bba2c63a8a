"""List the loops (backward branches) of one kernel's SASS with their
instruction mix: python scripts/sass_loops.py file.sass [min_len]."""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ins = []
for l in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, t) in enumerate(ins):
    m = re.search(r"\bBRA\b.*?0x([0-9a-f]+)", t)
    if m:
        tgt = int(m.group(1), 16)
        if tgt <= a and tgt in addr:
            loops.append((addr[tgt], i))
for lo, hi in sorted(set(loops)):
    body = ins[lo:hi + 1]
    if len(body) < minlen:
        continue
    ops = Counter()
    for _, t in body:
        t = re.sub(r"^@!?U?P[T0-9]+\s+", "", t)
        ops[t.split()[0].split(".")[0]] += 1
    fp64 = sum(v for k, v in ops.items() if k in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"))
    print(f"loop {body[0][0]:#06x}-{body[-1][0]:#06x}: {len(body)} inst, fp64 {fp64} "
          f"({100*fp64/len(body):.0f}%)  " + " ".join(f"{k}:{v}" for k, v in ops.most_common(18)))
