import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
M, K, lo, hi = 50, 64, int(sys.argv[1]), int(sys.argv[2])
prof = profile_heavy(M)
u = sample_batch(K, M, prof, 0.25, 1.0, seed=M)
u = {k: v[lo:hi] for k, v in u.items()}
eng = Engine(0)
og = eng.og(prof, u)
print("ok", og["status"])
'''
def run(lo, hi):
    try:
        r = subprocess.run([sys.executable, "-c", code, str(lo), str(hi)], capture_output=True, text=True, timeout=25)
        return r.returncode == 0 and "ok" in r.stdout
    except subprocess.TimeoutExpired:
        return False
lo, hi = 0, 64
print("whole", run(0, 64), flush=True)
while hi - lo > 1:
    mid = (lo + hi) // 2
    if not run(lo, mid): hi = mid
    elif not run(mid, hi): lo = mid
    else:
        print("both halves pass: interaction?", lo, mid, hi); break
print("failing range", lo, hi, flush=True)
