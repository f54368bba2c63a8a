"""Time the M=100 batched sweep (north_star target config) with the current
library: python scripts/m100_time.py [K] [M]  (COINFER_THREADS overrides the CTA width)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_06304_b200 import Engine, profile_heavy, sub_seed
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 100
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream())  # events on the launching stream
prof = profile_heavy(M)
u, st = eng.sample(prof, M, sub_seed(1, 1, np.arange(K, dtype=np.uint64)), 0.25, 1.0, device=True)
dev = {k: u[k] for k in ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline"]}
eng.sweep(prof, dev); torch.cuda.synchronize()
ts = []
for _ in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); eng.sweep(prof, dev); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print(f"M={M} K={K} threads={os.environ.get('COINFER_THREADS', 'auto')}: {min(ts):.2f} ms -> {K / min(ts) * 1e3 / 1e6:.3f} M inst/s")
