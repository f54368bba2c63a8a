import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
M = 4096
prof = profile_heavy(M)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(1, M, prof, 0.25, 1.0, seed=7).items()}
for _ in range(2): eng.og(prof, dev)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); eng.og(prof, dev); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
print(f"C4 M=4096: best {min(ts):.3f} ms median {sorted(ts)[2]:.3f} ms  lib={os.environ.get('COINFER_LIB','default')}")
