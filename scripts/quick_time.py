import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 50
eng = Engine(0)
print("fp64 peak lane-ops/s", eng.fp64_peak())
prof = profile_heavy(M)
t = time.time(); users = sample_batch(K, M, prof, seed=1); print("gen", time.time() - t)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
for mode in ["sweep", "og", "ipssa"]:
    for rep in range(3):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if mode == "sweep": eng.sweep(prof, dev)
        elif mode == "og": eng.og(prof, dev)
        else: eng.ipssa(prof, dev)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        print(f"{mode} K={K} M={M}: {ms:.2f} ms  -> {K/ms*1e3:.0f} inst/s")
