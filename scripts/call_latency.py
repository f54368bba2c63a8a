import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 10
prof = profile_heavy(M)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(1, M, prof, 0.25, 1.0, seed=7).items()}
fn = eng.ipssa if M == 10 else eng.og
for _ in range(3): fn(prof, dev)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): fn(prof, dev)
torch.cuda.synchronize()
print(f"M={M}: {(time.perf_counter()-t)/20*1e6:.1f} us wall per call")
