"""Small fixed workload for ncu: warm-up solve, then the profiled solves."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 50
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
eng = Engine(0)
prof = profile_heavy(M)
users = sample_batch(K, M, prof, seed=1)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
for _ in range(reps):
    eng.sweep(prof, dev)
torch.cuda.synchronize()
print("done")
