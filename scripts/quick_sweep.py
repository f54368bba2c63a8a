"""One C3 sweep launch (K instances, M=50, device inputs) for profiling."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_06304_b200 import Engine, profile_heavy, sub_seed
K = int(sys.argv[1]) if len(sys.argv) > 1 else 300000
eng = Engine(0)
prof = profile_heavy(50)
users, st = eng.sample(prof, 50, sub_seed(1, 1, np.arange(K, dtype=np.uint64)), 0.25, 1.0, device=True)
dev = {k: users[k] for k in ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline"]}
eng.sweep(prof, dev)
torch.cuda.synchronize()
