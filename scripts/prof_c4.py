import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
prof = profile_heavy(M)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(1, M, prof, 0.25, 1.0, seed=7).items()}
eng.og(prof, dev); torch.cuda.synchronize()
