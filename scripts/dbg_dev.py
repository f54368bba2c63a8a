import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
K = int(sys.argv[1]); mode = sys.argv[2]
eng = Engine(0)
prof = profile_heavy(50)
u = sample_batch(K, 50, prof, seed=1)
if sys.argv[3] == "dev":
    u = {k: torch.as_tensor(v, device="cuda") for k, v in u.items()}
out = eng.og(prof, u) if mode == "og" else eng.sweep(prof, u)
torch.cuda.synchronize()
print("ok")
