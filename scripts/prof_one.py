"""One solve launch for ncu: python scripts/prof_one.py K [mode]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
mode = sys.argv[2] if len(sys.argv) > 2 else "og"
eng = Engine(0)
prof = profile_heavy(50)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(K, 50, prof, seed=1).items()}
if mode == "og": eng.og(prof, dev)
elif mode == "ipssa": eng.ipssa(prof, dev)
else: eng.sweep(prof, dev)
torch.cuda.synchronize()
