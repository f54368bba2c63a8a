"""Development: where the pipelined kernel's teams wait (needs a -DCFB_PIPE_PROF
build via COINFER_LIB): python scripts/pipe_prof.py [instances] [M]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_06304_b200 import Engine, profile_heavy, sub_seed, _abi
K = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 50
eng = Engine(0)
prof = profile_heavy(M)
users, st = eng.sample(prof, M, sub_seed(1, 1, np.arange(K, dtype=np.uint64)), 0.25, 1.0, device=True)
dev = {k: users[k] for k in ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline"]}
eng.sweep(prof, dev); torch.cuda.synchronize()
lib = _abi.load_library()
buf = (C.c_ulonglong * 4)()
lib.coinfer_debug_pipe_cycles(buf, 1)
eng.sweep(prof, dev); torch.cuda.synchronize()
lib.coinfer_debug_pipe_cycles(buf, 1)
n = K
print(f"per instance (cycles, warp 0 of each team): G wait {buf[0]/n:.0f}  G busy {buf[1]/n:.0f}  "
      f"front/tail wait {buf[2]/n:.0f}  front/tail busy {buf[3]/n:.0f}")
