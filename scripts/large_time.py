"""Cycle split of the large path's short-row DP stages (needs a -DCFB_LARGE_TIMING build via COINFER_LIB)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch, _abi
eng = Engine(0)
M = 4096
prof = profile_heavy(M)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(1, M, prof, 0.25, 1.0, seed=7).items()}
eng.og(prof, dev); torch.cuda.synchronize()
buf = (C.c_ulonglong * 8)()
_abi.load_library().coinfer_debug_large_times(buf)
n = buf[3]
if n:
  print(f"short stages {n}, staged from global {buf[4]}; cycles per stage: setup+column {buf[0]/n:.0f}, "
        f"wait for G/pfit {buf[1]/n:.0f}, cells+sync {buf[2]/n:.0f}")
if buf[7]:
    print(f"fast DP stages {buf[7]}: cycles per stage issue+wait+read G/pfit {buf[5]/buf[7]:.0f}, "
          f"cells+stores+sync {buf[6]/buf[7]:.0f}")
