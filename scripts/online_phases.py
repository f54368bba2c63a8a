"""Per-phase SM cycles of solve_one inside the online driver (C5 light), per
solver call; needs a -DCFB_PHASE_TIMING build of online.cu via COINFER_LIB."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_light, sample_batch, _abi
from paper_2206_06304_b200.engine import OnlineConfig
eng = Engine(0)
M, E, H = 14, 1024, 20000
prof = profile_light(M)
users = sample_batch(1, M, prof, 0.2, 0.2, seed=7)
cfg = OnlineConfig("bernoulli", 0.25, 0.05, 0.2, 0.025, "og", "tw", 0, None, H)
lib = _abi.load_library()
buf = (C.c_ulonglong * 10)()
lib.coinfer_debug_online_phase_cycles(buf, 1)
out = eng.online(prof, users, cfg, list(range(1, E + 1)))
torch.cuda.synchronize()
lib.coinfer_debug_online_phase_cycles(buf, 1)
calls = int(out["counts"][:, 1].sum())
names = ["rows/pools/pfit", "G table", "IP-SSA out", "DP", "stitch (+b* when no submarks)", "check/sort/hoist", "best_i/backtrack", "b*"]
for i in [5, 0, 1, 2, 3, 6, 7, 4]:
    print(f"{names[i]:24s} {buf[i]/calls:10.0f} cycles/call")
print("calls", calls)
