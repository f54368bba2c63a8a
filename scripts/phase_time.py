"""Per-phase SM cycles of the fused kernel (needs a -DCFB_PHASE_TIMING build via COINFER_LIB):
python scripts/phase_time.py [instances] [M]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch, _abi
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
M = int(sys.argv[2]) if len(sys.argv) > 2 else 50
eng = Engine(0)
prof = profile_heavy(M)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(K, M, prof, seed=1).items()}
eng.sweep(prof, dev); torch.cuda.synchronize()
buf = (C.c_ulonglong * 18)()
lib = _abi.load_library()
lib.coinfer_debug_phase_cycles(buf, 1)
eng.sweep(prof, dev); torch.cuda.synchronize()
lib.coinfer_debug_phase_cycles(buf, 1)
names = ["rows/pools/pfit", "G table", "IP-SSA out", "DP", "group folds/final", "check/sort/hoist"]
tot = sum(buf[:6])
for i in [5, 0, 1, 2, 3, 4]:
    print(f"{names[i]:24s} {buf[i]/K:12.0f} cycles/instance  {buf[i]/tot*100:5.1f}%")
if buf[7]:
    print(f"G phase: {buf[6]/K:.0f} active lane-steps/instance, {buf[7]/K:.0f} warp-steps/instance, "
          f"lane utilisation {buf[6]/(32*buf[7])*100:.1f}%")
if buf[9]:
    print(f"IP-SSA G loop: {buf[8]/K:.0f} active lane-steps/instance, {buf[9]/K:.0f} warp-steps/instance, "
          f"lane utilisation {buf[8]/(32*buf[9])*100:.1f}%")
tn = ["best_i/order", "backtrack/gid", "gitem/b*/gbest", "stitch", "front: check", "front: rank/rec/lat", "front: b0/rlen/init"]
if any(buf[10:17]):
    for i in range(7):
        print(f"  tail {tn[i]:20s} {buf[10 + i]/K:10.0f} cycles/instance")
