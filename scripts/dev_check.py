"""Quick parity + timing of a development library (COINFER_LIB) on C3-shaped
N=4 batches: the CUDA engine vs the C oracle, bit for bit."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import checkers as ck
from paper_2206_06304_b200 import Engine, profile_heavy, profile_light, sample_batch
eng = Engine(0)
for M, K, light in [(50, 512, False), (20, 512, False), (14, 256, True), (100, 64, False), (7, 256, False)]:
    prof = profile_light(M) if light else profile_heavy(M)
    u = sample_batch(K, M, prof, 0.05 if light else 0.25, 0.2 if light else 1.0, seed=M)
    ip, og = eng.sweep(prof, u)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, u), where=f"M={M}")
    ck.assert_same_og(og, ck.oracle_og(prof, u), where=f"M={M}")
    print(f"parity ok M={M} K={K} light={light}")
K = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
prof = profile_heavy(50)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(K, 50, prof, seed=1).items()}
for mode in ["sweep", "og", "ipssa"]:
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if mode == "sweep": eng.sweep(prof, dev)
        elif mode == "og": eng.og(prof, dev)
        else: eng.ipssa(prof, dev)
        e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"{mode} K={K}: {best:.2f} ms -> {K/best*1e3:.0f} inst/s")
