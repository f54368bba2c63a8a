"""C5 (BASELINE.json configs[4]): online episodes, TW(0, OG), 10^5 slots.
usage: python scripts/bench_online.py [episodes] [horizon] [heavy|light] [tw|local]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_06304_b200 import Engine, profile_heavy, profile_light, sample_batch
from paper_2206_06304_b200.engine import OnlineConfig
E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
H = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
kind = sys.argv[3] if len(sys.argv) > 3 else "heavy"
M = 14
prof = profile_heavy(M) if kind == "heavy" else profile_light(M)
lo, hi, p = (0.25, 1.0, 0.05) if kind == "heavy" else (0.05, 0.2, 0.25)
users = sample_batch(1, M, prof, hi, hi, seed=7)  # the CLI: sample_scenario(users, fixed(l_high))
policy = sys.argv[4] if len(sys.argv) > 4 else "tw"
cfg = OnlineConfig("bernoulli", p, lo, hi, 0.025, "og", policy, 0, None, H)
eng = Engine(0)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
seeds = torch.arange(1, E + 1, dtype=torch.int64, device="cuda")
eng.online(prof, dev, OnlineConfig(**{**cfg.__dict__, "horizon": 100}), seeds[:256]); torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); out = eng.online(prof, dev, cfg, seeds); e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e)
c = out["counts"].cpu().numpy()
print(f"{kind}: {E} episodes x {H} slots in {ms:.1f} ms -> {E/(ms/1e3):.1f} episodes/s, "
      f"{E*H/(ms/1e3)/1e9:.3f} G slot/s; mean OG calls/episode {c[:,1].mean():.0f}, "
      f"tasks/call {c[:,2].sum()/max(c[:,1].sum(),1):.2f}, status ok {(out['status']==0).all().item()}")
