"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck):
python scripts/sanitize_smoke.py [large]   ("large": only the large-instance path)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import checkers as ck
from paper_2206_06304_b200 import Engine, profile_heavy, profile_light, sample_batch
from paper_2206_06304_b200.engine import OnlineConfig
eng = Engine(0)
ONLY_LARGE = sys.argv[1:] == ["large"]
for M, K, lo, hi in [] if ONLY_LARGE else [(50, 64, 0.25, 1.0), (20, 32, 0.5, 3.0), (100, 4, 0.25, 1.0), (176, 1, 0.5, 3.0), (7, 300, 0.25, 1.0)]:
    prof = profile_heavy(M)
    u = sample_batch(K, M, prof, lo, hi, seed=M)
    ip, og = eng.sweep(prof, u)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, u)); ck.assert_same_og(og, ck.oracle_og(prof, u))
    print("small path ok", M, K, flush=True)
# the pipelined persistent kernel (K >= 2048, M <= 64): teams, named barriers,
# mbarriers, the L2 G tables
for M, K, lo, hi, light in [] if ONLY_LARGE else [(50, 2100, 0.25, 1.0, False), (20, 2048, 0.05, 0.2, True), (64, 2048, 0.25, 1.0, False),
                             (100, 2048, 0.25, 1.0, False)]:
    prof = profile_light(M) if light else profile_heavy(M)
    u = sample_batch(K, M, prof, lo, hi, seed=M + 7)
    ip, og = eng.sweep(prof, u)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, u)); ck.assert_same_og(og, ck.oracle_og(prof, u))
    print("pipelined path ok", M, K, flush=True)
# large_dp (two warps, cp.async ring, named barriers) and large_finish
for M, lo, hi, light in [(300, 0.5, 3.0, False), (260, 0.25, 1.0, False), (300, 0.05, 0.2, True)]:
    prof = profile_light(M) if light else profile_heavy(M)
    u = sample_batch(1, M, prof, lo, hi, seed=M)
    ip, og = eng.sweep(prof, u)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, u)); ck.assert_same_og(og, ck.oracle_og(prof, u))
    print("large path ok", M, flush=True)
for kind, M, p in [] if ONLY_LARGE else [("heavy", 14, 0.05), ("light", 14, 0.25), ("heavy", 32, 0.3), ("heavy", 40, 0.2)]:
    prof = profile_heavy(M) if kind == "heavy" else profile_light(M)
    hi = 1.0 if kind == "heavy" else 0.2
    users = sample_batch(1, M, prof, hi, hi, seed=M)
    cfg = OnlineConfig("bernoulli", p, 0.25 if kind == "heavy" else 0.05, hi, 0.025, "og", "tw", 0, None, 600)
    out = eng.online(prof, users, cfg, [1, 2, 3])
    assert (np.asarray(out["status"]) == 0).all()
    print("online ok", kind, M, flush=True)
print("sanitize smoke done")
