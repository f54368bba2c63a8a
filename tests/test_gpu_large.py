"""The large-instance path (solve_large.cu: global-memory G/S, one warp per
row; the DP in large_dp -- two DP warps and a producer warp -- when every
row has <= 96 useful cells and its shared memory fits, else the
change-point DP of large_finish) — BASELINE config 4 (M = 4096 in one
instance).

Parity: vs the C oracle at M in the hundreds, and vs the (fixture-validated)
shared-memory path on many small instances by forcing the large path."""
import os
import subprocess
import sys

import numpy as np
import pytest

import checkers as ck
from paper_2206_06304_b200 import profile_heavy, profile_light, sample_batch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("M", [256, 300])
def test_large_vs_oracle(engine, M):
    prof = profile_heavy(M)
    users = sample_batch(2, M, prof, 0.25, 1.0, seed=M)
    ip, og = engine.sweep(prof, users)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, users), where="large ipssa")
    ck.assert_same_og(og, ck.oracle_og(prof, users), where="large og")


def test_large_loose_deadlines(engine):
    """Loose deadlines: many rows keep more than 64 useful cells, so the DP
    runs its whole-CTA stages as well as the single-warp ones."""
    M = 300
    prof = profile_heavy(M)
    users = sample_batch(2, M, prof, 0.5, 3.0, seed=11)
    sl = np.zeros(M + 1)
    for n in range(prof.N):
        sl[1:] = sl[1:] + prof.latency[n][:M]
    dl = np.sort(users["deadline"][0])
    rlen = [int(np.sum(dl[0] + sl[1:M - i + 1] <= dl[i])) for i in range(1, M)]
    assert sum(r > 64 for r in rlen) > 50 and sum(r <= 64 for r in rlen) > 50
    ip, og = engine.sweep(prof, users)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, users), where="large loose ipssa")
    ck.assert_same_og(og, ck.oracle_og(prof, users), where="large loose og")


def test_large_batch_streams_and_device_deadlines(engine):
    """A batch of large instances runs round-robin on the large-path streams
    (one workspace each): every instance equals the oracle, from host and
    from device memory, with per-instance IP-SSA deadlines read on the device."""
    import torch
    M, K = 200, 20
    prof = profile_heavy(M)
    users = sample_batch(K, M, prof, 0.25, 1.0, seed=21)
    dl = users["deadline"].min(axis=1) * np.linspace(1.0, 1.4, K)
    ipx = ck.oracle_ipssa(prof, users, deadline=dl)
    ogx = ck.oracle_og(prof, users)
    ck.assert_same_ip(engine.ipssa(prof, users, deadline=dl), ipx, where="large batch ipssa (host)")
    ck.assert_same_og(engine.og(prof, users), ogx, where="large batch og (host)")
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
    ipd = engine.ipssa(prof, dev, deadline=torch.as_tensor(dl, device="cuda"))
    ogd = engine.og(prof, dev)
    engine.synchronize()
    ck.assert_same_ip({k: v.cpu().numpy() for k, v in ipd.items()}, ipx, where="large batch ipssa (device)")
    ck.assert_same_og({k: v.cpu().numpy() for k, v in ogd.items()}, ogx, where="large batch og (device)")


def test_large_light_profile(engine):
    prof = profile_light(400)
    users = sample_batch(1, 400, prof, 0.05, 0.2, seed=5)
    og = engine.og(prof, users)
    ck.assert_same_og(og, ck.oracle_og(prof, users), where="large light og")


def test_forced_large_path_matches_small_path():
    """Run the golden fixtures and random batches through the large path in a
    subprocess (COINFER_FORCE_LARGE is read once per process)."""
    code = r'''
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import checkers as ck, golden_io
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
n = 0
for c in golden_io.all_cases():
    if c["kind"] == "fixed":
        continue
    if c["kind"] == "ipssa":
        ck.assert_same_ip(eng.ipssa(c["profile"], c["users"], c["deadline"]), c["expect"], where=c["name"])
    else:
        ck.assert_same_og(eng.og(c["profile"], c["users"]), c["expect"], where=c["name"])
    n += 1
prof = profile_heavy(60)
u = sample_batch(64, 60, prof, seed=9)
ip, og = eng.sweep(prof, u)
ck.assert_same_ip(ip, ck.oracle_ipssa(prof, u)); ck.assert_same_og(og, ck.oracle_og(prof, u))
print("forced-large ok", n)
'''
    env = dict(os.environ, COINFER_FORCE_LARGE="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "forced-large ok" in r.stdout


def test_c4_shape_properties(engine):
    """M = 4096 (config 4) on a second instance stream: runs, and the plan is
    internally consistent (energy = left fold of the group energies, groups
    cover the users in deadline order).  Bit-exact C4 parity against the
    O(M^3 N) oracle is tests/test_large_golden.py."""
    M = 4096
    prof = profile_heavy(M)
    users = sample_batch(1, M, prof, 0.25, 1.0, seed=4)
    og = engine.og(prof, users)
    assert og["status"][0] == 0 and og["fallback"][0] == 0
    g = og["n_groups"][0]
    e = 0.0
    for x in og["group_energy"][0][:g]:
        e += x
    assert e == og["energy"][0]
    assert og["group_size"][0][:g].sum() == M
    assert (np.diff(og["group_deadline"][0][:g]) >= 0).all()


def test_fast_dp_all_chunks_vs_oracle(engine):
    """Deadlines U[0.3, 1.5] at M = 300: every row keeps <= 96 useful cells
    but ~70 rows keep more than 64, so large_dp's second DP warp runs both
    of its chunks (cells i+32..i+95) and the 1-/2-chunk stage variants
    alternate; decisions bit-exact against the oracle."""
    M = 300
    prof = profile_heavy(M)
    users = sample_batch(2, M, prof, 0.3, 1.5, seed=1)
    sl = np.zeros(M + 1)
    for n in range(prof.N):
        sl[1:] = sl[1:] + prof.latency[n][:M]
    for k in range(2):
        dl = np.sort(users["deadline"][k])
        rlen = [int(np.sum(dl[0] + sl[1:M - i + 1] <= dl[i])) for i in range(1, M)]
        assert max(rlen) <= 96 and sum(r > 64 for r in rlen) > 30
    ip, og = engine.sweep(prof, users)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, users), where="fast dp ipssa")
    ck.assert_same_og(og, ck.oracle_og(prof, users), where="fast dp og")


@pytest.mark.parametrize("M", [7000, 8000])
def test_large_dp_shared_memory_limit(engine, M):
    """Near the largest sizes: at M = 7000 large_dp's shared memory (dense
    prefix-minimum ring + S0/q1/rlen per user) fits 227 KB, at M = 8000 it
    does not and large_finish runs the change-point DP instead.  Both
    plans are internally consistent (energy = left fold of the group
    energies, groups cover the users in deadline order, every user's
    energy and batch counts add up)."""
    prof = profile_heavy(M)
    users = sample_batch(1, M, prof, 0.25, 1.0, seed=M)
    og = engine.og(prof, users)
    assert og["status"][0] == 0 and og["fallback"][0] == 0
    g = og["n_groups"][0]
    e = 0.0
    for x in og["group_energy"][0][:g]:
        e += x
    assert e == og["energy"][0]
    assert og["group_size"][0][:g].sum() == M
    assert (np.diff(og["group_lo"][0][:g]) > 0).all() and og["group_lo"][0][0] == 0
    assert (np.diff(og["group_deadline"][0][:g]) >= 0).all()
    gu = og["group_of_user"][0]
    assert np.bincount(gu, minlength=g)[:g].tolist() == og["group_size"][0][:g].tolist()
