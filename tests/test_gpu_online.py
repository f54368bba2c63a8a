"""Online slot driver on the GPU vs the reference run_episode (online_sim.hpp).

Episodes must replay the reference slot for slot: per-slot reward, energy,
pending count and edge-busy time, and the episode totals/counts, bit for bit
(same mt19937_64 stream, same clipped sub-scenarios, same OG/IP-SSA plans)."""
import json
import os

import numpy as np
import pytest

import checkers as ck
from paper_2206_06304_b200.engine import OnlineConfig, ProfileArrays

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "online.json")))


def _case(c):
    p = c["profile"]
    prof = ProfileArrays(np.array(p["work"]), np.array(p["data_bits"]), np.array(p["latency"]))
    users = {k: np.array(v, dtype=np.float64) for k, v in c["users"].items()}
    return prof, users, OnlineConfig(**c["cfg"])


@pytest.mark.parametrize("c", GOLD, ids=[c["name"] for c in GOLD])
def test_golden_episode(engine, c):
    prof, users, cfg = _case(c)
    out = engine.online(prof, users, cfg, [c["seed"]], n_trace=1)
    exp = c["expect"]
    assert out["status"][0] == 0
    np.testing.assert_array_equal(out["trace_pending"][0], np.array(exp["trace_pending"]))
    np.testing.assert_array_equal(out["trace_edge_busy"][0], np.array(exp["trace_edge_busy"]))
    np.testing.assert_array_equal(out["trace_energy"][0], np.array(exp["trace_energy"]))
    np.testing.assert_array_equal(out["trace_reward"][0], np.array(exp["trace_reward"]))
    np.testing.assert_array_equal(out["totals"][0], np.array(exp["totals"]))
    np.testing.assert_array_equal(out["counts"][0], np.array(exp["counts"]))


def test_many_episodes_vs_reference(engine):
    """A batch of episodes with different seeds, each vs the reference run."""
    if ck.ref() is None:
        pytest.skip("oracle/_ref not built")
    c = next(c for c in GOLD if c["name"] == "cli_heavy_og_tw0_ep0")
    prof, users, cfg = _case(c)
    cfg.horizon = 3000
    seeds = [int(ck.ref().ref_sub_seed(1, 5, e)) for e in range(48)]
    out = engine.online(prof, users, cfg, seeds)
    for e in range(0, 48, 6):
        r = ck.ref_online(prof, users, cfg, seeds[e], trace=False)
        np.testing.assert_array_equal(out["totals"][e], r["totals"], err_msg=f"episode {e}")
        np.testing.assert_array_equal(out["counts"][e], r["counts"], err_msg=f"episode {e}")


def test_device_memory_and_identity(engine):
    import torch
    c = next(c for c in GOLD if c["name"] == "accounting_og_tw1")
    prof, users, cfg = _case(c)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
    out = engine.online(prof, dev, cfg, [c["seed"]] * 4, n_trace=2)
    engine.synchronize()
    tot = out["totals"].cpu().numpy()
    np.testing.assert_array_equal(tot[0], np.array(c["expect"]["totals"]))
    assert (tot == tot[0]).all()  # same seed, same episode
    # accounting identity (test_online_sim.cpp:231-248)
    assert tot[0, 2] == -(tot[0, 0] + tot[0, 1])


def test_contract_errors(engine):
    c = next(c for c in GOLD if c["name"] == "accounting_og_tw1")
    prof, users, cfg = _case(c)
    bad = {k: v.copy() for k, v in users.items()}
    bad["arrival"][0, 0] = 0.01
    bad["deadline"][0, 0] = 0.5
    out = engine.online(prof, bad, cfg, [1])
    assert out["status"][0] == ck._abi.ST_NOT_RELEASED
    low = OnlineConfig(**{**c["cfg"], "l_low": 0.01})  # below the 0.02 floor
    assert engine.online(prof, users, low, [1])["status"][0] == ck._abi.ST_FLOOR_ABOVE_LLOW
    with pytest.raises(ValueError):
        engine.online(prof, users, OnlineConfig(**{**c["cfg"], "slot": 0.0}), [1])
    with pytest.raises(ValueError):
        engine.online(prof, users, OnlineConfig(**{**c["cfg"], "p_arrive": 1.5}), [1])


# Configurations for the warp-parallel slot loop (users on lanes, the random
# stream split by prefix sums) against the lane-0 slot loop it replaces for
# M <= 32, which the golden episodes pin to the reference.
_SWEEP = [
    ("heavy", 14, dict(arrival="bernoulli", p_arrive=0.05, l_low=0.25, l_high=1.0, solver="og", policy="tw", window=0)),
    ("light", 14, dict(arrival="bernoulli", p_arrive=0.25, l_low=0.05, l_high=0.2, solver="og", policy="tw", window=0)),
    ("heavy", 32, dict(arrival="bernoulli", p_arrive=0.3, l_low=0.25, l_high=1.0, solver="og", policy="tw", window=2)),
    ("heavy", 1, dict(arrival="bernoulli", p_arrive=0.5, l_low=0.25, l_high=1.0, solver="og", policy="tw", window=0)),
    ("heavy", 9, dict(arrival="immediate", p_arrive=0.0, l_low=0.25, l_high=1.0, solver="ipssa", policy="tw", window=1)),
    ("heavy", 12, dict(arrival="bernoulli", p_arrive=1.0, l_low=0.4, l_high=0.4, solver="og", policy="tw", window=3)),
    ("light", 20, dict(arrival="bernoulli", p_arrive=0.6, l_low=0.05, l_high=0.2, solver="ipssa", policy="local", window=0)),
    ("heavy", 7, dict(arrival="bernoulli", p_arrive=0.0, l_low=0.25, l_high=1.0, solver="og", policy="tw", window=0)),
]


def _sweep_runs(engine, horizon, episodes):
    from paper_2206_06304_b200 import profile_heavy, profile_light, sample_batch
    res = []
    for kind, M, kw in _SWEEP:
        prof = profile_heavy(M) if kind == "heavy" else profile_light(M)
        hi = kw["l_high"]
        users = sample_batch(1, M, prof, hi, hi, seed=M)
        cfg = OnlineConfig(slot=0.025, horizon=horizon, **kw)
        out = engine.online(prof, users, cfg, list(range(1, episodes + 1)), n_trace=2)
        res.append({k: np.asarray(v) for k, v in out.items()})
    return res


def test_warp_slot_loop_matches_serial_loop(engine, tmp_path):
    import subprocess
    import sys
    code = r'''
import os, sys, pickle
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import test_gpu_online as t
from paper_2206_06304_b200 import Engine
pickle.dump(t._sweep_runs(Engine(0), 4000, 24), open(sys.argv[1], "wb"))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = str(tmp_path / "serial.pkl")
    r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, COINFER_ONLINE_SERIAL="1"), timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    import pickle
    serial = pickle.load(open(path, "rb"))
    warp = _sweep_runs(engine, 4000, 24)
    for (kind, M, kw), a, b in zip(_SWEEP, warp, serial):
        for k in a:
            np.testing.assert_array_equal(a[k], b[k], err_msg=f"{kind} M={M} {kw} {k}")
        assert (a["status"] == 0).all(), (kind, M, kw)


C5 = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "online_c5.json")))


@pytest.mark.parametrize("c", C5, ids=[c["name"] for c in C5])
def test_c5_full_horizon_episode(engine, c):
    """BASELINE config 5 at its full 10^5-slot horizon (heavy and light),
    slot for slot against the reference run_episode (tests/golden/
    make_online_c5.py): every 1,000-slot block of the trace must hash equal,
    and the episode totals and counts must be equal."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_online_c5 import block_digests
    prof, users, cfg = _case(c)
    out = engine.online(prof, users, cfg, [c["seed"]], n_trace=1)
    assert out["status"][0] == 0
    got = block_digests({k: out[k][0] for k in ("trace_reward", "trace_energy", "trace_pending",
                                                 "trace_edge_busy")})
    bad = [i for i, (x, y) in enumerate(zip(got, c["digests"])) if x != y]
    assert not bad, f"first differing block: slots {bad[0] * c['block']}..{(bad[0] + 1) * c['block'] - 1}"
    np.testing.assert_array_equal(out["totals"][0], np.array(c["totals"]))
    np.testing.assert_array_equal(out["counts"][0], np.array(c["counts"]))


def test_c5_batch_matches_single_episodes(engine):
    """Episodes batched together (one warp each) equal the same episodes run
    alone: the golden C5 seeds inside a batch of 64."""
    c = C5[0]
    prof, users, cfg = _case(c)
    seeds = [c["seed"]] + [c["seed"] + 1 + e for e in range(63)]
    out = engine.online(prof, users, cfg, seeds)
    np.testing.assert_array_equal(out["totals"][0], np.array(c["totals"]))
    np.testing.assert_array_equal(out["counts"][0], np.array(c["counts"]))
