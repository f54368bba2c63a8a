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
