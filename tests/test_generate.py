"""Scenario generation on the device (coinfer_sample_batch, SURVEY.md §8f
row 3) vs the reference generator (sample_scenario, scenario_gen.hpp:113-173,
through oracle/_ref): the mt19937_64 stream, positions-driven retries,
deadlines, f_max and kappa bit for bit; rates through CUDA's libm within a
few ulp of glibc's.  The CLI's seeding helper is checked on CPU."""
import numpy as np
import pytest

import checkers as ck
from paper_2206_06304_b200 import _abi, profile_heavy, profile_light, sub_seed


def test_sub_seed_matches_reference_and_library():
    r = ck.ref()
    lib = _abi.load_library()
    idx = np.array([0, 1, 2, 999_999, 123456789], dtype=np.uint64)
    ours = sub_seed(1, 1, idx)
    for i, k in enumerate(idx):
        assert int(ours[i]) == lib.coinfer_sub_seed(1, 1, int(k))
        if r is not None:
            assert int(ours[i]) == r.ref_sub_seed(1, 1, int(k))
    assert int(sub_seed(7, 5, [3])[0]) == lib.coinfer_sub_seed(7, 5, 3)


def _ref_batch(M, lo, hi, seeds, heavy):
    return ck.ref_sample_scenarios(len(seeds), M, lo, hi, seeds, heavy=heavy)[1]


@pytest.mark.gpu
@pytest.mark.parametrize("heavy,M,lo,hi", [(True, 50, 0.25, 1.0), (True, 10, 0.25, 0.25),
                                          (False, 14, 0.05, 0.2), (True, 100, 0.25, 1.0)])
def test_device_generator_matches_reference(engine, heavy, M, lo, hi):
    if ck.ref() is None:
        pytest.skip("oracle/_ref not built")
    prof = profile_heavy(M) if heavy else profile_light(M)
    seeds = sub_seed(1, 1, np.arange(300))
    got, st = engine.sample(prof, M, seeds, lo, hi)
    exp = _ref_batch(M, lo, hi, seeds, heavy)
    assert (st == 0).all()
    for f in ("f_min", "f_max", "kappa", "power_up", "arrival", "deadline", "power_down"):
        np.testing.assert_array_equal(got[f], exp[f], err_msg=f)
    rel = np.abs(got["rate_up"] - exp["rate_up"]) / exp["rate_up"]
    assert rel.max() < 1e-13, rel.max()
    np.testing.assert_array_equal(got["rate_down"], got["rate_up"])


@pytest.mark.gpu
def test_device_generator_device_memory_and_shards(engine):
    import torch
    prof = profile_heavy(50)
    seeds = sub_seed(1, 1, np.arange(5000))
    dev, st = engine.sample(prof, 50, seeds, 0.25, 1.0, device=True)
    host, _ = engine.sample(prof, 50, seeds, 0.25, 1.0)
    torch.cuda.synchronize()
    for f in _abi.USER_FIELDS:
        np.testing.assert_array_equal(dev[f].cpu().numpy(), host[f])
    part, _ = engine.sample(prof, 50, seeds[2500:], 0.25, 1.0)  # shard invariance
    np.testing.assert_array_equal(part["deadline"], host["deadline"][2500:])
    # and the generated instances solve
    ip, og = engine.sweep(prof, dev)
    torch.cuda.synchronize()
    assert (og["status"].cpu().numpy() == 0).all()


@pytest.mark.gpu
def test_generator_config_errors(engine):
    prof = profile_heavy(10)
    with pytest.raises(ValueError, match="deadline below the all-local floor"):
        engine.sample(prof, 10, [1, 2], 0.01, 0.01)
    with pytest.raises(ValueError, match="latency table shorter"):
        engine.sample(profile_heavy(5), 10, [1], 0.5, 0.5)
    with pytest.raises(ValueError, match="physical quantities"):
        engine.sample(prof, 10, [1], 0.5, 0.5, bandwidth=-1.0)
