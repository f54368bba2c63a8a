"""The reference's brute-force oracles on the device (oracles.hpp, SURVEY.md
§8f row 4) vs the reference's own oracles, then the Theorem 1/2 checks of
tests/test_oracles.cpp run at far larger sample counts:
  * oracle_structured == fixed_batch_schedule (rel 1e-9) — Alg. 1 is exact;
  * oracle_grouping_contiguous == og, bit for bit — the DP is exact;
  * oracle_grouping == og (rel 1e-9) for constant batch latency — contiguous
    groupings lose nothing."""
import numpy as np
import pytest

import checkers as ck
from paper_2206_06304_b200 import profile_heavy, profile_light, sample_batch

pytestmark = pytest.mark.gpu


def need_ref():
    if ck.ref() is None:
        pytest.skip("oracle/_ref not built")


def rel_gap(a, b):
    return np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-30)


def test_structured_reference_stream(engine):
    """OracleStructured.MatchesFixedBatchOnRandomInstances (test_oracles.cpp:41-60)."""
    need_ref()
    r = ck.ref()
    h = r.ref_rng_new(r.ref_mix_seed(101, 0))
    try:
        for i in range(60):
            M = int(r.ref_uniform_int(h, 1, 4))
            N = int(r.ref_uniform_int(h, 2, 4))
            prof, u = ck.ref_random_scenario(h, M, N, 0.5, True)
            b = int(r.ref_uniform_int(h, 1, M))
            dl = u["deadline"][:, 0].copy()
            got = engine.oracle_structured(prof, u, dl, [b])
            exp = ck.ref_oracle_structured(prof, u, dl, [b])
            assert got["status"][0] == 0
            for k in ("energy", "split", "fallback", "feasible"):
                np.testing.assert_array_equal(got[k], exp[k], err_msg=f"instance {i} {k}")
            fx = engine.fixed(prof, u, np.array([b], np.int32), dl)
            assert got["fallback"][0] == (1 - fx["pipeline_feasible"][0])
            assert rel_gap(fx["energy"][0], got["energy"][0]) < 1e-9
    finally:
        r.ref_rng_free(h)


def test_grouping_reference_streams(engine):
    """ContiguousBruteForceMatchesDp / ContiguousIsOptimalForConstantLatency."""
    need_ref()
    r = ck.ref()
    for seed, growth, n, contiguous in [(103, 0.5, 20, True), (104, 0.0, 12, False)]:
        h = r.ref_rng_new(r.ref_mix_seed(seed, 0))
        try:
            for i in range(n):
                M = int(r.ref_uniform_int(h, 2, 6))
                prof, u = ck.ref_random_scenario(h, M, 2 + i % 3, growth, False)
                got = engine.oracle_grouping(prof, u, contiguous)
                exp = ck.ref_oracle_groups(prof, u, contiguous)
                assert got["status"][0] == 0
                np.testing.assert_array_equal(got["energy"], exp["energy"], err_msg=f"{seed} {i}")
                np.testing.assert_array_equal(got["n_groups"], exp["n_groups"])
                if got["feasible"][0]:
                    np.testing.assert_array_equal(got["group_of_user"], exp["group_of_user"])
                og = engine.og(prof, u)
                if not got["feasible"][0]:
                    assert og["fallback"][0] == 1
                    continue
                assert og["fallback"][0] == 0
                if contiguous:
                    assert og["energy"][0] == got["energy"][0]
                    assert og["n_groups"][0] == got["n_groups"][0]
                else:
                    assert rel_gap(og["energy"][0], got["energy"][0]) < 1e-9
        finally:
            r.ref_rng_free(h)


def test_theorems_at_scale(engine):
    """The same checks on thousands of sample_scenario instances per launch."""
    # Alg. 1 vs exhaustive splits: M = 7 users (5^7 vectors each), random bounds
    prof = profile_heavy(7)
    u = sample_batch(2000, 7, prof, 0.25, 1.0, seed=41)
    dl = u["deadline"].min(axis=1)
    b = np.random.default_rng(1).integers(1, 8, 2000).astype(np.int32)
    o = engine.oracle_structured(prof, u, dl, b)
    fx = engine.fixed(prof, u, b, dl)
    ok = fx["status"] == 0
    assert (o["status"] == 0).all() and ok.mean() > 0.9
    assert (o["feasible"][ok] == 1).all()
    assert (rel_gap(fx["energy"][ok], o["energy"][ok]) < 1e-9).all()
    assert (o["fallback"][ok] == 1 - fx["pipeline_feasible"][ok]).all()
    # the grouping DP vs every cut pattern: M = 14 (8192 patterns each)
    prof = profile_heavy(14)
    u = sample_batch(4000, 14, prof, 0.25, 1.0, seed=42)
    o = engine.oracle_grouping(prof, u, True)
    og = engine.og(prof, u)
    assert (o["status"] == 0).all()
    feas = o["feasible"] == 1
    np.testing.assert_array_equal(og["fallback"], (~feas).astype(np.uint8))
    np.testing.assert_array_equal(og["energy"][feas], o["energy"][feas])
    # equal-energy groupings can differ between the DP's tie rule (smallest
    # prev) and the enumeration's (first cut pattern); there the reference's
    # own og must agree with ours
    diff = np.nonzero(feas & (og["n_groups"] != o["n_groups"]))[0]
    assert len(diff) <= 0.01 * len(feas)
    if len(diff) and ck.ref() is not None:
        sub = {k: v[diff] for k, v in u.items()}
        ck.assert_same_og(engine.og(prof, sub), ck.ref_og(prof, sub), where="tie instances")
    # contiguous groupings are optimal among all set partitions (flat latency)
    prof = profile_light(8)
    u = sample_batch(1000, 8, prof, 0.05, 0.2, seed=43)
    o = engine.oracle_grouping(prof, u, False)
    og = engine.og(prof, u)
    feas = o["feasible"] == 1
    assert feas.mean() > 0.5
    assert (rel_gap(og["energy"][feas], o["energy"][feas]) < 1e-9).all()


def test_enumeration_guards(engine):
    prof, u = ck.two_stage(10, 12)
    o = engine.oracle_grouping(prof, u, False)
    assert o["status"][0] == 25
    prof, u = ck.two_stage(17, 18)
    o = engine.oracle_grouping(prof, u, True)
    assert o["status"][0] == 25
    prof, u = ck.two_stage(14, 16)  # 3^14 > 2e6
    o = engine.oracle_structured(prof, u, [0.1], [4])
    assert o["status"][0] == 25
