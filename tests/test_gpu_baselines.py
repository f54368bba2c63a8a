"""Device schedule materialisation and the offline baselines (SURVEY.md §8f
rows 1-2) vs the reference, bit for bit.

  * coinfer_ipssa_schedule / coinfer_og_schedule: the Schedule ip_ssa / og
    return (x, batch_start, completion, freq), built and normalised on the
    GPU, vs the reference's (offline_solvers.hpp:155-185,357-386,
    schedule.hpp:93-113).
  * coinfer_baseline_batch: baseline(sc, LC | PS | FIFO | IPSSA_NP)
    (offline_solvers.hpp:390-612), SolveResult and Schedule.
  * coinfer_best_partition: best_partition / local_only_choice (:62-117).
Instances: the reference tests' own generators (testutil::random_scenario
with the suites' seeds), CLI-style sample_scenario batches, the golden
fixtures, and edge cases (f_min > 0, arrivals, ties, infeasible users)."""
import numpy as np
import pytest

import checkers as ck
import golden_io
from paper_2206_06304_b200 import profile_heavy, profile_light, sample_batch

pytestmark = pytest.mark.gpu

MODES = ["LC", "PS", "FIFO", "IPSSA_NP"]


def need_ref():
    if ck.ref() is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")


def random_cases(seed, n, users_of, subtasks_of, growth, equal):
    r = ck.ref()
    h = r.ref_rng_new(r.ref_mix_seed(seed, 0))
    try:
        return [ck.ref_random_scenario(h, users_of(i), subtasks_of(i), growth, equal(i))
                for i in range(n)]
    finally:
        r.ref_rng_free(h)


def _check_baseline(engine, prof, users, mode, where):
    got, gs = engine.baseline(prof, users, mode)
    exp, es = ck.ref_baseline(prof, users, mode)
    ck.assert_same_ip(got, exp, where=f"{where} {mode}")
    ck.assert_same_schedule(gs, es, exp["status"], where=f"{where} {mode}")
    return exp["status"]


@pytest.mark.parametrize("mode", MODES)
def test_baselines_reference_suite_streams(engine, mode):
    """The instance streams of test_offline_solvers.cpp's baseline tests."""
    need_ref()
    cases = (random_cases(81, 20, lambda i: 1 + i % 6, lambda i: 2 + i % 3, 0.5, lambda i: i % 2 == 0)
             + random_cases(82, 20, lambda i: 1 + i % 6, lambda i: 2 + i % 3, 0.5, lambda i: i % 2 == 0)
             + random_cases(83, 20, lambda i: 1 + i % 6, lambda i: 2 + i % 3, 0.5, lambda i: True)
             + random_cases(77, 25, lambda i: 1 + i % 5, lambda i: 2 + i % 3, 0.4, lambda i: True))
    for i, (prof, u) in enumerate(cases):
        _check_baseline(engine, prof, u, mode, f"case {i}")


@pytest.mark.parametrize("mode", MODES)
def test_baselines_two_stage_kats(engine, mode):
    need_ref()
    for users in (1, 2, 3):
        prof, u = ck.two_stage(users)
        _check_baseline(engine, prof, u, mode, f"two_stage({users})")
    prof, u = ck.two_stage(2)
    u["rate_up"][0, 1] = 2e6  # FIFO: the faster user reserves first
    _check_baseline(engine, prof, u, mode, "two_stage rates")
    prof, u = ck.two_stage(2)
    prof.data_bits[0] = 2e4  # IPSSA_NP offloads the whole task
    _check_baseline(engine, prof, u, mode, "two_stage light input")
    prof, u = ck.two_stage(1)
    u["deadline"][:] = 0.015  # below the local floor: every baseline throws
    st = _check_baseline(engine, prof, u, mode, "unreachable")
    assert st[0] == 1


@pytest.mark.parametrize("mode", MODES)
def test_baselines_cli_batches(engine, mode):
    """C3-shaped batches (heavy and light profiles), many instances per launch."""
    need_ref()
    for prof, u in [(profile_heavy(50), sample_batch(256, 50, profile_heavy(50), 0.25, 1.0, seed=11)),
                    (profile_light(14), sample_batch(256, 14, profile_light(14), 0.05, 0.2, seed=12))]:
        st = _check_baseline(engine, prof, u, mode, "cli")
        assert (st == 0).mean() > 0.5


@pytest.mark.parametrize("mode", MODES)
def test_baselines_edge_cases(engine, mode):
    need_ref()
    prof = profile_heavy(12)
    u = sample_batch(64, 12, prof, 0.25, 1.0, seed=3)
    rng = np.random.default_rng(5)
    u["f_min"] = rng.uniform(0.0, 0.5, u["f_min"].shape) * u["f_max"]
    u["arrival"] = rng.uniform(0.0, 0.05, u["arrival"].shape)
    u["deadline"] = u["deadline"] + u["arrival"]
    u["kappa"][::7] = 0.0
    u["power_up"][::5] = 0.0
    u["deadline"][::9, 0] = 0.03  # unreachable user -> domain_error
    _check_baseline(engine, prof, u, mode, "edge")
    bad = {k: v.copy() for k, v in u.items()}
    bad["kappa"][1, 2] = -1.0
    bad["rate_up"][2, 0] = 0.0
    got, _ = engine.baseline(prof, bad, mode)
    assert got["status"][1] == 11 and got["status"][2] == 12


def test_ipssa_and_og_schedules_match_reference(engine):
    need_ref()
    cases = [(c["profile"], c["users"], c["deadline"], c["kind"]) for c in golden_io.all_cases()
             if c["kind"] in ("ipssa", "og")]
    prof = profile_heavy(50)
    u = sample_batch(128, 50, prof, 0.25, 1.0, seed=21)
    cases += [(prof, u, None, "ipssa"), (prof, u, None, "og")]
    cases += [(p, uu, None, k) for p, uu in random_cases(80, 10, lambda i: 2 + i % 5,
                                                         lambda i: 2 + i % 3, 0.4, lambda i: False)
              for k in ("ipssa", "og")]
    for i, (p, uu, dl, kind) in enumerate(cases):
        if kind == "ipssa":
            solved = engine.ipssa(p, uu, dl)
            got = engine.ipssa_schedule(p, uu, solved, dl)
        else:
            solved = engine.og(p, uu)
            got = engine.og_schedule(p, uu, solved)
        exp = ck.ref_schedule(p, uu, kind, dl)
        np.testing.assert_array_equal(solved["status"], exp["status"])
        ck.assert_same_schedule(got, exp, exp["status"], where=f"case {i} {kind}")


def test_schedules_from_device_memory(engine):
    import torch
    need_ref()
    prof = profile_heavy(30)
    u = sample_batch(64, 30, prof, 0.25, 1.0, seed=8)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in u.items()}
    og = engine.og(prof, dev)
    sched = engine.og_schedule(prof, dev, og)
    ip = engine.ipssa(prof, dev)
    isched = engine.ipssa_schedule(prof, dev, ip)
    base, bs = engine.baseline(prof, dev, "PS")
    torch.cuda.synchronize()
    ck.assert_same_schedule(sched, ck.ref_schedule(prof, u, "og"), og["status"].cpu(), "og dev")
    ck.assert_same_schedule(isched, ck.ref_schedule(prof, u, "ipssa"), ip["status"].cpu(), "ip dev")
    exp, es = ck.ref_baseline(prof, u, "PS")
    ck.assert_same_ip(base, exp, where="PS dev")
    ck.assert_same_schedule(bs, es, exp["status"], "PS dev")


def test_best_partition_queries(engine):
    """best_partition / local_only_choice, incl. the reference tests' KATs
    (test_offline_solvers.cpp:56-110): f = 1/7 split 1, tie -> larger split,
    f_min floor, nothing fits."""
    prof, u = ck.two_stage(1)
    q = {k: v.reshape(1, 1) for k, v in u.items()}
    s = np.array([[0.08, 0.09]])
    r = engine.best_partition(prof, q, s)
    assert r["split"][0] == 1 and r["feasible"][0] == 1
    # EXPECT_DOUBLE_EQ in the reference test: within 4 ULPs (the budget
    # 0.09 - 0.02 - 0 is not exactly 0.07)
    assert abs(r["freq"][0] - 0.01 / 0.07) <= 4 * np.spacing(0.01 / 0.07)
    assert abs(r["energy"][0] - (3.0 / 49.0 + 0.02)) < 1e-12
    q0 = dict(q, kappa=np.zeros((1, 1)), power_up=np.zeros((1, 1)))
    r = engine.best_partition(prof, q0, s)
    assert r["split"][0] == 2 and r["energy"][0] == 0.0
    assert abs(r["freq"][0] - 0.2) <= 4 * np.spacing(0.2)  # EXPECT_DOUBLE_EQ
    r = engine.best_partition(prof, dict(q, f_min=np.full((1, 1), 0.5)), s)
    assert r["freq"][0] >= 0.5
    r = engine.best_partition(prof, dict(q, deadline=np.full((1, 1), -1.0)), np.array([[-1.0, -1.0]]))
    assert r["feasible"][0] == 0 and np.isinf(r["energy"][0]) and np.isnan(r["freq"][0])
    r = engine.best_partition(prof, q, None)  # local_only_choice at the user's deadline
    assert r["split"][0] == 2 and r["feasible"][0] == 1
    assert abs(r["freq"][0] - 0.2) <= 4 * np.spacing(0.2)
    # split 0: nothing local, freq NaN
    r = engine.best_partition(prof, dict(q, rate_up=np.full((1, 1), 1e9)), np.array([[0.08, 0.09]]))
    assert r["split"][0] in (0, 1, 2)
