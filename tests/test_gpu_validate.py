"""validate() on the device (coinfer_validate_batch) vs
the reference's validate (schedule.hpp:139-209): per-constraint violation
counts, worst slack and the exception the reference throws, on solver
schedules (which must validate clean — SPEC acceptance #3, feasibility
fuzz, here at 200k-instance scale) and on corrupted schedules."""
import numpy as np
import pytest

import checkers as ck
from paper_2206_06304_b200 import profile_heavy, profile_light, sample_batch

pytestmark = pytest.mark.gpu


def need_ref():
    if ck.ref() is None:
        pytest.skip("oracle/_ref not built")


def _same(got, exp, where):
    g = {k: ck._to_np(v) for k, v in got.items()}
    np.testing.assert_array_equal(g["status"], exp["status"], err_msg=f"{where} status")
    np.testing.assert_array_equal(g["counts"], exp["counts"], err_msg=f"{where} counts")
    np.testing.assert_array_equal(g["min_slack"], exp["min_slack"], err_msg=f"{where} slack")


def _schedules(engine, prof, u):
    ip = engine.ipssa(prof, u)
    og = engine.og(prof, u)
    out = [("ipssa", engine.ipssa_schedule(prof, u, ip), ip["status"]),
           ("og", engine.og_schedule(prof, u, og), og["status"])]
    for mode in ("PS", "FIFO", "IPSSA_NP", "LC"):
        r, s = engine.baseline(prof, u, mode)
        out.append((mode, s, r["status"]))
    return out


def test_solver_schedules_validate_clean(engine):
    need_ref()
    for prof, u in [(profile_heavy(50), sample_batch(128, 50, profile_heavy(50), 0.25, 1.0, seed=31)),
                    (profile_light(14), sample_batch(128, 14, profile_light(14), 0.05, 0.2, seed=32))]:
        for name, s, st in _schedules(engine, prof, u):
            ok = np.asarray(st) == 0
            got = engine.validate(prof, u, s)
            exp = ck.ref_validate(prof, u, s)
            _same(got, exp, name)
            assert (got["counts"][ok] == 0).all(), name


def test_corrupted_schedules_match_reference(engine):
    need_ref()
    prof = profile_heavy(20)
    u = sample_batch(256, 20, prof, 0.25, 1.0, seed=33)
    rng = np.random.default_rng(7)
    seen = set()
    for name, s, st in _schedules(engine, prof, u):
        s = {k: np.array(ck._to_np(v)) for k, v in s.items()}
        K, M, N = s["x"].shape
        # late / early completions, shifted batches, wrong release times
        s["completion"] += rng.choice([0.0, 0.0, 0.01, -0.01, 1e-10, -1e-8], size=s["completion"].shape)
        s["batch_start"] += rng.choice([0.0, 0.0, 0.0, -0.02, 0.03], size=s["batch_start"].shape)
        # mixed / emptied batches, local placements, bad ids, non-positive freq
        for k in range(0, K, 3):
            m, n = rng.integers(M), rng.integers(N)
            nb = int(s["n_batches"][k])
            s["x"][k, m, n] = rng.integers(0, nb + 1) if rng.random() < 0.9 else nb + 1
        s["freq"][::17] = 0.0
        s["freq"][::29] = -1.0
        got = engine.validate(prof, u, s, tol=1e-9)
        exp = ck.ref_validate(prof, u, s, tol=1e-9)
        _same(got, exp, name)
        assert (exp["counts"].sum(axis=1) > 0).mean() > 0.3  # the corruption bites
        seen |= set(exp["status"].tolist())
    assert {0, 19, 23} <= seen  # clean, bad batch id, f <= 0 all exercised


def test_schedules_from_device_memory_and_tolerance(engine):
    import torch
    need_ref()
    prof = profile_heavy(30)
    u = sample_batch(64, 30, prof, 0.25, 1.0, seed=34)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in u.items()}
    og = engine.og(prof, dev)
    s = engine.og_schedule(prof, dev, og)
    for tol in (1e-9, 0.0):
        got = engine.validate(prof, dev, s, tol=tol)
        torch.cuda.synchronize()
        _same(got, ck.ref_validate(prof, u, {k: v.cpu() for k, v in s.items()}, tol=tol), f"tol {tol}")


def test_acceptance_feasibility_at_scale(engine):
    """SPEC acceptance #3 (every solver schedule validates) on 200k C3
    instances, solved, materialised and validated on the device."""
    import torch
    prof = profile_heavy(50)
    K = 200_000
    u = sample_batch(K, 50, prof, 0.25, 1.0, seed=35)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in u.items()}
    og = engine.og(prof, dev)
    s = engine.og_schedule(prof, dev, og)
    v = engine.validate(prof, dev, s)
    ip = engine.ipssa(prof, dev)
    si = engine.ipssa_schedule(prof, dev, ip)
    vi = engine.validate(prof, dev, si)
    torch.cuda.synchronize()
    for st, val in ((og["status"], v), (ip["status"], vi)):
        ok = st.cpu().numpy() == 0
        assert ok.mean() > 0.99
        assert (val["status"].cpu().numpy() == 0).all()
        assert (val["counts"].cpu().numpy()[ok] == 0).all()
