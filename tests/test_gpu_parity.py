"""Parity of the CUDA engine (libcoinfer_b200.so, sm_100a) with the reference.

Decisions (splits, batch bounds, batch sizes, groupings, fallback flags,
statuses) must be bit-exact; energies and frequencies are compared bit-exact
too (the kernels reproduce the reference's operation order with no FMA
contraction), which is stricter than the north star's 1e-9 relative.
"""
import numpy as np
import pytest

import checkers as ck
import golden_io
from paper_2206_06304_b200 import profile_heavy, profile_light, sample_batch
from paper_2206_06304_b200.engine import ProfileArrays

pytestmark = pytest.mark.gpu

CASES = golden_io.all_cases()


def run_engine(engine, c, device=False):
    users = c["users"]
    dl, b = c["deadline"], c["b"]
    if device:
        import torch
        users = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
        dl = None if dl is None else torch.as_tensor(dl, device="cuda")
        b = None if b is None else torch.as_tensor(b, device="cuda")
    if c["kind"] == "ipssa":
        out = engine.ipssa(c["profile"], users, dl)
    elif c["kind"] == "fixed":
        out = engine.fixed(c["profile"], users, b, dl)
    else:
        out = engine.og(c["profile"], users)
    if device:
        engine.synchronize()
    return out


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_golden_fixture(engine, c):
    out = run_engine(engine, c)
    if c["kind"] == "og":
        ck.assert_same_og(out, c["expect"], where=c["name"])
    else:
        ck.assert_same_ip(out, c["expect"], where=c["name"])


@pytest.mark.parametrize("c", [c for c in CASES if c["name"].startswith(("C3", "C2", "two_stage2", "contract"))],
                         ids=lambda c: c["name"])
def test_golden_fixture_device_memory(engine, c):
    out = run_engine(engine, c, device=True)
    if c["kind"] == "og":
        ck.assert_same_og(out, c["expect"], where=c["name"])
    else:
        ck.assert_same_ip(out, c["expect"], where=c["name"])


def random_profile(rng, N, b_max, growth_max=0.5):
    base = rng.uniform(0.002, 0.02, N)
    growth = rng.uniform(0.0, growth_max, N)
    lat = base[:, None] * (1.0 + growth[:, None] * np.arange(b_max, dtype=np.float64)[None, :])
    bits = rng.uniform(1e4, 2e6, N + 1)
    bits[-1] = 0.0
    return ProfileArrays(base.copy(), bits, np.ascontiguousarray(lat))


def random_users(rng, K, M, prof, margin=(1.05, 3.0), fmin=False, arrival=False, equal=False):
    """testutil::random_scenario-style users (helpers.hpp:42-101), numpy RNG."""
    alpha = rng.uniform(1.0, 4.0, (K, M))
    rho = rng.uniform(1.0, 150.0, (K, M))
    f_max = 1.0 / alpha
    kappa = rho * 300.0 * alpha * alpha
    rate = rng.uniform(1e6, 2e7, (K, M))
    floor = prof.work.sum() / f_max
    arr = rng.uniform(0.0, 0.01, (K, M)) if arrival else np.zeros((K, M))
    dl = arr + floor * rng.uniform(*margin, (K, M))
    if equal:
        dl[:] = dl.max(axis=1, keepdims=True)
    f_min = f_max * rng.uniform(0.0, 0.5, (K, M)) if fmin else np.zeros((K, M))
    one = np.ones((K, M))
    return dict(f_min=f_min, f_max=f_max, kappa=kappa, rate_up=rate, power_up=one,
                arrival=arr, deadline=dl, rate_down=rate.copy(), power_down=one.copy())


def check_sweep(engine, prof, users):
    ip, og = engine.sweep(prof, users)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, users), where="ipssa")
    ck.assert_same_og(og, ck.oracle_og(prof, users), where="og")
    return ip, og


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 7, 8, 13, 16, 31, 32, 33, 40, 64, 65, 100])
def test_random_vs_oracle_sizes(engine, M):
    rng = np.random.default_rng(1000 + M)
    for N in (1, 2, 4, 7):
        prof = random_profile(rng, N, M + 2)
        users = random_users(rng, 24 if M <= 40 else 6, M, prof)
        check_sweep(engine, prof, users)


@pytest.mark.parametrize("M,lo,hi", [(150, 0.5, 3.0), (176, 0.5, 3.0), (176, 20.0, 40.0), (176, 0.25, 1.0), (255, 0.5, 3.0)])
def test_small_path_largest_sizes(engine, M, lo, hi):
    """The shared-memory path at its largest instances (M = 176, the largest
    whose triangle fits in shared memory; 255 takes the large path): byte
    row and chunk tables, useful lengths from a few cells up to whole rows
    (loose deadlines: every group fits after every other)."""
    prof = profile_heavy(M)
    users = sample_batch(2, M, prof, lo, hi, seed=M)
    check_sweep(engine, prof, users)


@pytest.mark.parametrize("variant", ["fmin", "arrival", "equal", "tight", "loose", "flat", "N16"])
def test_random_vs_oracle_variants(engine, variant):
    rng = np.random.default_rng(hash(variant) % 2**32)
    M, K, N = 20, 40, 4
    kw = {}
    growth = 0.5
    if variant == "fmin":
        kw["fmin"] = True
    if variant == "arrival":
        kw["arrival"] = True
    if variant == "equal":
        kw["equal"] = True
    if variant == "tight":
        kw["margin"] = (1.0, 1.2)
    if variant == "loose":
        kw["margin"] = (5.0, 40.0)
    if variant == "flat":
        growth = 0.0
    if variant == "N16":
        N = 16
    prof = random_profile(rng, N, M + 2, growth)
    check_sweep(engine, prof, random_users(rng, K, M, prof, **kw))


def test_ties_kappa_power_zero(engine):
    """kappa = 0 and p_u = 0 make every split cost 0: pure tie-breaking."""
    rng = np.random.default_rng(7)
    prof = random_profile(rng, 3, 12)
    users = random_users(rng, 30, 10, prof)
    users["kappa"][:, ::2] = 0.0
    users["power_up"][:, 1::3] = 0.0
    check_sweep(engine, prof, users)


def test_heavy_profile_C3_sample(engine):
    """BASELINE config 3 shape (M=50, heavy, deadlines U[0.25,1]) vs the oracle."""
    prof = profile_heavy(50)
    users = sample_batch(2048, 50, prof, 0.25, 1.0, seed=11)
    check_sweep(engine, prof, users)


@pytest.mark.parametrize("M,K,light", [(40, 2048, False), (64, 2048, False), (72, 2048, True), (100, 2048, False)])
def test_pipelined_kernel_shapes(engine, M, K, light):
    """Batches of >= 2048 instances run the pipelined kernel (solve_pipe_kernel)
    in each of its team shapes: four CTAs per SM (M = 40), two (64, 72), one
    (100).  Every instance against the oracle for M <= 72; at M = 100 the
    first 256 and the last 64 (the oracle's O(M^3 N) cost)."""
    prof = profile_light(M) if light else profile_heavy(M)
    users = sample_batch(K, M, prof, 0.05 if light else 0.25, 0.2 if light else 1.0, seed=M + 3)
    ip, og = engine.sweep(prof, users)
    parts = [(0, K)] if M <= 72 else [(0, 256), (K - 64, K)]
    for k0, k1 in parts:
        sub = ck.slice_users(users, k0, k1)
        ck.assert_same_ip({k: v[k0:k1] for k, v in ip.items()}, ck.oracle_ipssa(prof, sub), where=f"M={M} [{k0},{k1})")
        ck.assert_same_og({k: v[k0:k1] for k, v in og.items()}, ck.oracle_og(prof, sub), where=f"M={M} [{k0},{k1})")


def test_pipelined_kernel_single_solver(engine):
    """IP-SSA alone and OG alone through the pipelined kernel (>= 2048
    instances): the G phase runs only that solver's chains."""
    prof = profile_heavy(50)
    users = sample_batch(2048, 50, prof, 0.25, 1.0, seed=77)
    ck.assert_same_ip(engine.ipssa(prof, users), ck.oracle_ipssa(prof, users), where="ipssa only")
    ck.assert_same_og(engine.og(prof, users), ck.oracle_og(prof, users), where="og only")


def test_pipelined_kernel_invalid_and_infeasible_instances(engine):
    """Instances that fail Scenario::check, or have no feasible plan, inside a
    pipelined batch: their statuses, and every other instance's solution."""
    prof = profile_heavy(50)
    users = sample_batch(2048, 50, prof, 0.25, 1.0, seed=91)
    users = {k: v.copy() for k, v in users.items()}
    users["kappa"][3, 7] = -1.0          # COINFER_ST_NEG_KAPPA
    users["rate_up"][100, 0] = 0.0       # bad rate
    users["deadline"][777, 5] = users["arrival"][777, 5]  # deadline not after arrival
    users["deadline"][1500, :] = 1e-9    # nobody can finish: infeasible
    users["f_max"][2047, 3] = -2.0       # bad frequency
    ip, og = engine.sweep(prof, users)
    ck.assert_same_ip(ip, ck.oracle_ipssa(prof, users), where="pipelined, invalid rows")
    ck.assert_same_og(og, ck.oracle_og(prof, users), where="pipelined, invalid rows")
    assert (np.asarray(og["status"])[[3, 100, 777, 2047]] != 0).all()


def test_light_profile_online_shape(engine):
    prof = profile_light(14)
    users = sample_batch(512, 14, prof, 0.05, 0.2, seed=12)
    check_sweep(engine, prof, users)


def test_fixed_batch_vs_oracle(engine):
    rng = np.random.default_rng(5)
    for M in (1, 6, 30):
        prof = random_profile(rng, 3, M + 2)
        users = random_users(rng, 50, M, prof)
        b = rng.integers(1, M + 1, 50).astype(np.int32)
        dl = users["deadline"].min(axis=1) * rng.uniform(0.5, 1.2, 50)
        out = engine.fixed(prof, users, b, dl)
        ck.assert_same_ip(out, ck.oracle_fixed(prof, users, b, dl))


def test_device_and_host_paths_agree(engine):
    import torch
    prof = profile_heavy(50)
    users = sample_batch(1000, 50, prof, seed=3)
    ip_h, og_h = engine.sweep(prof, users)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
    ip_d, og_d = engine.sweep(prof, dev)
    engine.synchronize()
    ck.assert_same_ip(ip_h, ip_d)
    ck.assert_same_og(og_h, og_d)


def test_host_pipeline_chunks_agree_with_device(engine):
    """Host batches of >= 65536 instances go through the chunked two-stream
    pipeline (up to 64 chunks of >= 16384); their results must equal one
    device launch."""
    import torch
    prof = profile_heavy(12)
    users = sample_batch(140_000, 12, prof, 0.25, 1.0, seed=13)
    ip_h, og_h = engine.sweep(prof, users)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
    ip_d, og_d = engine.sweep(prof, dev)
    engine.synchronize()
    ck.assert_same_ip(ip_h, ip_d)
    ck.assert_same_og(og_h, og_d)


def test_full_size_properties(engine):
    """At large batch sizes: shard invariance, internal consistency, and a
    sampled oracle check (size-independent properties)."""
    import torch
    K, M = 200_000, 50
    prof = profile_heavy(M)
    users = sample_batch(K, M, prof, seed=21)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
    ip, og = engine.sweep(prof, dev)
    engine.synchronize()
    ip = {k: v.cpu().numpy() for k, v in ip.items()}
    og = {k: v.cpu().numpy() for k, v in og.items()}
    assert (ip["status"] == 0).all() and (og["status"] == 0).all()
    # shard invariance: re-solving a slice gives the same bits
    sl = ck.slice_users(users, 12345, 12345 + 777)
    ip2, og2 = engine.sweep(prof, sl)
    ck.assert_same_ip({k: v[12345:12345 + 777] for k, v in ip.items()}, ip2)
    ck.assert_same_og({k: v[12345:12345 + 777] for k, v in og.items()}, og2)
    # OG never loses to the single-group solve beyond fold-order rounding
    assert (og["energy"] <= ip["energy"] * (1 + 1e-12)).all()
    # plan energy = left fold of group energies, batch sizes within bounds
    for k in range(0, K, 9973):
        g = og["n_groups"][k]
        e = 0.0
        for x in og["group_energy"][k][:g]:
            e += x
        assert e == og["energy"][k]
        bs = og["group_batch_size"][k][:g]
        assert (np.diff(bs, axis=1) >= 0).all()
        assert (bs[:, -1] <= og["group_b"][k][:g]).all()
        assert og["group_size"][k][:g].sum() == M
    # sampled oracle check
    idx = np.arange(0, K, K // 300)
    sub = {n: v[idx] for n, v in users.items()}
    ck.assert_same_ip({k: v[idx] for k, v in ip.items()}, ck.oracle_ipssa(prof, sub))
    ck.assert_same_og({k: v[idx] for k, v in og.items()}, ck.oracle_og(prof, sub))


def test_cuda_library_really_loaded(engine):
    before = engine.launches
    prof, users = ck.two_stage(2)
    engine.ipssa(prof, users)
    assert engine.launches == before + 1
    maps = open("/proc/self/maps").read()
    assert "libcoinfer_b200.so" in maps


@pytest.mark.gpu
def test_count_work_counts_the_same_solve(engine):
    """coinfer_count_work (bench.py's roofline credit) runs the instrumented
    solve: deterministic counts, one instance count per instance, chain
    steps at least the chain starts, and the plain sweep's decisions."""
    prof = profile_heavy(50)
    users = sample_batch(300, 50, prof, 0.25, 1.0, seed=77)
    a = engine.count_work(prof, users)
    b = engine.count_work(prof, users)
    assert a == b
    assert a["instances"] == 300
    assert a["og_chain_steps"] >= a["chain_starts"] > 0 and a["ip_chain_steps"] > 0
    assert a["dp_cells"] > 0 and a["bstar_steps"] > 0
    # [7]: the b* steps of instances whose groups do not all take their
    # largest admissible bound (group_b == group_size), the instances where
    # the pipelined kernel's speculative b* falls back to the full pass
    ip, og = engine.sweep(prof, users)
    miss = [k for k in range(300) if og["status"][k] == 0 and not og["fallback"][k]
            and any(og["group_b"][k][g] != og["group_size"][k][g] for g in range(og["n_groups"][k]))]
    assert 0 <= a["bstar_miss_steps"] <= a["bstar_steps"]
    assert (a["bstar_miss_steps"] > 0) == (len(miss) > 0)
    assert 0 < len(miss) < 300  # both branches occur at this size
