"""The CPU oracle (oracle/coinfer_oracle.c) pinned against the reference:
golden fixtures from the unmodified reference headers plus the reference
tests' own known answers.  CPU only."""
import math

import numpy as np
import pytest

import checkers as ck
import golden_io

CASES = golden_io.all_cases()


def run_oracle(c, fast=True):
    if c["kind"] == "ipssa":
        return ck.oracle_ipssa(c["profile"], c["users"], c["deadline"])
    if c["kind"] == "fixed":
        return ck.oracle_fixed(c["profile"], c["users"], c["b"], c["deadline"])
    return ck.oracle_og(c["profile"], c["users"], fast=fast)


@pytest.mark.parametrize("c", CASES, ids=[c["name"] for c in CASES])
def test_oracle_matches_reference_fixture(c):
    out = run_oracle(c)
    if c["kind"] == "og":
        ck.assert_same_og(out, c["expect"], where=c["name"])
        if c["users"]["deadline"].shape[1] <= 16:
            ck.assert_same_og(run_oracle(c, fast=False), c["expect"], where=c["name"] + " direct")
    else:
        ck.assert_same_ip(out, c["expect"], where=c["name"])


def by_name(name):
    return next(c for c in CASES if c["name"] == name)


K2 = 3.0 / 49.0 + 0.02  # kTwoStageSplitEnergy (test_offline_solvers.cpp:20)


def double_eq(a, b):
    """GoogleTest EXPECT_DOUBLE_EQ: within 4 ULPs."""
    return abs(a - b) <= 4 * np.spacing(max(abs(a), abs(b)))


def test_kat_two_stage():
    o = run_oracle(by_name("two_stage_fixed_b1"))
    assert o["split"][0, 0] == 1 and list(o["batch_size"][0]) == [0, 1]
    assert abs(o["energy"][0] - K2) < 1e-12
    assert double_eq(o["freq"][0, 0], 0.01 / 0.07)
    o = run_oracle(by_name("two_stage2_ipssa"))
    assert o["batch_bound"][0] == 2 and abs(o["energy"][0] - 2 * K2) < 1e-12
    assert abs(o["user_energy"][0, 0] - K2) < 1e-12  # Metrics.TwoUserSplitSchedule


def test_kat_ties_floor_fallback():
    o = run_oracle(by_name("tie_larger_split_fixed"))
    assert o["split"][0, 0] == 2 and o["energy"][0] == 0.0 and double_eq(o["freq"][0, 0], 0.2)
    o = run_oracle(by_name("freq_floor_fixed"))
    assert o["freq"][0, 0] >= 0.5
    if o["split"][0, 0] == 1:
        assert abs(o["energy"][0] - (300.0 * 0.01 * 0.25 + 0.02)) < 1e-12
    o = run_oracle(by_name("pipeline_fallback_fixed"))
    assert o["pipeline_feasible"][0] == 0 and o["split"][0, 0] == 2
    assert abs(o["energy"][0] - 300.0 * 0.02 * (2.0 / 3.0) ** 2) < 1e-12
    assert run_oracle(by_name("unreachable_fixed"))["status"][0] == ck._abi.ST_INFEASIBLE
    o = run_oracle(by_name("many_users_fixed_b200"))
    assert o["batch_size"][0, 1] == 200


def test_kat_contracts():
    o = run_oracle(by_name("contract_og"))
    assert list(o["status"]) == [10, 11, 12, 13, 14, 15, 11]
    assert run_oracle(by_name("short_table_og"))["status"][0] == ck._abi.ST_SHORT_TABLE
    assert run_oracle(by_name("zero_bound_fixed"))["status"][0] == ck._abi.ST_ZERO_BOUND
    assert run_oracle(by_name("bound_past_table_fixed"))["status"][0] == ck._abi.ST_BOUND_PAST_TABLE


def test_og_equal_deadlines_collapse_bitwise():
    # Og.EqualDeadlinesCollapseToOneGroup (test_offline_solvers.cpp:179-190)
    for i in range(10):
        og = run_oracle(by_name(f"og_equal_seed79_{i}"))
        ip = run_oracle(by_name(f"ipssa_equal_seed79_{i}"))
        assert og["n_groups"][0] == 1
        assert og["energy"][0] == ip["energy"][0]


def test_og_matches_brute_force_optima():
    # OracleGrouping.ContiguousBruteForceMatchesDp / ContiguousIsOptimalForConstantLatency
    for c in CASES:
        ex = c["extra"]
        if "contiguous_energy" in ex:
            o = run_oracle(c)
            if ex["contiguous_groups"] < 0:
                assert o["fallback"][0] == 1
            else:
                assert o["fallback"][0] == 0
                assert o["energy"][0] == ex["contiguous_energy"]
                assert o["n_groups"][0] == ex["contiguous_groups"]
        if "partition_energy" in ex:
            o = run_oracle(c)
            if ex["partition_groups"] >= 0:
                e, f = o["energy"][0], ex["partition_energy"]
                assert abs(e - f) / max(abs(e), abs(f), 1e-30) < 1e-9


def test_og_fast_equals_direct_gtable():
    """The O(M^3 N) shared-fold G table equals per-cell try_ip_ssa bit for bit."""
    import ctypes as C
    from paper_2206_06304_b200.engine import Packed
    for c in golden_io.load("cli")[:3] + golden_io.load("random")[50:90]:
        prof, users = c["profile"], c["users"]
        K, M = users["deadline"].shape
        if M > 20:
            users = {k: v[:1, :20] for k, v in users.items()}
            M = 20
        pk = Packed(prof, users, 0, False, False)
        for fast in (0, 1):
            G = np.zeros((M, M))
            B = np.zeros((M, M), dtype=np.int32)
            ck.oracle().oracle_og_gtable(C.byref(pk.profile), C.byref(pk.users), 0, fast,
                                         G.ctypes.data_as(C.POINTER(C.c_double)),
                                         B.ctypes.data_as(C.POINTER(C.c_int32)))
            if fast == 0:
                G0, B0 = G.copy(), B.copy()
        np.testing.assert_array_equal(G, G0)
        fin = np.isfinite(G0)
        np.testing.assert_array_equal(B[fin], B0[fin])


def test_og_fast_b_collapse_equals_direct_gtable():
    """Rows whose pipeline stops fitting inside the row (b0 <= M - i) take the
    collapsed all-local pass and the dead-chain cut of the fast form; it must
    still equal per-cell try_ip_ssa bit for bit (M = 60, tight deadlines)."""
    import ctypes as C
    from paper_2206_06304_b200 import profile_heavy, sample_batch
    from paper_2206_06304_b200.engine import Packed
    M = 60
    prof = profile_heavy(M)
    users = sample_batch(2, M, prof, 0.25, 0.6, seed=77)
    pk = Packed(prof, users, 0, False, False)
    for k in range(2):
        out = {}
        for fast in (0, 1):
            G = np.zeros((M, M))
            B = np.zeros((M, M), dtype=np.int32)
            ck.oracle().oracle_og_gtable(C.byref(pk.profile), C.byref(pk.users), k, fast,
                                         G.ctypes.data_as(C.POINTER(C.c_double)),
                                         B.ctypes.data_as(C.POINTER(C.c_int32)))
            out[fast] = (G, B)
        (G0, B0), (G1, B1) = out[0], out[1]
        np.testing.assert_array_equal(G1, G0)
        fin = np.isfinite(G0)
        assert fin.sum() > M  # finite groups beyond the diagonal
        np.testing.assert_array_equal(B1[fin], B0[fin])
        assert (B0[fin] > 20).any()  # collapsed bounds (b >= b0 ~ 20 at l = 0.25) won cells
    ck.assert_same_og(ck.oracle_og(prof, users, fast=True), ck.oracle_og(prof, users, fast=False),
                      where="fast vs direct og")
