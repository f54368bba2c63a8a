"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run in the dev container (needs /root/reference, built by `make -C oracle`):
    python tests/golden/make_golden.py

Every case records inputs (profile + SoA users) and the reference's outputs
through the same ABI the CUDA engine exports.  Instance streams replay the
reference's own tests with their seeds (test_offline_solvers.cpp,
test_oracles.cpp, acceptance_main.cpp, test_online_sim.cpp) plus CLI-style
scenarios (sample_scenario + profile_heavy/light seeded with sub_seed, as
coinfer_main.cpp:47-50,348-350 does).  JSON floats round-trip exactly.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import checkers as ck  # noqa: E402
from paper_2206_06304_b200.engine import ProfileArrays  # noqa: E402

R = ck.ref()
assert R is not None, "build oracle/_ref first (make -C oracle)"


def enc(a):
    a = np.asarray(a)
    return a.tolist()


def case(name, kind, prof, users, deadline=None, b=None, expect=None, extra=None):
    return dict(name=name, kind=kind,
                profile=dict(work=enc(prof.work), data_bits=enc(prof.data_bits),
                             latency=enc(prof.latency)),
                users={k: enc(v) for k, v in users.items()},
                deadline=None if deadline is None else enc(deadline),
                b=None if b is None else enc(b), expect={k: enc(v) for k, v in expect.items()},
                extra=extra or {})


def solve(name, kind, prof, u, deadline=None, b=None, extra=None):
    if kind == "ipssa":
        out = ck.ref_ipssa(prof, u, deadline)
    elif kind == "fixed":
        out = ck.ref_fixed(prof, u, b, deadline)
    elif kind == "og":
        out = ck.ref_og(prof, u)
    else:
        raise ValueError(kind)
    return case(name, kind, prof, u, deadline, b, out, extra)


def cat(cases_users):
    """Stack single-instance user dicts sharing one profile."""
    keys = cases_users[0].keys()
    return {k: np.concatenate([u[k] for u in cases_users], 0) for k in keys}


def kat_cases():
    out = []
    prof, u = ck.two_stage(1)
    out.append(solve("two_stage_ipssa", "ipssa", prof, u, [0.1]))
    out.append(solve("two_stage_fixed_b1", "fixed", prof, u, [0.1], [1]))
    out.append(solve("two_stage_og", "og", prof, u))
    prof2, u2 = ck.two_stage(2)
    out.append(solve("two_stage2_ipssa", "ipssa", prof2, u2, [0.1]))
    out.append(solve("two_stage2_fixed_b2", "fixed", prof2, u2, [0.1], [2]))
    out.append(solve("two_stage2_og", "og", prof2, u2))
    # TieGoesToLargerSplit (test_offline_solvers.cpp:68-80)
    p, v = ck.two_stage(1)
    v["kappa"][:] = 0.0
    v["power_up"][:] = 0.0
    out.append(solve("tie_larger_split_fixed", "fixed", p, v, [0.1], [1]))
    out.append(solve("tie_larger_split_ipssa", "ipssa", p, v, [0.1]))
    # RespectsFrequencyFloor (:82-92)
    p, v = ck.two_stage(1)
    v["f_min"][:] = 0.5
    out.append(solve("freq_floor_fixed", "fixed", p, v, [0.1], [1]))
    # FallsBackToLocalWhenPipelineTooLong (:133-143)
    p, v = ck.two_stage(1)
    p = ProfileArrays(p.work, p.data_bits, np.full((2, 8), 0.05))
    v["deadline"][:] = 0.03
    out.append(solve("pipeline_fallback_fixed", "fixed", p, v, [0.03], [1]))
    out.append(solve("pipeline_fallback_ipssa", "ipssa", p, v, [0.03]))
    out.append(solve("pipeline_fallback_og", "og", p, v))
    # ThrowsWhenDeadlineUnreachable (:145-149)
    p, v = ck.two_stage(1)
    v["deadline"][:] = 0.015
    out.append(solve("unreachable_fixed", "fixed", p, v, [0.015], [1]))
    out.append(solve("unreachable_ipssa", "ipssa", p, v, [0.015]))
    out.append(solve("unreachable_og", "og", p, v))
    # StaggeredDeadlinesSplitWhenPipelinesFit (:192-205)
    p, v = ck.two_stage(2)
    lat = np.array([[0.01] + [0.02] * 7, [0.01] + [0.02] * 7])
    p = ProfileArrays(p.work, p.data_bits, lat)
    v["deadline"][0] = [0.1, 0.2]
    out.append(solve("staggered_og", "og", p, v))
    out.append(solve("staggered_ipssa_0.1", "ipssa", p, v, [0.1]))
    # ClipThresholdFeedsSolverClippedDeadlines (test_online_sim.cpp:97-116)
    p, v = ck.two_stage(2)
    v["deadline"][0] = [0.3, 0.5]
    out.append(solve("clipped_og", "og", p, v))
    # ManyUsersStaysFeasible (:351-356)
    p, v = ck.two_stage(200, 200)
    out.append(solve("many_users_fixed_b200", "fixed", p, v, [0.1], [200]))
    # OG lc fallback: no contiguous grouping works, everyone still local-feasible
    p, v = ck.two_stage(2)
    p = ProfileArrays(p.work, p.data_bits, np.full((2, 8), 0.1))
    v["deadline"][0] = [0.1, 0.1001]
    v["f_max"][0] = [1.0, 0.02 / 0.10005]
    out.append(solve("og_lc_fallback", "og", p, v))
    # contract violations, one per Scenario::check test (core_model.hpp:88-99)
    bad = []
    for field, val in [("f_max", 0.0), ("kappa", -1.0), ("rate_up", 0.0), ("power_up", -1.0),
                       ("arrival", -1.0), ("deadline", 0.0)]:
        p, v = ck.two_stage(3)
        v[field][0, 1] = val
        bad.append(v)
    p, v = ck.two_stage(3)
    v["f_min"][0, 2] = 2.0  # f_min > f_max
    v["kappa"][0, 0] = -5.0  # first failing user wins
    bad.append(v)
    bu = cat(bad)
    out.append(solve("contract_ipssa", "ipssa", p, bu))
    out.append(solve("contract_og", "og", p, bu))
    out.append(solve("contract_fixed", "fixed", p, bu, None, [1] * bu["deadline"].shape[0]))
    p, v = ck.two_stage(9, 8)  # latency table shorter than the user count
    out.append(solve("short_table_og", "og", p, v))
    p, v = ck.two_stage(2)
    out.append(solve("zero_bound_fixed", "fixed", p, v, [0.1], [0]))
    out.append(solve("bound_past_table_fixed", "fixed", p, v, [0.1], [9]))
    return out


def stream(seed, salt, n, make):
    rng = R.ref_rng_new(R.ref_mix_seed(seed, salt))
    try:
        return [make(rng, i) for i in range(n)]
    finally:
        R.ref_rng_free(rng)


def random_cases():
    out = []
    # test_offline_solvers.cpp:159-177 (ip_ssa at deadline[0], equal deadlines)
    for seed, fn in [(77, lambda i: (1 + i % 5, 2 + i % 3, 0.4)), (78, lambda i: (2 + i % 5, 2 + i % 4, 0.5))]:
        inst = stream(seed, 0, 25, lambda rng, i: ck.ref_random_scenario(rng, *fn(i), True))
        for i, (p, u) in enumerate(inst):
            out.append(solve(f"ipssa_seed{seed}_{i}", "ipssa", p, u, u["deadline"][:, 0]))
    # test_offline_solvers.cpp:179-217 (og)
    inst = stream(79, 0, 10, lambda rng, i: ck.ref_random_scenario(rng, 2 + i % 4, 2 + i % 3, 0.5, True))
    for i, (p, u) in enumerate(inst):
        out.append(solve(f"og_equal_seed79_{i}", "og", p, u))
        out.append(solve(f"ipssa_equal_seed79_{i}", "ipssa", p, u, u["deadline"][:, 0]))
    inst = stream(80, 0, 10, lambda rng, i: ck.ref_random_scenario(rng, 2 + i % 5, 2 + i % 3, 0.4, False))
    for i, (p, u) in enumerate(inst):
        out.append(solve(f"og_seed80_{i}", "og", p, u))

    # test_oracles.cpp:76-114 with the brute-force optima recorded
    def mk103(rng, i):
        M = int(R.ref_uniform_int(rng, 2, 6))
        return ck.ref_random_scenario(rng, M, 2 + i % 3, 0.5, False)

    for i, (p, u) in enumerate(stream(103, 0, 20, mk103)):
        ng = C.c_int32()
        c = solve(f"og_contig_seed103_{i}", "og", p, u)
        pk = ck.Packed(p, u, 0, False, True)
        e = R.ref_oracle_grouping_contiguous(C.byref(pk.profile), C.byref(pk.users), 0, C.byref(ng))
        c["extra"] = dict(contiguous_energy=e, contiguous_groups=ng.value)
        out.append(c)

    def mk104(rng, i):
        M = int(R.ref_uniform_int(rng, 2, 6))
        return ck.ref_random_scenario(rng, M, 2 + i % 3, 0.0, False)

    for i, (p, u) in enumerate(stream(104, 0, 12, mk104)):
        c = solve(f"og_setpart_seed104_{i}", "og", p, u)
        pk = ck.Packed(p, u, 0, False, True)
        ng = C.c_int32()
        e = R.ref_oracle_grouping(C.byref(pk.profile), C.byref(pk.users), 0, C.byref(ng))
        c["extra"] = dict(partition_energy=e, partition_groups=ng.value)
        out.append(c)

    # acceptance_main.cpp:46-69 (split search), first 60 of the 200
    def mk701(rng, i):
        M = int(R.ref_uniform_int(rng, 1, 4))
        N = int(R.ref_uniform_int(rng, 2, 4))
        p, u = ck.ref_random_scenario(rng, M, N, 0.0, True)
        b = int(R.ref_uniform_int(rng, 1, M))
        return p, u, b

    for i, (p, u, b) in enumerate(stream(701, 1, 60, mk701)):
        out.append(solve(f"fixed_accept1_{i}", "fixed", p, u, u["deadline"][:, 0], [b]))

    # acceptance_main.cpp:76-108 (grouping vs brute force), first 40
    def mk702(rng, i):
        M = int(R.ref_uniform_int(rng, 2, 6))
        N = int(R.ref_uniform_int(rng, 2, 4))
        return ck.ref_random_scenario(rng, M, N, 0.0, False)

    for i, (p, u) in enumerate(stream(702, 1, 40, mk702)):
        out.append(solve(f"og_accept2_{i}", "og", p, u))
    return out


def cli_cases():
    """CLI-style scenarios: sample_scenario(mt19937_64(sub_seed(1,1,k)))."""
    out = []
    seeds = [R.ref_sub_seed(1, 1, k) for k in range(8)]
    p, u = ck.ref_sample_scenarios(1, 10, 0.25, 0.25, seeds[:1])
    out.append(solve("C1_ipssa_M10", "ipssa", p, u, [0.25]))
    out.append(solve("C1_og_M10", "og", p, u))
    p, u = ck.ref_sample_scenarios(8, 50, 0.25, 1.0, seeds)
    out.append(solve("C3_ipssa_M50", "ipssa", p, u))
    out.append(solve("C3_og_M50", "og", p, u))
    p, u = ck.ref_sample_scenarios(1, 100, 0.25, 1.0, seeds[:1])
    out.append(solve("C2_og_M100", "og", p, u))
    out.append(solve("C2_ipssa_M100", "ipssa", p, u))
    p, u = ck.ref_sample_scenarios(6, 14, 0.05, 0.2, seeds[:6], heavy=False)
    out.append(solve("light_og_M14", "og", p, u))
    out.append(solve("light_ipssa_M14", "ipssa", p, u))
    p, u = ck.ref_sample_scenarios(4, 15, 0.25, 0.25, seeds[:4], bandwidth=5e6)
    out.append(solve("fixed025_og_M15_5MHz", "og", p, u))
    return out


def online_cases():
    """run_episode traces from the reference: the reference tests' own online
    setups (test_online_sim.cpp) and CLI-style episodes (coinfer_main.cpp:482-573)."""
    from paper_2206_06304_b200.engine import OnlineConfig
    out = []

    def ep(name, prof, u, cfg, seed):
        r = ck.ref_online(prof, u, cfg, seed)
        assert r["rc"] == 0, name
        out.append(dict(name=name, profile=dict(work=enc(prof.work), data_bits=enc(prof.data_bits),
                                                latency=enc(prof.latency)),
                        users={k: enc(v) for k, v in u.items()}, cfg=cfg.__dict__, seed=int(seed),
                        expect={k: enc(v) for k, v in r.items() if k != "rc"}))

    # test_online_sim.cpp:231-248, 250-268, 320-335, 157-176, 209-229
    p, u = ck.two_stage(3)
    ep("accounting_og_tw1", p, u, OnlineConfig("bernoulli", 0.35, 0.1, 0.4, 0.025, "og", "tw", 1, 0.4, 400), 23)
    p, u = ck.two_stage(4)
    ep("reproduce_ipssa_tw2", p, u, OnlineConfig("bernoulli", 0.4, 0.1, 0.4, 0.025, "ipssa", "tw", 2, 0.4, 250), 31)
    p, u = ck.two_stage(5)
    ep("deadline_safe_og_tw3", p, u, OnlineConfig("bernoulli", 0.6, 0.08, 0.5, 0.025, "og", "tw", 3, 0.2, 600), 41)
    ep("deadline_safe_ipssa_tw3", p, u, OnlineConfig("bernoulli", 0.6, 0.08, 0.5, 0.025, "ipssa", "tw", 3, 0.2, 600), 41)
    p, u = ck.two_stage(3)
    ep("certain_arrival_local", p, u, OnlineConfig("bernoulli", 1.0, 0.1, 0.4, 0.025, "og", "local", 0, None, 200), 17)
    ep("immediate_local", p, u, OnlineConfig("immediate", 1.0, 0.1, 0.4, 0.025, "og", "local", 0, None, 200), 17)
    # CLI online path: sample_scenario(users, fixed(l_high)) with sub_seed(root, 1, 0)
    s0 = R.ref_sub_seed(1, 1, 0)
    p, u = ck.ref_sample_scenarios(1, 14, 1.0, 1.0, [s0], heavy=True)
    for ep_i in range(2):
        ep(f"cli_heavy_og_tw0_ep{ep_i}", p, u, OnlineConfig("bernoulli", 0.05, 0.25, 1.0, 0.025, "og", "tw", 0, None, 4000),
           R.ref_sub_seed(1, 5, ep_i))
    ep("cli_heavy_ipssa_tw2", p, u, OnlineConfig("bernoulli", 0.1, 0.25, 1.0, 0.025, "ipssa", "tw", 2, None, 4000),
       R.ref_sub_seed(1, 5, 7))
    p, u = ck.ref_sample_scenarios(1, 14, 0.2, 0.2, [s0], heavy=False)
    ep("cli_light_og_tw0", p, u, OnlineConfig("bernoulli", 0.25, 0.05, 0.2, 0.025, "og", "tw", 0, None, 4000),
       R.ref_sub_seed(1, 5, 0))
    p, u = ck.ref_sample_scenarios(1, 6, 1.0, 1.0, [s0], heavy=False)
    ep("cli_default_light_tw2", p, u, OnlineConfig("bernoulli", 0.25, 0.25, 1.0, 0.025, "og", "tw", 2, None, 2000),
       R.ref_sub_seed(1, 5, 3))
    return out


def main():
    for name, fn in [("kat", kat_cases), ("random", random_cases), ("cli", cli_cases),
                     ("online", online_cases)]:
        cases = fn()
        path = os.path.join(HERE, f"{name}.json")
        with open(path, "w") as f:
            json.dump(cases, f, separators=(",", ":"))
        print(path, len(cases), "cases", os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
