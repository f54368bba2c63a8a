"""Test-side access to the CPU checkers (oracle/), never used by the product.

  oracle()  -> oracle/liboracle.so         plain-C restatement (always buildable)
  ref()     -> oracle/_ref/libcoinfer_ref.so  the unmodified reference headers
               (built in the dev container from /root/reference; None if absent)

Both export the product ABI's SoA entry points, so the same Packed structs
drive them and the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2206_06304_b200 import _abi
from paper_2206_06304_b200.engine import Packed

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libcoinfer_ref.so")

_P, _U = C.POINTER(_abi.Profile), C.POINTER(_abi.Users)
_IO, _OO = C.POINTER(_abi.IpssaOut), C.POINTER(_abi.OgOut)
_dp, _i32p = C.POINTER(C.c_double), C.POINTER(C.c_int32)

ORACLE_SYMBOLS = {
    "oracle_ipssa_batch": (C.c_int, [_P, _U, _dp, _IO]),
    "oracle_fixed_batch": (C.c_int, [_P, _U, _dp, _i32p, _IO]),
    "oracle_og_batch": (C.c_int, [_P, _U, _OO, C.c_int]),
    "oracle_og_gtable": (C.c_int, [_P, _U, C.c_int64, C.c_int, _dp, _i32p]),
}

REF_SYMBOLS = {
    "ref_ipssa_batch": (C.c_int, [_P, _U, _dp, _IO]),
    "ref_fixed_batch": (C.c_int, [_P, _U, _dp, _i32p, _IO]),
    "ref_og_batch": (C.c_int, [_P, _U, _OO]),
    "ref_oracle_grouping_contiguous": (C.c_double, [_P, _U, C.c_int64, _i32p]),
    "ref_oracle_grouping": (C.c_double, [_P, _U, C.c_int64, _i32p]),
    "ref_sweep_threads": (C.c_double, [_P, _U, C.POINTER(C.c_int64), C.c_int64, C.c_int, C.c_int,
                                       C.c_int, _dp, _dp]),
    "ref_schedule_batch": (C.c_int, [_P, _U, _dp, C.c_int, _i32p, C.POINTER(_abi.ScheduleOut)]),
    "ref_validate_batch": (C.c_int, [_P, _U, C.POINTER(_abi.ScheduleOut), C.c_double, _i32p, _i32p, _dp]),
    "ref_baseline_batch": (C.c_int, [_P, _U, C.c_int, _IO, C.POINTER(_abi.ScheduleOut)]),
    "ref_oracle_structured": (C.c_double, [_P, _U, C.c_int64, C.c_double, C.c_int32,
                                           C.POINTER(C.c_uint8), C.POINTER(C.c_uint8),
                                           C.POINTER(C.c_uint8)]),
    "ref_oracle_groups": (C.c_double, [_P, _U, C.c_int64, C.c_int, _i32p, _i32p]),
    "ref_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "ref_sub_seed": (C.c_uint64, [C.c_uint64, C.c_uint64, C.c_uint64]),
    "ref_rng_new": (C.c_void_p, [C.c_uint64]),
    "ref_rng_free": (None, [C.c_void_p]),
    "ref_rng_next": (C.c_uint64, [C.c_void_p]),
    "ref_uniform_int": (C.c_uint64, [C.c_void_p, C.c_uint64, C.c_uint64]),
    "ref_uniform_real": (C.c_double, [C.c_void_p, C.c_double, C.c_double]),
    "ref_random_scenario": (None, [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double]
                            + [_dp] * 10),
    "ref_profile": (None, [C.c_int, C.c_int, _dp, _dp, _dp]),
    "ref_sample_scenario": (C.c_int, [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                      C.c_uint64] + [_dp] * 9),
    "ref_online_episode": (C.c_int, [_P, _U, C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_uint64, C.c_int, C.c_double, C.c_int64, _dp,
                                     C.POINTER(C.c_int64), _dp, _dp, _i32p, _dp]),
}

_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"),
                            os.path.join(ROOT, "oracle", "liboracle.so")], check=True)
        _oracle = _abi.bind(C.CDLL(ORACLE_SO), ORACLE_SYMBOLS)
    return _oracle


def ref():
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = _abi.bind(C.CDLL(REF_SO), REF_SYMBOLS)
    return _ref


def _call_ip(fn, profile, users, deadline=None, b=None):
    pk = Packed(profile, users, _abi.MEM_HOST, True, False)
    d = None if deadline is None else np.ascontiguousarray(deadline, dtype=np.float64)
    dp = d.ctypes.data_as(_dp) if d is not None else None
    if b is None:
        rc = fn(C.byref(pk.profile), C.byref(pk.users), dp, C.byref(pk.out_ip))
    else:
        bb = np.ascontiguousarray(b, dtype=np.int32)
        rc = fn(C.byref(pk.profile), C.byref(pk.users), dp, bb.ctypes.data_as(_i32p),
                C.byref(pk.out_ip))
    assert rc == 0, rc
    return Packed.arrays(pk.out_ip)


def oracle_ipssa(profile, users, deadline=None):
    return _call_ip(oracle().oracle_ipssa_batch, profile, users, deadline)


def oracle_fixed(profile, users, b, deadline=None):
    return _call_ip(oracle().oracle_fixed_batch, profile, users, deadline, b)


def oracle_og(profile, users, fast=True):
    pk = Packed(profile, users, _abi.MEM_HOST, False, True)
    assert oracle().oracle_og_batch(C.byref(pk.profile), C.byref(pk.users), C.byref(pk.out_og),
                                    1 if fast else 0) == 0
    return Packed.arrays(pk.out_og)


def ref_ipssa(profile, users, deadline=None):
    return _call_ip(ref().ref_ipssa_batch, profile, users, deadline)


def ref_fixed(profile, users, b, deadline=None):
    return _call_ip(ref().ref_fixed_batch, profile, users, deadline, b)


def ref_og(profile, users):
    pk = Packed(profile, users, _abi.MEM_HOST, False, True)
    assert ref().ref_og_batch(C.byref(pk.profile), C.byref(pk.users), C.byref(pk.out_og)) == 0
    return Packed.arrays(pk.out_og)


def _sched_struct(pk):
    return pk._alloc(_abi.SCHEDULE_FIELDS, _abi.ScheduleOut, None, _abi.MEM_HOST, None)


def ref_schedule(profile, users, kind, deadline=None):
    """The Schedule the reference's ip_ssa (kind "ipssa") or og returns, SoA."""
    pk = Packed(profile, users, _abi.MEM_HOST, False, False)
    so = _sched_struct(pk)
    st = np.zeros(pk.K, np.int32)
    d = None if deadline is None else np.ascontiguousarray(deadline, dtype=np.float64)
    assert ref().ref_schedule_batch(C.byref(pk.profile), C.byref(pk.users),
                                    d.ctypes.data_as(_dp) if d is not None else None,
                                    0 if kind == "ipssa" else 1, st.ctypes.data_as(_i32p),
                                    C.byref(so)) == 0
    out = Packed.arrays(so)
    out["status"] = st
    return out


def ref_baseline(profile, users, mode):
    """baseline(sc, BaselineMode[mode]) through the reference: (SolveResult, Schedule)."""
    pk = Packed(profile, users, _abi.MEM_HOST, True, False)
    so = _sched_struct(pk)
    rc = ref().ref_baseline_batch(C.byref(pk.profile), C.byref(pk.users),
                                  _abi.BASELINE_MODES[mode], C.byref(pk.out_ip), C.byref(so))
    assert rc == 0, rc
    return Packed.arrays(pk.out_ip), Packed.arrays(so)


def ref_validate(profile, users, sched, tol=1e-9):
    """validate() through the reference: status, counts per constraint id, worst slack."""
    pk = Packed(profile, users, _abi.MEM_HOST, False, False)
    arrays = {k: np.ascontiguousarray(_to_np(v)) for k, v in sched.items()}
    ptrs = [arrays[n].ctypes.data_as(t) for n, t, _ in _abi.SCHEDULE_FIELDS]
    so = _abi.ScheduleOut(*ptrs)
    K = pk.K
    st = np.zeros(K, np.int32)
    cnt = np.zeros((K, _abi.N_CONSTRAINTS), np.int32)
    sl = np.zeros(K)
    assert ref().ref_validate_batch(C.byref(pk.profile), C.byref(pk.users), C.byref(so), float(tol),
                                    st.ctypes.data_as(_i32p), cnt.ctypes.data_as(_i32p),
                                    sl.ctypes.data_as(_dp)) == 0
    return dict(status=st, counts=cnt, min_slack=sl)


def ref_oracle_structured(profile, users, deadline, b):
    """oracle_structured per instance through the reference."""
    pk = Packed(profile, users, _abi.MEM_HOST, False, False)
    K, M = pk.K, pk.M
    out = dict(energy=np.zeros(K), split=np.zeros((K, M), np.uint8), fallback=np.zeros(K, np.uint8),
               feasible=np.zeros(K, np.uint8))
    for k in range(K):
        sp = np.zeros(M, np.uint8)
        fb, fe = C.c_uint8(), C.c_uint8()
        out["energy"][k] = ref().ref_oracle_structured(C.byref(pk.profile), C.byref(pk.users), k,
                                                       float(deadline[k]), int(b[k]),
                                                       sp.ctypes.data_as(C.POINTER(C.c_uint8)),
                                                       C.byref(fb), C.byref(fe))
        out["split"][k], out["fallback"][k], out["feasible"][k] = sp, fb.value, fe.value
    return out


def ref_oracle_groups(profile, users, contiguous):
    """oracle_grouping(_contiguous) per instance through the reference."""
    pk = Packed(profile, users, _abi.MEM_HOST, False, False)
    K, M = pk.K, pk.M
    out = dict(energy=np.zeros(K), n_groups=np.zeros(K, np.int32), group_of_user=np.zeros((K, M), np.int32))
    for k in range(K):
        ng = C.c_int32()
        gu = np.zeros(M, np.int32)
        out["energy"][k] = ref().ref_oracle_groups(C.byref(pk.profile), C.byref(pk.users), k,
                                                   1 if contiguous else 0, C.byref(ng),
                                                   gu.ctypes.data_as(_i32p))
        out["n_groups"][k], out["group_of_user"][k] = ng.value, gu
    return out


def assert_same_schedule(a: dict, b: dict, status, where=""):
    """Schedules of the solved instances (status 0) equal bit for bit."""
    ok = np.asarray(_to_np(status)) == 0
    nb_a, nb_b = _to_np(a["n_batches"]), _to_np(b["n_batches"])
    np.testing.assert_array_equal(nb_a[ok], nb_b[ok], err_msg=f"{where} n_batches")
    for key in ("x", "completion", "freq"):
        np.testing.assert_array_equal(_to_np(a[key])[ok], _to_np(b[key])[ok], err_msg=f"{where} {key}")
    bs_a, bs_b = _to_np(a["batch_start"]), _to_np(b["batch_start"])
    for k in np.nonzero(ok)[0]:
        n = int(nb_a[k])
        np.testing.assert_array_equal(bs_a[k].reshape(-1)[:n], bs_b[k].reshape(-1)[:n],
                                      err_msg=f"{where} batch_start[{k}]")


# --------------------------------------------------------------- comparison

IP_KEYS = ["status", "batch_bound", "pipeline_feasible", "energy", "split", "freq",
           "user_energy", "batch_size"]
OG_KEYS = ["status", "fallback", "energy", "n_groups", "order", "group_of_user", "split", "freq",
           "user_energy", "group_lo", "group_size", "group_b", "group_deadline", "group_energy",
           "group_batch_size"]


def _to_np(x):
    if hasattr(x, "cpu"):
        return x.cpu().numpy()
    return np.asarray(x)


def mask_valid(out: dict, kind: str, M: int):
    """Entries that are defined (status OK; groups below n_groups)."""
    st = _to_np(out["status"])
    ok = st == 0
    return ok


def assert_same_ip(a: dict, b: dict, exact_energy=True, rtol=1e-9, where=""):
    a = {k: _to_np(v) for k, v in a.items()}
    b = {k: _to_np(v) for k, v in b.items()}
    np.testing.assert_array_equal(a["status"], b["status"], err_msg=f"status {where}")
    ok = a["status"] == 0
    for k in ["batch_bound", "pipeline_feasible", "split", "batch_size"]:
        if k in a and k in b:
            np.testing.assert_array_equal(a[k][ok], b[k][ok], err_msg=f"{k} {where}")
    for k in ["energy", "freq", "user_energy"]:
        if k in a and k in b:
            if exact_energy:
                np.testing.assert_array_equal(a[k][ok], b[k][ok], err_msg=f"{k} {where}")
            else:
                np.testing.assert_allclose(a[k][ok], b[k][ok], rtol=rtol, atol=0,
                                           err_msg=f"{k} {where}")


def assert_same_og(a: dict, b: dict, exact_energy=True, rtol=1e-9, where=""):
    a = {k: _to_np(v) for k, v in a.items()}
    b = {k: _to_np(v) for k, v in b.items()}
    np.testing.assert_array_equal(a["status"], b["status"], err_msg=f"status {where}")
    ok = a["status"] == 0
    for k in ["fallback", "n_groups", "order", "group_of_user", "split"]:
        if k in a and k in b:
            np.testing.assert_array_equal(a[k][ok], b[k][ok], err_msg=f"{k} {where}")
    for k in ["energy", "freq", "user_energy"]:
        if k in a and k in b:
            if exact_energy:
                np.testing.assert_array_equal(a[k][ok], b[k][ok], err_msg=f"{k} {where}")
            else:
                np.testing.assert_allclose(a[k][ok], b[k][ok], rtol=rtol, atol=0,
                                           err_msg=f"{k} {where}")
    # per-group arrays: only the first n_groups entries are defined
    ng = a["n_groups"]
    for idx in np.nonzero(ok)[0]:
        g = int(ng[idx])
        for k in ["group_lo", "group_size", "group_b", "group_batch_size"]:
            if k in a and k in b:
                np.testing.assert_array_equal(a[k][idx][:g], b[k][idx][:g],
                                              err_msg=f"{k} inst {idx} {where}")
        for k in ["group_deadline", "group_energy"]:
            if k in a and k in b:
                if exact_energy:
                    np.testing.assert_array_equal(a[k][idx][:g], b[k][idx][:g],
                                                  err_msg=f"{k} inst {idx} {where}")
                else:
                    np.testing.assert_allclose(a[k][idx][:g], b[k][idx][:g], rtol=rtol,
                                               err_msg=f"{k} inst {idx} {where}")


# ------------------------------------------------------------ instance makers

def two_stage(users=1, b_max=8):
    """testutil::two_stage (tests/helpers.hpp:17-38) as one-instance SoA."""
    from paper_2206_06304_b200.engine import ProfileArrays
    prof = ProfileArrays(np.array([0.01, 0.01]), np.array([1e6, 2e4, 0.0]),
                         np.full((2, b_max), 0.01))
    one = np.ones((1, users))
    u = dict(f_min=0 * one, f_max=one * 1.0, kappa=one * 300.0, rate_up=one * 1e6,
             rate_down=one * 1e6, power_up=one * 1.0, power_down=one * 1.0, arrival=0 * one,
             deadline=one * 0.1)
    return prof, u


def ref_random_scenario(rng_handle, users, subtasks, growth_max, equal, margin_max=3.0):
    """testutil::random_scenario through the reference (needs oracle/_ref)."""
    from paper_2206_06304_b200.engine import ProfileArrays
    r = ref()
    bmax = users + 2
    work = np.zeros(subtasks)
    bits = np.zeros(subtasks + 1)
    lat = np.zeros(subtasks * bmax)
    arrs = [np.zeros((1, users)) for _ in range(7)]
    r.ref_random_scenario(rng_handle, users, subtasks, growth_max, 1 if equal else 0, margin_max,
                          *[a.ctypes.data_as(_dp) for a in [work, bits, lat] + arrs])
    prof = ProfileArrays(work, bits, lat.reshape(subtasks, bmax))
    names = ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline"]
    u = dict(zip(names, arrs))
    u["rate_down"] = u["rate_up"].copy()
    u["power_down"] = u["power_up"].copy()
    return prof, u


def ref_sample_scenarios(n_inst, M, low, high, seeds, heavy=True, bandwidth=1e6):
    """sample_scenario + profile_heavy/light through the reference, one seed per instance."""
    from paper_2206_06304_b200.engine import ProfileArrays
    r = ref()
    work, bits, lat = np.zeros(4), np.zeros(5), np.zeros(4 * M)
    r.ref_profile(1 if heavy else 0, M, work.ctypes.data_as(_dp), bits.ctypes.data_as(_dp),
                  lat.ctypes.data_as(_dp))
    prof = ProfileArrays(work, bits, lat.reshape(4, M))
    names = ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline",
             "rate_down", "power_down"]
    u = {n: np.zeros((n_inst, M)) for n in names}
    for k in range(n_inst):
        row = [np.zeros(M) for _ in names]
        assert r.ref_sample_scenario(1 if heavy else 0, M, low, high, bandwidth, int(seeds[k]),
                                     *[a.ctypes.data_as(_dp) for a in row]) == 0
        for n, a in zip(names, row):
            u[n][k] = a
    return prof, u


def slice_users(u, k0, k1):
    return {n: v[k0:k1] for n, v in u.items()}


def ref_online(profile, users, cfg, seed, trace=True):
    """run_episode(OnlineEnv(scenario 0 of users, ...), TimeWindowPolicy(window, l_high),
    horizon, seed) through the reference (needs oracle/_ref).  Returns a dict
    like Engine.online for one episode."""
    import ctypes as C
    pk = Packed(profile, users, _abi.MEM_HOST, False, False)
    H = int(cfg.horizon)
    totals = np.zeros(4)
    counts = np.zeros(6, dtype=np.int64)
    rw, en, bu = np.zeros(H), np.zeros(H), np.zeros(H)
    pe = np.zeros(H, dtype=np.int32)
    rc = ref().ref_online_episode(
        C.byref(pk.profile), C.byref(pk.users), 1 if cfg.solver == "og" else 0, cfg.p_arrive,
        1 if cfg.arrival == "immediate" else 0, cfg.l_low, cfg.l_high, cfg.slot, int(seed),
        -1 if cfg.policy == "local" else int(cfg.window),
        cfg.l_high if cfg.threshold is None else cfg.threshold, H, totals.ctypes.data_as(_dp), counts.ctypes.data_as(C.POINTER(C.c_int64)),
        rw.ctypes.data_as(_dp), en.ctypes.data_as(_dp), pe.ctypes.data_as(_i32p),
        bu.ctypes.data_as(_dp))
    return dict(rc=rc, totals=totals[:3], counts=counts, trace_reward=rw, trace_energy=en,
                trace_pending=pe, trace_edge_busy=bu)
