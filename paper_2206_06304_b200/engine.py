"""Batch solver engine: the Python face of the C ABI (include/coinfer_b200.h).

Inputs are structure-of-arrays batches: every user field is a (n_inst, M)
float64 array, either numpy (host memory; the call stages it through the
GPU) or a CUDA torch tensor (device memory; the call enqueues on the
engine's stream and returns device tensors without synchronising).

All solving happens in the sm_100a kernels of libcoinfer_b200.so; there is
no CPU code path behind these calls.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, Optional

import numpy as np

from . import _abi

try:  # torch is plumbing only (device memory, streams)
    import torch
except Exception:  # pragma: no cover
    torch = None


@dataclass
class ProfileArrays:
    """DnnProfile in flat form (core_model.hpp:17-53)."""
    work: np.ndarray        # [N]
    data_bits: np.ndarray   # [N+1]
    latency: np.ndarray     # [N, b_max], F_n(b) at [n-1, b-1]

    @property
    def N(self) -> int:
        return int(self.work.shape[0])

    @property
    def b_max(self) -> int:
        return int(self.latency.shape[1])


def as_profile(p) -> ProfileArrays:
    if isinstance(p, ProfileArrays):
        return p
    lat = np.ascontiguousarray(np.asarray(p.latency, dtype=np.float64))
    if lat.ndim == 1:
        lat = lat.reshape(len(p.work), -1)
    return ProfileArrays(np.ascontiguousarray(np.asarray(p.work, dtype=np.float64)),
                         np.ascontiguousarray(np.asarray(p.data_bits, dtype=np.float64)), lat)


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _ptr(x, ctype):
    if x is None:
        return C.cast(None, C.POINTER(ctype))
    if _is_torch(x):
        return C.cast(C.c_void_p(x.data_ptr()), C.POINTER(ctype))
    return x.ctypes.data_as(C.POINTER(ctype))


_CT = {"d": C.c_double, "i": C.c_int32, "u": C.c_uint8}
_NP = {"d": np.float64, "i": np.int32, "u": np.uint8}
_TT = {"d": "float64", "i": "int32", "u": "uint8"}


def _kind(ctype) -> str:
    return {C.POINTER(C.c_double): "d", C.POINTER(C.c_int32): "i",
            C.POINTER(C.c_uint8): "u"}[ctype]


_PINNED = {}


def _pinned_buffer(owner, name, shape, dtype):
    """Reusable page-locked staging array (allocating pinned memory per call
    costs more than the copy).  Results in it are overwritten by the next
    pinned call with the same output.  `owner` (the output struct) is part of
    the key: IP-SSA and OG share field names (status, energy, split, ...)."""
    key = (owner, name, tuple(shape), np.dtype(dtype).str)
    a = _PINNED.get(key)
    if a is None:
        a = torch.empty(shape, dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True).numpy()
        _PINNED[key] = a
    return a


class Packed:
    """ctypes structs for one call plus the arrays they point into."""

    def __init__(self, profile, users: Dict, mem: int, want_ip=True, want_og=False,
                 device=None, ip_fields=None, og_fields=None, pinned=False):
        self.pinned = pinned
        self.p = as_profile(profile)
        self.keep = [self.p.work, self.p.data_bits, self.p.latency]
        self.profile = _abi.Profile(self.p.N, self.p.b_max, _ptr(self.p.work, C.c_double),
                                    _ptr(self.p.data_bits, C.c_double),
                                    _ptr(self.p.latency, C.c_double))
        ref = users["deadline"]
        K, M = int(ref.shape[0]), int(ref.shape[1])
        self.K, self.M, self.N = K, M, self.p.N
        ptrs = {}
        for f in _abi.USER_FIELDS:
            a = users.get(f)
            if a is not None:
                if _is_torch(a):
                    a = a.contiguous()
                    assert a.dtype == torch.float64
                else:
                    a = np.ascontiguousarray(a, dtype=np.float64)
                self.keep.append(a)
            ptrs[f] = _ptr(a, C.c_double)
        self.users = _abi.Users(K, M, mem, *[ptrs[f] for f in _abi.USER_FIELDS])
        self.out_ip = self._alloc(_abi.IPSSA_FIELDS, _abi.IpssaOut, ip_fields, mem, device) \
            if want_ip else None
        self.out_og = self._alloc(_abi.OG_FIELDS, _abi.OgOut, og_fields, mem, device) \
            if want_og else None

    def _alloc(self, fields, struct, only, mem, device):
        dims = {"K": self.K, "KM": self.K * self.M, "KN": self.K * self.N,
                "KMN": self.K * self.M * self.N, "KMN1": self.K * self.M * (self.N + 1)}
        shapes = {"K": (self.K,), "KM": (self.K, self.M), "KN": (self.K, self.N),
                  "KMN": (self.K, self.M, self.N), "KMN1": (self.K, self.M, self.N + 1)}
        arrays, ptrs = {}, []
        for name, ctype, dim in fields:
            k = _kind(ctype)
            if only is not None and name not in only:
                ptrs.append(C.cast(None, ctype))
                continue
            if mem == _abi.MEM_DEVICE:
                a = torch.empty(shapes[dim], dtype=getattr(torch, _TT[k]), device=device)
            elif self.pinned:  # page-locked host outputs: D2H at full PCIe speed
                a = _pinned_buffer(struct.__name__, name, shapes[dim], _NP[k])
            else:
                a = np.zeros(shapes[dim], dtype=_NP[k])
            arrays[name] = a
            ptrs.append(_ptr(a, _CT[k]))
            assert dims[dim] >= 0
        s = struct(*ptrs)
        s._arrays = arrays
        return s

    @staticmethod
    def arrays(out) -> Dict:
        return dict(out._arrays) if out is not None else None


class SolverError(RuntimeError):
    pass


class Engine:
    """One CUDA device, one stream, one solver context."""

    def __init__(self, device: int = 0):
        self.lib = _abi.load_library()
        self.device = device
        self.ctx = self.lib.coinfer_ctx_create(device)
        if not self.ctx:
            raise SolverError(f"coinfer: cannot create a context on CUDA device {device}")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.coinfer_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream) -> None:
        """Run on a torch.cuda.Stream (or raw cudaStream_t int); None = own stream."""
        if stream is None:
            self._check(self.lib.coinfer_ctx_reset_stream(self.ctx))
            return
        h = getattr(stream, "cuda_stream", stream)
        self._check(self.lib.coinfer_ctx_set_stream(self.ctx, C.c_void_p(h)))

    def synchronize(self) -> None:
        self._check(self.lib.coinfer_ctx_synchronize(self.ctx))

    def fp64_peak(self) -> float:
        """Measured fp64-pipe throughput of this GPU (instructions x lanes / s)."""
        v = C.c_double()
        self._check(self.lib.coinfer_probe_fp64(self.ctx, C.byref(v)))
        return v.value

    @property
    def launches(self) -> int:
        return int(self.lib.coinfer_ctx_launch_count(self.ctx))

    def _check(self, rc: int) -> None:
        if rc != _abi.OK:
            msg = self.lib.coinfer_last_error(self.ctx).decode()
            if rc in (_abi.E_ARG, _abi.E_PROFILE):
                raise ValueError(msg)
            raise SolverError(f"coinfer error {rc}: {msg}")

    def _mem(self, users) -> int:
        if _is_torch(users["deadline"]):
            # device batches run on torch's current stream, so tensor lifetimes,
            # ordering and torch.cuda.Event timing all follow torch's stream
            s = torch.cuda.current_stream(self.device)
            self.lib.coinfer_ctx_set_stream(self.ctx, C.c_void_p(s.cuda_stream))
            return _abi.MEM_DEVICE
        self.lib.coinfer_ctx_reset_stream(self.ctx)
        return _abi.MEM_HOST

    def _aux(self, x, mem, dtype):
        if x is None:
            return None
        if mem == _abi.MEM_DEVICE:
            return x.contiguous() if _is_torch(x) else torch.as_tensor(
                np.asarray(x), device=f"cuda:{self.device}")
        return np.ascontiguousarray(x, dtype=dtype)

    def ipssa(self, profile, users: Dict, deadline=None, fields=None):
        """IP-SSA for every instance (ip_ssa, offline_solvers.hpp:219-224)."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, True, False, f"cuda:{self.device}", ip_fields=fields)
        d = self._aux(deadline, mem, np.float64)
        self._check(self.lib.coinfer_ipssa_batch(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                                 _ptr(d, C.c_double), C.byref(pk.out_ip)))
        return Packed.arrays(pk.out_ip)

    def fixed(self, profile, users: Dict, b, deadline=None, fields=None):
        """Alg. 1 at bound b (fixed_batch_schedule, offline_solvers.hpp:208-214)."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, True, False, f"cuda:{self.device}", ip_fields=fields)
        d = self._aux(deadline, mem, np.float64)
        bb = self._aux(b, mem, np.int32)
        self._check(self.lib.coinfer_fixed_batch(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                                 _ptr(d, C.c_double), _ptr(bb, C.c_int32),
                                                 C.byref(pk.out_ip)))
        return Packed.arrays(pk.out_ip)

    def og(self, profile, users: Dict, fields=None):
        """OG optimal grouping for every instance (og, offline_solvers.hpp:286-388)."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, False, True, f"cuda:{self.device}", og_fields=fields)
        self._check(self.lib.coinfer_og_batch(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                              C.byref(pk.out_og)))
        return Packed.arrays(pk.out_og)

    def _schedule_out(self, pk, mem):
        return pk._alloc(_abi.SCHEDULE_FIELDS, _abi.ScheduleOut, None, mem, f"cuda:{self.device}")

    @staticmethod
    def _as_struct(struct, fields, arrays):
        ptrs = []
        for name, ctype, _ in fields:
            a = arrays.get(name)
            ptrs.append(C.cast(None, ctype) if a is None else _ptr(a, _CT[_kind(ctype)]))
        return struct(*ptrs)

    def ipssa_schedule(self, profile, users: Dict, solved: Dict, deadline=None):
        """The Schedule of IP-SSA / fixed-bound decisions `solved` (as returned by
        ipssa() / fixed()), built and normalised on the device
        (try_fixed_batch:155-185, normalize)."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, False, False)
        d = self._aux(deadline, mem, np.float64)
        so = self._schedule_out(pk, mem)
        ins = self._as_struct(_abi.IpssaOut, _abi.IPSSA_FIELDS, solved)
        self._check(self.lib.coinfer_ipssa_schedule(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                                    _ptr(d, C.c_double), C.byref(ins), C.byref(so)))
        return Packed.arrays(so)

    def og_schedule(self, profile, users: Dict, solved: Dict):
        """The Schedule of an OG plan (og:357-386 + normalize), on the device."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, False, False)
        so = self._schedule_out(pk, mem)
        ins = self._as_struct(_abi.OgOut, _abi.OG_FIELDS, solved)
        self._check(self.lib.coinfer_og_schedule(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                                 C.byref(ins), C.byref(so)))
        return Packed.arrays(so)

    def baseline(self, profile, users: Dict, mode: str, schedule: bool = True, fields=None):
        """baseline(sc, BaselineMode) for every instance (offline_solvers.hpp:390-612):
        mode in LC / PS / FIFO / IPSSA_NP.  Returns (SolveResult arrays,
        schedule arrays or None)."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, True, False, f"cuda:{self.device}", ip_fields=fields)
        so = self._schedule_out(pk, mem) if schedule else None
        self._check(self.lib.coinfer_baseline_batch(
            self.ctx, C.byref(pk.profile), C.byref(pk.users), _abi.BASELINE_MODES[mode],
            C.byref(pk.out_ip), C.byref(so) if so is not None else None))
        return Packed.arrays(pk.out_ip), (Packed.arrays(so) if so is not None else None)

    def validate(self, profile, users: Dict, sched: Dict, tol: float = 1e-9):
        """validate(schedule, scenario, tol) for every instance (schedule.hpp:139-209):
        status [K], counts [K, 7] per constraint id (_abi.CONSTRAINT_IDS order)
        and the most negative slack [K].  `sched` as returned by *_schedule()
        or baseline()."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, False, False)
        so = self._as_struct(_abi.ScheduleOut, _abi.SCHEDULE_FIELDS, sched)
        K = pk.K
        if mem == _abi.MEM_DEVICE:
            dev = f"cuda:{self.device}"
            st = torch.empty(K, dtype=torch.int32, device=dev)
            cnt = torch.empty((K, _abi.N_CONSTRAINTS), dtype=torch.int32, device=dev)
            sl = torch.empty(K, dtype=torch.float64, device=dev)
        else:
            st = np.zeros(K, np.int32)
            cnt = np.zeros((K, _abi.N_CONSTRAINTS), np.int32)
            sl = np.zeros(K)
        self._check(self.lib.coinfer_validate_batch(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                                    C.byref(so), float(tol), _ptr(st, C.c_int32),
                                                    _ptr(cnt, C.c_int32), _ptr(sl, C.c_double)))
        return dict(status=st, counts=cnt, min_slack=sl)

    def oracle_structured(self, profile, users: Dict, deadline, b):
        """oracle_structured(sc, deadline[k], b[k]) (oracles.hpp:28-93) on the GPU:
        exhaustive over the (N+1)^M split vectors; host memory."""
        pk = Packed(profile, users, _abi.MEM_HOST, False, False)
        K, M = pk.K, pk.M
        d = np.ascontiguousarray(deadline, dtype=np.float64)
        bb = np.ascontiguousarray(b, dtype=np.int32)
        out = dict(status=np.zeros(K, np.int32), energy=np.zeros(K), split=np.zeros((K, M), np.uint8),
                   fallback=np.zeros(K, np.uint8), feasible=np.zeros(K, np.uint8))
        self.lib.coinfer_ctx_reset_stream(self.ctx)
        self._check(self.lib.coinfer_oracle_structured_batch(
            self.ctx, C.byref(pk.profile), C.byref(pk.users), _ptr(d, C.c_double), _ptr(bb, C.c_int32),
            _ptr(out["status"], C.c_int32), _ptr(out["energy"], C.c_double), _ptr(out["split"], C.c_uint8),
            _ptr(out["fallback"], C.c_uint8), _ptr(out["feasible"], C.c_uint8)))
        return out

    def oracle_grouping(self, profile, users: Dict, contiguous: bool = True):
        """oracle_grouping_contiguous / oracle_grouping (oracles.hpp:131-225) on the
        GPU: every cut pattern (M <= 16) or every set partition (M <= 9); host memory."""
        pk = Packed(profile, users, _abi.MEM_HOST, False, False)
        K, M = pk.K, pk.M
        out = dict(status=np.zeros(K, np.int32), energy=np.zeros(K), n_groups=np.zeros(K, np.int32),
                   group_of_user=np.zeros((K, M), np.int32), feasible=np.zeros(K, np.uint8))
        self.lib.coinfer_ctx_reset_stream(self.ctx)
        self._check(self.lib.coinfer_oracle_grouping_batch(
            self.ctx, C.byref(pk.profile), C.byref(pk.users), 1 if contiguous else 0,
            _ptr(out["status"], C.c_int32), _ptr(out["energy"], C.c_double),
            _ptr(out["n_groups"], C.c_int32), _ptr(out["group_of_user"], C.c_int32),
            _ptr(out["feasible"], C.c_uint8)))
        return out

    def sample(self, profile, M: int, seeds, low: float = 0.25, high: float = 1.0,
               device: bool = False, **cfg):
        """sample_scenario (scenario_gen.hpp:113-173) on the GPU, one instance
        per seed (std::mt19937_64(seed)); `cfg` overrides ScenarioConfig
        fields (bandwidth, alpha, shadow_sigma_db, ...).  low == high: fixed
        deadlines.  Returns the SoA user dict (numpy, or CUDA tensors with
        device=True) and per-instance status."""
        c = _abi.SampleCfg()
        self.lib.coinfer_sample_cfg_defaults(C.byref(c))
        for k, v in cfg.items():
            setattr(c, k, float(v))
        c.deadline_uniform = 0 if low == high else 1
        c.deadline_low, c.deadline_high = float(low), float(high)
        p = as_profile(profile)
        pk_prof = _abi.Profile(p.N, p.b_max, _ptr(p.work, C.c_double), _ptr(p.data_bits, C.c_double),
                               _ptr(p.latency, C.c_double))
        K = len(seeds)
        if device:
            dev = f"cuda:{self.device}"
            s = self.lib.coinfer_ctx_set_stream(self.ctx, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))
            sd = torch.as_tensor(np.asarray(seeds, dtype=np.uint64).view(np.int64), device=dev)
            out = {f: torch.empty((K, M), dtype=torch.float64, device=dev) for f in _abi.USER_FIELDS}
            st = torch.empty(K, dtype=torch.int32, device=dev)
            mem = _abi.MEM_DEVICE
        else:
            self.lib.coinfer_ctx_reset_stream(self.ctx)
            sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
            out = {f: np.zeros((K, M)) for f in _abi.USER_FIELDS}
            st = np.zeros(K, np.int32)
            mem = _abi.MEM_HOST
        u = _abi.Users(K, M, mem, *[_ptr(out[f], C.c_double) for f in _abi.USER_FIELDS])
        self._check(self.lib.coinfer_sample_batch(self.ctx, C.byref(pk_prof), C.byref(c),
                                                  _ptr(sd, C.c_uint64), C.byref(u), _ptr(st, C.c_int32)))
        return out, st

    def sub_seed(self, root: int, component: int, index) -> np.ndarray:
        """The CLI's per-instance seeds sub_seed(root, component, k) (coinfer_main.cpp:47-50)."""
        idx = np.atleast_1d(np.asarray(index, dtype=np.uint64))
        return np.array([self.lib.coinfer_sub_seed(root, component, int(i)) for i in idx], dtype=np.uint64)

    def best_partition(self, profile, users: Dict, s=None):
        """best_partition (s: [n, N] start times) or local_only_choice (s None)
        for n single-user queries (users fields of shape (n, 1)); host memory."""
        pk = Packed(profile, users, _abi.MEM_HOST, False, False)
        n = pk.K
        split = np.zeros(n, np.int32)
        freq, energy = np.zeros(n), np.zeros(n)
        feas = np.zeros(n, np.uint8)
        sa = None if s is None else np.ascontiguousarray(s, dtype=np.float64)
        self.lib.coinfer_ctx_reset_stream(self.ctx)
        self._check(self.lib.coinfer_best_partition(
            self.ctx, C.byref(pk.profile), C.byref(pk.users), _ptr(sa, C.c_double),
            _ptr(split, C.c_int32), _ptr(freq, C.c_double), _ptr(energy, C.c_double),
            _ptr(feas, C.c_uint8)))
        return dict(split=split, freq=freq, energy=energy, feasible=feas)

    def sweep(self, profile, users: Dict, ipssa=True, og=True, ip_fields=None, og_fields=None,
              pinned=False):
        """IP-SSA at the smallest deadline and OG, fused, for every instance.

        pinned=True (host batches): outputs land in reusable page-locked
        buffers that the next pinned call overwrites."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, ipssa, og, f"cuda:{self.device}", ip_fields=ip_fields,
                    og_fields=og_fields, pinned=pinned)
        self._check(self.lib.coinfer_sweep_batch(
            self.ctx, C.byref(pk.profile), C.byref(pk.users),
            C.byref(pk.out_ip) if ipssa else None, C.byref(pk.out_og) if og else None))
        return Packed.arrays(pk.out_ip), Packed.arrays(pk.out_og)

    COUNTERS = ["og_chain_steps", "ip_chain_steps", "local_steps", "bstar_steps", "chain_starts",
                "dp_cells", "instances", "bstar_miss_steps"]

    def count_work(self, profile, users: Dict):
        """The fused sweep's executed work units (coinfer_count_work: the
        instrumented solve kernel, same decisions), as a dict of COUNTERS."""
        mem = self._mem(users)
        pk = Packed(profile, users, mem, True, True, f"cuda:{self.device}", ip_fields=["status"],
                    og_fields=["status"])
        c = (C.c_uint64 * 8)()
        self._check(self.lib.coinfer_count_work(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                                C.byref(pk.out_ip), C.byref(pk.out_og), c))
        return dict(zip(self.COUNTERS, [int(x) for x in c]))


@dataclass
class OnlineConfig:
    """ArrivalModel + OnlineEnv + policy settings (online_sim.hpp:26-39,69-91,301-336)."""
    arrival: str = "bernoulli"   # or "immediate"
    p_arrive: float = 0.25
    l_low: float = 0.25
    l_high: float = 1.0
    slot: float = 0.025
    solver: str = "og"           # or "ipssa"
    policy: str = "tw"           # TimeWindowPolicy(window, l_high), or "local"
    window: int = 0
    threshold: Optional[float] = None  # TimeWindowPolicy threshold; None = l_high (the CLI's choice)
    horizon: int = 100_000

    def to_c(self) -> "_abi.OnlineCfg":
        return _abi.OnlineCfg(
            _abi.ARRIVAL_IMMEDIATE if self.arrival == "immediate" else _abi.ARRIVAL_BERNOULLI,
            _abi.SOLVER_OG if self.solver == "og" else _abi.SOLVER_IPSSA,
            _abi.POLICY_LOCAL if self.policy == "local" else _abi.POLICY_TW,
            int(self.window), float(self.p_arrive), float(self.l_low), float(self.l_high),
            float(self.slot), float(self.l_high if self.threshold is None else self.threshold),
            int(self.horizon))


def _online(self, profile, scenarios: Dict, cfg: OnlineConfig, seeds, n_trace: int = 0,
            final_state: bool = False):
    """run_episode for every seed (one GPU warp per episode).  Episode e runs
    scenario e % n_scenarios.  Returns status, totals [E,3] (total_energy,
    total_forced_cost, total_reward), counts [E,6] (forced_count,
    solver_calls, solver_tasks, solver_groups, batches, batched_tasks) and,
    for the first n_trace episodes, per-slot reward/energy/pending/edge_busy/
    action/forced.  final_state: also the OnlineEnv state after the last slot
    ([E, 2M+1]: deadlines, expiries, edge_busy) and the rng outputs consumed."""
    mem = self._mem(scenarios)
    pk = Packed(profile, scenarios, mem, False, False)
    E = int(len(seeds))
    T = int(n_trace) * int(cfg.horizon)
    dev = f"cuda:{self.device}"

    def alloc(shape, np_dtype, t_dtype):
        if mem == _abi.MEM_DEVICE:
            return torch.zeros(shape, dtype=t_dtype, device=dev)
        return np.zeros(shape, dtype=np_dtype)

    if mem == _abi.MEM_DEVICE:
        sd = seeds if _is_torch(seeds) else torch.as_tensor(np.asarray(seeds, dtype=np.uint64).view(np.int64), device=dev)
    else:
        sd = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    out = dict(status=alloc((E,), np.int32, torch.int32 if torch else None),
               totals=alloc((E, 3), np.float64, torch.float64 if torch else None),
               counts=alloc((E, 6), np.int64, torch.int64 if torch else None))
    if T:
        out.update(trace_reward=alloc((n_trace, cfg.horizon), np.float64, torch.float64),
                   trace_energy=alloc((n_trace, cfg.horizon), np.float64, torch.float64),
                   trace_pending=alloc((n_trace, cfg.horizon), np.int32, torch.int32),
                   trace_edge_busy=alloc((n_trace, cfg.horizon), np.float64, torch.float64),
                   trace_action=alloc((n_trace, cfg.horizon), np.int32, torch.int32),
                   trace_forced=alloc((n_trace, cfg.horizon), np.int32, torch.int32))
    if final_state:
        out.update(final_state=alloc((E, 2 * pk.M + 1), np.float64, torch.float64),
                   draws=alloc((E,), np.int64, torch.int64))
    oo = _abi.OnlineOut(_ptr(out["status"], C.c_int32), _ptr(out["totals"], C.c_double),
                        _ptr(out["counts"], C.c_int64), int(n_trace) if T else 0,
                        _ptr(out.get("trace_reward"), C.c_double),
                        _ptr(out.get("trace_energy"), C.c_double),
                        _ptr(out.get("trace_pending"), C.c_int32),
                        _ptr(out.get("trace_edge_busy"), C.c_double),
                        _ptr(out.get("trace_action"), C.c_int32),
                        _ptr(out.get("trace_forced"), C.c_int32),
                        _ptr(out.get("final_state"), C.c_double),
                        _ptr(out.get("draws"), C.c_int64))
    c = cfg.to_c()
    self._check(self.lib.coinfer_online_run(self.ctx, C.byref(pk.profile), C.byref(pk.users),
                                            C.byref(c), _ptr(sd, C.c_uint64), E, C.byref(oo)))
    return out


Engine.online = _online
