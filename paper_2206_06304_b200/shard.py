"""Instance sharding for multi-GPU sweeps.

Instances are independent (the reference solvers are pure), so a
multi-GPU sweep gives each rank its own contiguous instance range and runs
the solve with no data-path collective.  The only collective is one
all-reduce of a few summary statistics after the solve, and the timing is the
max over ranks.

Weak scaling: every rank owns `per_rank` instances, so the job grows with the
GPU count.  Inputs are drawn per 4096-instance block keyed by the block's
GLOBAL index, so instance k has the same bytes however the job is sharded
(shard invariance is tested).
"""
from __future__ import annotations

from typing import Dict, Tuple

import numpy as np

BLOCK = 4096
USER_FIELDS = ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline"]


def shard_range(per_rank: int, rank: int, world: int) -> Tuple[int, int]:
    """Global instance range [lo, hi) owned by `rank` (weak scaling)."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    return per_rank * rank, per_rank * (rank + 1)


def block_seed(seed: int, block: int) -> int:
    return seed * 1_000_003 + block


def make_instances(profile, M: int, lo: int, hi: int, seed: int = 1, low: float = 0.25,
                   high: float = 1.0) -> Dict[str, np.ndarray]:
    """Instances [lo, hi) of the global stream (sample_scenario distribution)."""
    from .scenarios import sample_batch
    parts = []
    for start in range(lo - lo % BLOCK, hi, BLOCK):
        blk = sample_batch(BLOCK, M, profile, low, high, seed=block_seed(seed, start // BLOCK))
        a, b = max(lo, start) - start, min(hi, start + BLOCK) - start
        parts.append({k: blk[k][a:b] for k in USER_FIELDS})
    if not parts:
        return {k: np.zeros((0, M)) for k in USER_FIELDS}
    return {k: np.ascontiguousarray(np.concatenate([p[k] for p in parts], 0)) for k in USER_FIELDS}


SUMMARY_KEYS = ["ipssa_energy_sum", "og_energy_sum", "og_groups", "og_fallbacks",
                "failed_instances"]
HASH_KEYS = ["decision_hash_sum", "decision_hash_xor"]
# the decisions every instance hashes (the e2e leg's outputs, bench.py)
IP_HASH_FIELDS = ["status", "batch_bound", "energy", "split", "user_energy"]
OG_HASH_FIELDS = ["status", "energy", "n_groups", "group_of_user", "split", "user_energy"]

_FNV = 0x100000001B3
_M1 = -0x40A7B892E31B1A47  # 0xBF58476D1CE4E5B9 as int64
_M2 = -0x6B2FB644ECCEEE15  # 0x94D049BB133111EB as int64


def _as_i64(xp, a):
    """Bits of `a` as int64 (fp64: the IEEE bit pattern; integers: value)."""
    if xp.__name__ == "torch":
        return a.view(xp.int64) if a.dtype == xp.float64 else a.to(xp.int64)
    a = np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a.astype(np.int64)


def _shr(xp, x, s):  # logical right shift of int64
    return (x >> s) & ((1 << (64 - s)) - 1)


def decision_hash(xp, ip: Dict, og: Dict):
    """Per-instance 64-bit hash of the decisions: IP-SSA
    status, bound, energy bits, splits and per-user energy bits; OG status,
    energy bits, group count, group of every user, splits and per-user
    energy bits.  FNV-1a-style mixing over the fields, then the splitmix64
    finaliser; int64 arithmetic wraps identically in numpy and torch.
    Instances a solver did not solve hash only their status (their other
    outputs are not written)."""
    K = ip["status"].shape[0]
    if xp.__name__ == "torch":
        h = xp.full((K,), -0x340D631B7BDDDCDB, dtype=xp.int64, device=ip["status"].device)
    else:
        h = np.full((K,), -0x340D631B7BDDDCDB, dtype=np.int64)
    with np.errstate(over="ignore"):
        for out, fields in ((ip, IP_HASH_FIELDS), (og, OG_HASH_FIELDS)):
            ok = out["status"] == 0
            for f in fields:
                v = _as_i64(xp, out[f])
                cols = [v] if v.ndim == 1 else [v[:, j] for j in range(v.shape[1])]
                for c in cols:
                    c = c if f == "status" else xp.where(ok, c, xp.zeros_like(c))
                    h = (h ^ c) * _FNV
        h = (h ^ _shr(xp, h, 30)) * _M1
        h = (h ^ _shr(xp, h, 27)) * _M2
        h = h ^ _shr(xp, h, 31)
    return h


def _xor_reduce(xp, h):
    """XOR of a 1-D int64 array, as a 0-d array of the same module."""
    if h.shape[0] == 0:
        return h.sum()  # 0
    while h.shape[0] > 1:
        if h.shape[0] & 1:
            h = (xp.cat if xp.__name__ == "torch" else np.concatenate)([h, h[:1] * 0])
        n = h.shape[0] // 2
        h = h[:n] ^ h[n:]
    return h[0]


def summary_stats(xp, ip: Dict, og: Dict):
    """Per-rank summary of a sweep's results (torch tensors or numpy arrays),
    `xp` the array module (torch or numpy): (fp64 vector: energy sums over
    solved instances, group / fallback / failure counts; int64 pair: the
    wrapping sum and the XOR of the per-instance decision hashes)."""
    ok = (ip["status"] == 0) & (og["status"] == 0)
    if xp.__name__ == "torch":
        f64 = lambda a: a.to(xp.float64)  # noqa: E731
        zero = xp.zeros((), dtype=xp.float64, device=og["status"].device)
        stack = xp.stack
    else:
        f64 = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
        zero = np.float64(0.0)
        stack = np.stack
    sol = og["status"] == 0
    stats = stack([
        xp.where(ok, f64(ip["energy"]), zero).sum(), xp.where(ok, f64(og["energy"]), zero).sum(),
        xp.where(sol, f64(og["n_groups"]), zero).sum(), xp.where(sol, f64(og["fallback"]), zero).sum(),
        f64(~ok).sum()])
    h = decision_hash(xp, ip, og)
    with np.errstate(over="ignore"):
        hashes = stack([h.sum(), _xor_reduce(xp, h)])  # int64 sum wraps mod 2^64
    return stats, hashes


def reduce_summary(summary, dist=None):
    """Combine the per-rank summaries over ranks, the job's only collective:
    an all-reduce (sum) of the statistics and an all-gather of the hash pairs
    (sum wraps mod 2^64; XOR, which NCCL does not reduce, is folded here)."""
    stats, hashes = summary
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        import torch
        dist.all_reduce(stats)
        parts = [torch.zeros_like(hashes) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, hashes)
        hs = [p.tolist() for p in parts]
    else:
        hs = [[int(x) for x in (hashes.tolist() if hasattr(hashes, "tolist") else hashes)]]
    hsum, hxor = 0, 0
    for a, b in hs:
        hsum = (hsum + int(a)) & 0xFFFFFFFFFFFFFFFF
        hxor ^= int(b) & 0xFFFFFFFFFFFFFFFF
    out = dict(zip(SUMMARY_KEYS, [float(x) for x in stats.tolist()]))
    out.update(decision_hash_sum=f"{hsum:016x}", decision_hash_xor=f"{hxor:016x}")
    return out


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Job time = the slowest rank's device time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
