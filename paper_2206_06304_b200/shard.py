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
                "failed_instances", "og_split_checksum"]


def summary_stats(xp, ip: Dict, og: Dict):
    """Per-rank summary of a sweep's results (torch tensors or numpy arrays):
    energy sums over solved instances, group / fallback / failure counts and a
    split checksum.  `xp` is the array module (torch or numpy)."""
    ok = (ip["status"] == 0) & (og["status"] == 0)
    M = og["split"].shape[1]
    if xp.__name__ == "torch":
        w = 1 + xp.arange(M, device=og["split"].device, dtype=xp.float64)
        f64 = lambda a: a.to(xp.float64)  # noqa: E731
        zero = xp.zeros((), dtype=xp.float64, device=og["split"].device)
        stack = xp.stack
    else:
        w = 1 + np.arange(M, dtype=np.float64)
        f64 = lambda a: np.asarray(a, dtype=np.float64)  # noqa: E731
        zero = np.float64(0.0)
        stack = np.stack
    return stack([
        xp.where(ok, f64(ip["energy"]), zero).sum(), xp.where(ok, f64(og["energy"]), zero).sum(),
        f64(og["n_groups"]).sum(), f64(og["fallback"]).sum(), f64(~ok).sum(),
        (f64(og["split"]) * w).sum()])


def reduce_summary(stats, dist=None):
    """All-reduce (sum) the summary vector over ranks; the job's only collective."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(stats)
    return dict(zip(SUMMARY_KEYS, [float(x) for x in stats.tolist()]))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Job time = the slowest rank's device time."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
