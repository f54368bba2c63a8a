"""bench.py's work models (CPU): the units the launch processes (rlen-truncated
OG rows) against SURVEY.md §8d's count of the reference's units, and the
useful-length rule against the C oracle's DP (a cell past its row's useful
length never has a fitting prev)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2206_06304_b200 import profile_heavy, sample_batch  # noqa: E402


def _sumlat(prof, M):
    sl = np.zeros(M + 1)
    for n in range(prof.N):  # sum_latency, in the reference's order of additions
        sl[1:] = sl[1:] + prof.latency[n][:M]
    return sl


def test_pruned_model_bounded_by_reference_count():
    prof = profile_heavy(50)
    u = sample_batch(300, 50, prof, 0.25, 1.0, seed=3)
    w_og, w_ip = bench.work_model(prof, u)
    w_pr = bench.pruned_work_model(prof, u, chunk=64)
    assert 0 < w_pr < w_og
    # C3-like deadlines: the truncated rows carry well under the full count
    assert 0.25 < (w_pr + w_ip) / (w_og + w_ip) < 0.6


def test_pruned_model_equals_reference_count_when_every_row_is_useful():
    # deadlines so loose that every group fits after every other: rlen(i) = M - i
    prof = profile_heavy(12)
    u = sample_batch(20, 12, prof, 50.0, 60.0, seed=4)
    u["deadline"] = 50.0 + np.random.default_rng(4).permuted(np.tile(np.arange(12.0), (20, 1)), axis=1)
    sl = _sumlat(prof, 12)
    dl = np.sort(u["deadline"], axis=1)
    assert (dl[:, :1] + sl[12] <= dl[:, 1:]).all()
    w_og, _ = bench.work_model(prof, u)
    assert bench.pruned_work_model(prof, u) == w_og


def test_useful_length_matches_feasible_prev_prefix():
    """rlen(i) is exactly the set of sizes whose cell has pfit >= 1
    (offline_solvers.hpp:229-232: groups_fit(dl[prev], dl[i], size))."""
    prof = profile_heavy(40)
    u = sample_batch(50, 40, prof, 0.25, 1.0, seed=5)
    sl = _sumlat(prof, 40)
    for k in range(50):
        dl = np.sort(u["deadline"][k])
        for i in range(1, 40):
            for size in range(1, 40 - i + 1):
                pfit = int(np.sum(dl[:i] + sl[size] <= dl[i]))
                rl = int(np.sum(dl[0] + sl[1:40 - i + 1] <= dl[i]))
                assert (pfit >= 1) == (size <= rl)
