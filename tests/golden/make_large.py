"""Generate tests/golden/large.npz: BASELINE config 4 (M = 4096) plans and
large-path reference plans.  Run in the dev container after `make -C oracle`:
    python tests/golden/make_large.py

  c4_heavy   BASELINE C4 itself: one M = 4096 instance, profile_heavy,
             deadlines U[0.25, 1.0], sample_scenario(mt19937_64(sub_seed(1, 1, 0)))
             by the REFERENCE generator (oracle/_ref).  Expected OG plan and
             IP-SSA solve from the C oracle's O(M^3 N) form (the reference's og
             needs ~52 core-days here); that form is pinned to the
             reference cell for cell (tests/test_oracle_golden.py) and to the
             reference's whole plans at M = 256 (ref256_* below).
  c4_light   the same stream with profile_light and deadlines U[0.05, 1.0]:
             80 groups, so the DP's parent chain and the stitch get exercised
             (c4_heavy has 2 groups).
  ref256_heavy / ref256_light
             M = 256 instances solved by the UNMODIFIED reference (oracle/_ref
             og and ip_ssa, ~40 s each): the large path against the reference
             itself, not only against the restatement.

Every array keeps its exact bits (npz, no text round trip)."""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import checkers as ck  # noqa: E402

R = ck.ref()
assert R is not None, "build oracle/_ref first (make -C oracle)"


def put(store, name, prof, users, og, ip):
    store[f"{name}/work"] = prof.work
    store[f"{name}/data_bits"] = prof.data_bits
    store[f"{name}/latency"] = prof.latency
    for k, v in users.items():
        store[f"{name}/users/{k}"] = v
    for k, v in og.items():
        store[f"{name}/og/{k}"] = v
    for k, v in ip.items():
        store[f"{name}/ip/{k}"] = v


def main():
    store = {}
    seed = R.ref_sub_seed(1, 1, 0)
    for name, M, lo, hi, heavy, by_ref in [("c4_heavy", 4096, 0.25, 1.0, True, False),
                                          ("c4_light", 4096, 0.05, 1.0, False, False),
                                          ("ref256_heavy", 256, 0.25, 1.0, True, True),
                                          ("ref256_light", 256, 0.05, 0.2, False, True)]:
        prof, users = ck.ref_sample_scenarios(1, M, lo, hi, [seed], heavy=heavy)
        t = time.time()
        if by_ref:
            og, ip = ck.ref_og(prof, users), ck.ref_ipssa(prof, users)
        else:
            og, ip = ck.oracle_og(prof, users, fast=True), ck.oracle_ipssa(prof, users)
        assert og["status"][0] == 0 and ip["status"][0] == 0, name
        print(name, f"{time.time() - t:.1f} s", "groups", og["n_groups"][0], flush=True)
        put(store, name, prof, users, og, ip)
    path = os.path.join(HERE, "large.npz")
    np.savez_compressed(path, **store)
    print(path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
