"""Generate tests/golden/online_c5.json: BASELINE config 5 episodes at their
full horizon (10^5 slots) from the UNMODIFIED reference run_episode
(oracle/_ref), for slot-for-slot parity of the GPU online driver.

  heavy: sample_scenario(14 users, profile_heavy, fixed(l_high)) with
         mt19937_64(sub_seed(1, 1, 0)); Bernoulli p = 0.05, deadlines
         U[0.25, 1.0]; OG; slot 0.025 s; TimeWindowPolicy(0, l_high)
         (coinfer_main.cpp:482-573, Table IV)
  light: the same with profile_light, p = 0.25, U[0.05, 0.2]

Episode e is seeded sub_seed(1, 5, e).  The per-slot trace (reward, energy,
pending count, edge-busy time) is stored as one SHA-1 digest per 1,000-slot
block of its exact bytes, plus the episode totals and counts; a mismatch
names the block.  Run in the dev container: python tests/golden/make_online_c5.py"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import checkers as ck  # noqa: E402
from paper_2206_06304_b200.engine import OnlineConfig  # noqa: E402

BLOCK = 1000
HORIZON = 100_000


def block_digests(tr):
    """SHA-1 per BLOCK slots of the four trace arrays' exact bytes."""
    out = []
    H = len(tr["trace_reward"])
    for b0 in range(0, H, BLOCK):
        h = hashlib.sha1()
        for k, dt in (("trace_reward", np.float64), ("trace_energy", np.float64),
                      ("trace_pending", np.int32), ("trace_edge_busy", np.float64)):
            h.update(np.ascontiguousarray(np.asarray(tr[k][b0:b0 + BLOCK], dtype=dt)).tobytes())
        out.append(h.hexdigest())
    return out


def main():
    R = ck.ref()
    assert R is not None, "build oracle/_ref first (make -C oracle)"
    s0 = R.ref_sub_seed(1, 1, 0)
    cases = []
    for name, heavy, l_cfg, p, lo, hi in [("c5_heavy", True, 1.0, 0.05, 0.25, 1.0),
                                          ("c5_light", False, 0.2, 0.25, 0.05, 0.2)]:
        prof, users = ck.ref_sample_scenarios(1, 14, l_cfg, l_cfg, [s0], heavy=heavy)
        cfg = OnlineConfig("bernoulli", p, lo, hi, 0.025, "og", "tw", 0, None, HORIZON)
        for e in range(2):
            seed = int(R.ref_sub_seed(1, 5, e))
            t = time.time()
            r = ck.ref_online(prof, users, cfg, seed, trace=True)
            assert r["rc"] == 0
            print(name, e, f"{time.time() - t:.1f} s", "solver calls", int(r["counts"][1]), flush=True)
            cases.append(dict(name=f"{name}_ep{e}",
                              profile=dict(work=prof.work.tolist(), data_bits=prof.data_bits.tolist(),
                                           latency=prof.latency.tolist()),
                              users={k: v.tolist() for k, v in users.items()}, cfg=cfg.__dict__, seed=seed,
                              block=BLOCK, digests=block_digests(r), totals=r["totals"].tolist(),
                              counts=r["counts"].tolist()))
    path = os.path.join(HERE, "online_c5.json")
    json.dump(cases, open(path, "w"), separators=(",", ":"))
    print(path, os.path.getsize(path) // 1024, "KiB")


if __name__ == "__main__":
    main()
