"""Load tests/golden/*.json (made by tests/golden/make_golden.py from the reference)."""
import json
import os

import numpy as np

from paper_2206_06304_b200.engine import ProfileArrays

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_DT = {"status": np.int32, "batch_bound": np.int32, "pipeline_feasible": np.uint8,
       "split": np.uint8, "batch_size": np.int32, "fallback": np.uint8, "n_groups": np.int32,
       "order": np.int32, "group_of_user": np.int32, "group_lo": np.int32,
       "group_size": np.int32, "group_b": np.int32, "group_batch_size": np.int32}


def load(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        cases = json.load(f)
    out = []
    for c in cases:
        p = c["profile"]
        prof = ProfileArrays(np.array(p["work"], dtype=np.float64),
                             np.array(p["data_bits"], dtype=np.float64),
                             np.array(p["latency"], dtype=np.float64))
        users = {k: np.array(v, dtype=np.float64) for k, v in c["users"].items()}
        exp = {k: np.array(v, dtype=_DT.get(k, np.float64)) for k, v in c["expect"].items()}
        dl = None if c["deadline"] is None else np.array(c["deadline"], dtype=np.float64)
        b = None if c["b"] is None else np.array(c["b"], dtype=np.int32)
        out.append(dict(name=c["name"], kind=c["kind"], profile=prof, users=users, deadline=dl,
                        b=b, expect=exp, extra=c["extra"]))
    return out


def all_cases():
    return load("kat") + load("random") + load("cli")


def load_large():
    """tests/golden/large.npz (made by tests/golden/make_large.py): name ->
    dict(profile, users, og, ip) with exact bits."""
    z = np.load(os.path.join(GOLDEN, "large.npz"))
    out = {}
    for key in z.files:
        name, rest = key.split("/", 1)
        d = out.setdefault(name, dict(users={}, og={}, ip={}, p={}))
        if rest.startswith(("users/", "og/", "ip/")):
            kind, field = rest.split("/", 1)
            d[kind][field] = z[key]
        else:
            d["p"][rest] = z[key]
    for d in out.values():
        p = d.pop("p")
        d["profile"] = ProfileArrays(p["work"], p["data_bits"], p["latency"])
    return out
