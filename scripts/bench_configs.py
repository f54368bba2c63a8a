"""Timings of the non-headline BASELINE configs on one B200:
C1 (IP-SSA, M=10), C2 (OG, M=100, one instance), C4 (OG, M=4096, one
instance) — device-resident inputs, CUDA events, best of 5 after warm-up."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import time
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch, _abi
from paper_2206_06304_b200.engine import Packed
eng = Engine(0)
res = {}
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best
for name, M, K, lo, hi, mode in [("C1", 10, 1, 0.25, 0.25, "ipssa"), ("C2", 100, 1, 0.25, 1.0, "og"),
                                  ("C2x1000", 100, 1000, 0.25, 1.0, "og"), ("C4", 4096, 1, 0.25, 1.0, "og")]:
    prof = profile_heavy(M)
    u = sample_batch(K, M, prof, lo, hi, seed=7)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in u.items()}
    fn = (lambda: eng.ipssa(prof, dev)) if mode == "ipssa" else (lambda: eng.og(prof, dev))
    ms = timeit(fn, 3 if M > 1000 else 5)
    res[name] = {"M": M, "instances": K, "ms": ms, "instances_per_s": K / ms * 1e3}
    # the C-ABI call alone (outputs allocated once, as a C/C++ caller would):
    # launch + completion, host wall clock, best of 50
    pk = Packed(prof, dev, _abi.MEM_DEVICE, mode == "ipssa", mode != "ipssa", "cuda:0")
    call = ((lambda: eng.lib.coinfer_ipssa_batch(eng.ctx, C.byref(pk.profile), C.byref(pk.users), None,
                                                  C.byref(pk.out_ip)))
            if mode == "ipssa" else
            (lambda: eng.lib.coinfer_og_batch(eng.ctx, C.byref(pk.profile), C.byref(pk.users),
                                              C.byref(pk.out_og))))
    lat = []
    for _ in range(3 if M > 1000 else 50):
        t0 = time.perf_counter()
        assert call() == 0
        eng.synchronize()
        lat.append(time.perf_counter() - t0)
    res[name]["abi_call_ms"] = min(lat) * 1e3
    print(name, json.dumps(res[name]), flush=True)
