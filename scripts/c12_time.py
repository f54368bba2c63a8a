"""C1 (IP-SSA, M=10) and C2 (OG, M=100) single-instance device time per
C-ABI call (CUDA events, best-of median): python scripts/c12_time.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch, _abi
from paper_2206_06304_b200.engine import Packed
eng = Engine(0)
eng.set_stream(torch.cuda.current_stream())  # events below are on torch's stream
res = []
for name, M, lo, hi, mode in [("C1", 10, 0.25, 0.25, "ipssa"), ("C2", 100, 0.25, 1.0, "og")]:
    prof = profile_heavy(M)
    dev = {k: torch.as_tensor(v, device="cuda") for k, v in sample_batch(1, M, prof, lo, hi, seed=7).items()}
    pk = Packed(prof, dev, _abi.MEM_DEVICE, mode == "ipssa", mode != "ipssa", "cuda:0")
    if mode == "ipssa":
        call = lambda: eng.lib.coinfer_ipssa_batch(eng.ctx, ctypes.byref(pk.profile), ctypes.byref(pk.users), None,
                                                   ctypes.byref(pk.out_ip))
    else:
        call = lambda: eng.lib.coinfer_og_batch(eng.ctx, ctypes.byref(pk.profile), ctypes.byref(pk.users),
                                                ctypes.byref(pk.out_og))
    for _ in range(20):
        rc = call()
        assert rc == 0, (name, rc, eng.lib.coinfer_last_error(eng.ctx) if hasattr(eng.lib, 'coinfer_last_error') else '')
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(200): call()
    e.record(); torch.cuda.synchronize()
    res.append(f"{name} {s.elapsed_time(e) / 200 * 1e3:.1f} us")
print(f"WIDE={os.environ.get('COINFER_WIDE', 'default')}: " + ", ".join(res))
