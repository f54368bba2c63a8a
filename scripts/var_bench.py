"""Time + check development variants (scripts/variants.sh) on the GPU:
    python scripts/var_bench.py build/var_a.so build/var_b.so ...
Each library runs in its own process: parity of the fused sweep against the C
oracle on C3-shaped and other batches, then the C3 sweep (1M instances, M=50,
inputs generated on the device like bench.py), best of 5 launches."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, time
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import checkers as ck
from paper_2206_06304_b200 import Engine, profile_heavy, profile_light, sample_batch, sub_seed
eng = Engine(0)
NOCHECK = bool(os.environ.get("VB_NOCHECK"))  # timing-only experiment builds (CFB_EXP_*)
for M, K, light in ([] if NOCHECK else [(50, 1024, False), (20, 512, False), (14, 256, True), (100, 64, False), (7, 256, False), (33, 256, True), (50, 4096, False), (20, 4096, True), (64, 4096, False), (1, 4096, False), (3, 3000, True), (100, 2048, False), (90, 2100, True)]):
    prof = profile_light(M) if light else profile_heavy(M)
    u = sample_batch(K, M, prof, 0.05 if light else 0.25, 0.2 if light else 1.0, seed=M + 1000)
    ip, og = eng.sweep(prof, u)
    ipx = ck.oracle_ipssa(prof, u)
    ck.assert_same_ip(ip, ipx, where=f"M={M}")
    ck.assert_same_og(og, ck.oracle_og(prof, u), where=f"M={M}")
    ck.assert_same_ip(eng.ipssa(prof, u), ipx, where=f"M={M} ipssa only")
prof = profile_heavy(50)
K = int(os.environ.get("VB_K", "1000000"))
seeds = sub_seed(1, 1, np.arange(K, dtype=np.uint64))
users, st = eng.sample(prof, 50, seeds, 0.25, 1.0, device=True)
dev = {k: users[k] for k in ["f_min", "f_max", "kappa", "rate_up", "power_up", "arrival", "deadline"]}
chk = {k: v[:2000].cpu().numpy() for k, v in dev.items()}
ip, og = eng.sweep(prof, dev)
ipc = {k: v[:2000].cpu().numpy() for k, v in ip.items()}
ogc = {k: v[:2000].cpu().numpy() for k, v in og.items()}
if not NOCHECK:
    ck.assert_same_ip(ipc, ck.oracle_ipssa(prof, chk), where="C3 head")
    ck.assert_same_og(ogc, ck.oracle_og(prof, chk), where="C3 head")
ts = []
for rep in range(5):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); eng.sweep(prof, dev); e.record(); torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
print(f"RESULT {os.path.basename(os.environ['COINFER_LIB'])}: {'unchecked' if NOCHECK else 'parity ok'}; C3 sweep K={K}: best {min(ts):.2f} ms "
      f"median {sorted(ts)[2]:.2f} ms -> {K / min(ts) * 1e3 / 1e6:.3f} M inst/s")
'''.replace("ROOT", repr(ROOT))

for lib in sys.argv[1:]:
    env = dict(os.environ, COINFER_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
    lines = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
    print(lines[0] if lines else f"FAIL {lib}: rc={r.returncode}\n{r.stdout[-1500:]}\n{r.stderr[-2500:]}", flush=True)
