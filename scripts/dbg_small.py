import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import checkers as ck
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
M, K = int(sys.argv[1]), int(sys.argv[2])
prof = profile_heavy(M)
u = sample_batch(K, M, prof, 0.25, 1.0, seed=M)
ip = eng.ipssa(prof, u)
print("ipssa done", flush=True)
ck.assert_same_ip(ip, ck.oracle_ipssa(prof, u))
print("ipssa parity ok", flush=True)
og = eng.og(prof, u)
print("og done", flush=True)
ck.assert_same_og(og, ck.oracle_og(prof, u))
print("og parity ok", flush=True)
