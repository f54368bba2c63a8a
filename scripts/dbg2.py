import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import checkers as ck
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
prof, users = ck.two_stage(1)
r = eng.ipssa(prof, users, [0.1]); print("ipssa two_stage:", r["status"], r["energy"], r["split"])
r = eng.og(prof, users); print("og two_stage:", r["status"], r["energy"])
p = profile_heavy(50); u = sample_batch(4, 50, p, seed=3)
ip, og = eng.sweep(p, u); print("sweep:", ip["energy"], og["energy"])
print("oracle:", ck.oracle_ipssa(p, u)["energy"], ck.oracle_og(p, u)["energy"])
