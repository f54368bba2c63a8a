import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_06304_b200 import Engine, profile_heavy, sample_batch
eng = Engine(0)
M, K = int(sys.argv[1]), int(sys.argv[2])
prof = profile_heavy(M)
u = sample_batch(K, M, prof, 0.25, 1.0, seed=M)
og = eng.og(prof, u)
print("og done", og["status"][:8])
