import sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np, torch
import checkers as ck, json
from paper_2206_06304_b200 import Engine
from paper_2206_06304_b200.engine import OnlineConfig, ProfileArrays
eng = Engine(0)
prof, users = ck.two_stage(1)
G = json.load(open("tests/golden/online.json"))
c = next(c for c in G if c["name"] == "accounting_og_tw1")
p = c["profile"]; P = ProfileArrays(np.array(p["work"]), np.array(p["data_bits"]), np.array(p["latency"]))
U = {k: np.array(v) for k, v in c["users"].items()}
ok = OnlineConfig(**c["cfg"])
print("online ok:", eng.online(P, U, ok, [1])["status"], "launches", eng.launches)
r = eng.ipssa(prof, users, [0.1]); print("after online ok:", r["status"], r["energy"], "launches", eng.launches)
r = eng.ipssa(prof, users, [0.1]); print("again:", r["status"], r["energy"], "launches", eng.launches)
dev = {k: torch.as_tensor(v, device="cuda") for k, v in users.items()}
r = eng.ipssa(prof, dev, torch.tensor([0.1], device="cuda")); torch.cuda.synchronize(); print("device:", r["status"], r["energy"])
e2 = Engine(0)
r = e2.ipssa(prof, users, [0.1]); print("fresh engine:", r["status"], r["energy"])
print("cuda err:", torch.cuda.synchronize())
