"""Where does the non-K4 time of an SP2 iteration go?  Python vs native call time."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200 import _native as nat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), 64)
lib = nat.load()
orig = lib.spamm_sp2_step
acc = {"t": 0.0, "n": 0}
class Wrap:
    def __init__(self, fn): self.fn = fn
    def __call__(self, *a):
        t = time.perf_counter(); r = self.fn(*a); acc["t"] += time.perf_counter() - t; acc["n"] += 1; return r
for rep in range(4):
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
lib.spamm_sp2_step = Wrap(orig)
for rep in range(5):
    acc["t"] = 0; acc["n"] = 0
    torch.cuda.synchronize(); t = time.perf_counter()
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    torch.cuda.synchronize(); w = time.perf_counter() - t
    print("solve %.2f ms, native step calls %d = %.2f ms, rest %.2f ms" % (w * 1e3, acc["n"], acc["t"] * 1e3, (w - acc["t"]) * 1e3), flush=True)
# sync round trip latency
x = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(1000):
    x += 1; x.item()
print("torch tiny kernel + item round trip: %.1f us" % ((time.perf_counter() - t) * 1e3))
