import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import decay_pair, water_cluster
da, db = decay_pair(256, 0.1, (0, 1))
a, b = sp.build_from_dense(da, 64), sp.build_from_dense(db, 64)
c, st = sp.multiply(a, b, 1e-8, kernel="ozaki"); torch.cuda.synchronize(); print("AB ok", flush=True)
c, st = sp.multiply(a, a, 1e-8, kernel="ozaki"); torch.cuda.synchronize(); print("AA ok", flush=True)
h, n_occ = water_cluster(30, seed=0)
x = sp.build_from_dense(h, 64)
c, st = sp.multiply(x, x, 1e-8, kernel="ozaki"); torch.cuda.synchronize(); print("XX ok", flush=True)
p, st = sp.sp2_solve(x, n_occ, 1e-7, kernel="ozaki", criterion="fro"); torch.cuda.synchronize(); print("sp2 ok", st.iteration, flush=True)
