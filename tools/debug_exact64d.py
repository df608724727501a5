import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1403_7458_b200 as sp
from conftest import golden, pyramid_flat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
gd = golden("cfg4_sp2"); cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(h, 64)
pe, ste = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6, kernel="exact", max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 100)
t = np.array(ste.trace_history); g = gd["traces"][:len(t)]
print(ste.iteration, np.flatnonzero(t != g)[:10], flush=True)
# same run with a device sync after every library call
from paper_1403_7458_b200 import _native as nat
orig = nat.check
def check_sync(rc):
    torch.cuda.synchronize(); return orig(rc)
nat.check = check_sync
import paper_1403_7458_b200.kernel as K, paper_1403_7458_b200.quadtree as Q, paper_1403_7458_b200.sp2 as S
pe, ste = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6, kernel="exact")
t = np.array(ste.trace_history); g = gd["traces"][:len(t)]
print("synced", ste.iteration, np.flatnonzero(t != g)[:10], flush=True)
import gc
gc.disable()
nat.check = orig
pe, ste = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6, kernel="exact")
t = np.array(ste.trace_history); g = gd["traces"][:len(t)]
print("nogc", ste.iteration, np.flatnonzero(t != g)[:10], flush=True)
