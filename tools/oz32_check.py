"""K4z at Nb = 32 (leaf_ozaki32.cu): products against the exact kernel and an
extended-precision product, symmetry, and cfg3 SP2 (iterations, time) against
DMMA."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def case(name, da, db, tau):
    a = sp.build_from_dense(da, 32)
    b = a if db is da else sp.build_from_dense(db, 32)
    ce, se = sp.multiply(a, b, tau, kernel="exact")
    co, so = sp.multiply(a, b, tau, kernel="ozaki")
    de, do = sp.to_dense(ce), sp.to_dense(co)
    n = de.shape[0]
    xa = np.zeros((n, n), np.longdouble); xa[:da.shape[0], :da.shape[1]] = da
    xb = np.zeros((n, n), np.longdouble); xb[:db.shape[0], :db.shape[1]] = db
    ex = xa @ xb
    f = lambda c: float(np.linalg.norm((c - ex).astype(np.float64)) / np.linalg.norm(ex.astype(np.float64)))
    print(f"{name}: counts {so.counts_equal(se)} vs exact {rel(do, de):.2e}; vs extended: exact "
          f"{f(de):.2e} ozaki {f(do):.2e}; symmetric {np.array_equal(do, do.T)}", flush=True)


da, db = decay_pair(1024, 0.1, (0, 1))
case("decay A*B", da, db, 0.0)
case("decay A*A", da, da, 0.0)
h, _ = water_cluster(30, seed=0)
case("water30 H*H", h, h, 0.0)
rng = np.random.default_rng(3)
x = rng.uniform(-1, 1, (500, 500)) * np.exp(rng.uniform(-30, 5, (500, 500)))
case("wide", x, x, 0.0)
case("wide sym", x + x.T, x + x.T, 0.0)
cfg = CONFIGS[3]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
res = {}
for kern in ("dmma", "ozaki", "dmma", "ozaki"):
    sp.sp2_solve(f, n_occ, cfg.tau, kernel=kern, criterion="fro", fro_tol=1e-6)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, kernel=kern, criterion="fro", fro_tol=1e-6, timed=True)
    e1.record()
    e1.synchronize()
    res[kern] = (sp.to_dense(p), st)
    print(f"cfg3 {kern}: solve {e0.elapsed_time(e1):.2f} ms K4 {st.ms_leaf:.2f} ms iters {st.iteration}",
          flush=True)
print(f"cfg3 P ozaki vs dmma {rel(res['ozaki'][0], res['dmma'][0]):.2e}, same iterations "
      f"{res['ozaki'][1].iteration == res['dmma'][1].iteration}, same products "
      f"{res['ozaki'][1].leaf_products == res['dmma'][1].leaf_products}")
