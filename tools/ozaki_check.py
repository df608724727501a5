"""K4z (INT8-sliced leaf products) on the GPU: accuracy against the exact
(bitwise-reference) leaf kernel, symmetry, SP2 iteration count and timing
against the DMMA kernel.  Usage: python tools/ozaki_check.py [--quick]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import decay_pair, water_cluster, CONFIGS  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def product_case(name, a, b, tau, da=None, db=None):
    ce, se = sp.multiply(a, b, tau, kernel="exact")
    cd, sd = sp.multiply(a, b, tau, kernel="dmma")
    co, so = sp.multiply(a, b, tau, kernel="ozaki")
    de, dd, do = sp.to_dense(ce), sp.to_dense(cd), sp.to_dense(co)
    sym = np.array_equal(do, do.T)
    print(f"{name}: tasks {so.leaf_products}=={se.leaf_products} "
          f"dmma err {rel(dd, de):.2e} ozaki err {rel(do, de):.2e} "
          f"max|d| {np.abs(do - de).max():.2e} ozaki symmetric {sym}", flush=True)
    if da is not None and tau == 0.0:
        n = de.shape[0]
        xa = np.zeros((n, n), np.longdouble)
        xb = np.zeros((n, n), np.longdouble)
        xa[:da.shape[0], :da.shape[1]] = da
        xb[:db.shape[0], :db.shape[1]] = db
        ex = xa @ xb
        nrm = float(np.linalg.norm(ex.astype(np.float64)))
        f = lambda c: float(np.linalg.norm((c - ex).astype(np.float64))) / nrm
        print(f"    vs extended precision: exact {f(de):.2e} dmma {f(dd):.2e} ozaki {f(do):.2e}")
    return rel(do, de)


def main():
    torch.cuda.set_device(0)
    errs = []
    da, db = decay_pair(1024, 0.1, (0, 1))
    a, b = sp.build_from_dense(da, 64), sp.build_from_dense(db, 64)
    errs.append(product_case("decay A*B 1024", a, b, 1e-8))
    errs.append(product_case("decay A*A 1024", a, a, 1e-8))
    h, n_occ = water_cluster(30, seed=0)
    hh = sp.build_from_dense(h, 64)
    errs.append(product_case("water30 H*H", hh, hh, 1e-8))
    errs.append(product_case("water30 H*H tau0", hh, hh, 0.0, h, h))
    # wide dynamic range inside rows
    rng = np.random.default_rng(3)
    n = 512
    x = rng.uniform(-1, 1, (n, n)) * np.exp(rng.uniform(-30, 5, (n, n)))
    xa = sp.build_from_dense(x, 64)
    xs = sp.build_from_dense(x + x.T, 64)
    errs.append(product_case("wide-range A*A", xa, xa, 0.0, x, x))
    errs.append(product_case("wide-range sym", xs, xs, 0.0, x + x.T, x + x.T))
    if "--quick" in sys.argv:
        print("max err", max(errs))
        return
    cfg = CONFIGS[4]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
    res = {}
    for kern in ("dmma", "ozaki", "dmma", "ozaki"):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p, st = sp.sp2_solve(f, n_occ, cfg.tau, kernel=kern, criterion="fro", fro_tol=1e-6,
                             timed=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        res[kern] = (sp.to_dense(p), st)
        print(f"cfg4 sp2 {kern}: iters {st.iteration} wall {dt * 1e3:.1f} ms "
              f"leaf {st.ms_leaf:.1f} ms executed {st.executed_flops / st.ms_leaf / 1e9:.1f} TF/s "
              f"ref-equiv {st.flops / st.ms_leaf / 1e9:.1f} TF/s", flush=True)
    pd, sd = res["dmma"]
    po, so = res["ozaki"]
    print(f"P rel err ozaki vs dmma {rel(po, pd):.2e}; iterations {so.iteration} vs {sd.iteration}; "
          f"leaf_products equal {so.leaf_products == sd.leaf_products}")
    print("max product err", max(errs))


if __name__ == "__main__":
    main()
