import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_1403_7458_b200 as sp
from oracle import spamm_oracle as O
from conftest import golden, pyramid_flat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
gd = golden("cfg4_sp2")
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(h, 64); of = O.from_dense(h, 64)
x = sp.sp2_init(f, sp.gershgorin_bounds(f)); ox = O.sp2_init(of, O.gershgorin_bounds(of))
for it in range(40):
    c, st = sp.multiply(x, x, cfg.tau, kernel="exact")
    oc, ost, _ = O.multiply(ox, ox, cfg.tau, threads=16)
    d, od = sp.to_dense(c), O.to_dense(oc)
    tx, otx = sp.trace(x), O.trace(ox); tq, otq = sp.trace(c), O.trace(oc)
    ok = np.array_equal(d, od)
    print(it, "C", ok, "tr", tx == otx, tq == otq, "visited", st.visited == ost["visited"], "pyr", np.array_equal(pyramid_flat(c._tier_norms), pyramid_flat(oc.tier_norms)), flush=True)
    if not ok:
        idx = np.argwhere(d != od); print(len(idx), idx[:5], d[tuple(idx[0])], od[tuple(idx[0])]); break
    br = abs(tq - n_occ) <= abs(2 * tx - tq - n_occ)
    if br:
        x, ox = c, oc
    else:
        x = sp.add_scaled(2.0, x, -1.0, c); ox = O.add_scaled(2.0, ox, -1.0, oc)
        ed, oed = sp.to_dense(x), O.to_dense(ox)
        if not np.array_equal(ed, oed):
            idx = np.argwhere(ed != oed); print("EXPAND differs", len(idx), idx[:5], ed[tuple(idx[0])], oed[tuple(idx[0])]); break
    if not np.array_equal(pyramid_flat(x._tier_norms), pyramid_flat(ox.tier_norms)):
        print("pyramid of x differs"); 
        for t, (p, q) in enumerate(zip(x._tier_norms, ox.tier_norms)):
            if not np.array_equal(p, q): print(" tier", t, np.argwhere(p != q)[:3])
        break
