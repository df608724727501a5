import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import __graft_entry__ as g
g.smoke()
import paper_1403_7458_b200 as sp
from oracle import spamm_oracle as O
from paper_1403_7458_b200.synth import water_cluster
rng = np.random.default_rng(3)
for n, nb in [(37, 4), (100, 8), (64, 16), (200, 32), (300, 64), (7, 2), (1, 1), (20, 128)]:
    d = rng.standard_normal((n, n)); d[np.abs(d) < 1.0] = 0
    a = sp.build_from_dense(d, nb); oa = O.from_dense(d, nb)
    ok_n = all(np.array_equal(x, y) for x, y in zip(a._tier_norms, oa.tier_norms))
    ok_rt = np.array_equal(sp.to_dense(a), d)
    for tau in (0.0, 1e-2, 1.0):
        c, st = sp.multiply(a, a, tau); oc, ost, _ = O.multiply(oa, oa, tau)
        ce, _ = sp.multiply(a, a, tau, kernel="exact")
        ref = O.to_dense(oc)
        den = max(np.linalg.norm(ref), 1e-300)
        print(n, nb, tau, ok_n, ok_rt, st.visited == ost["visited"], st.culled == ost["culled"],
              "rel", np.linalg.norm(sp.to_dense(c) - ref) / den, "exact", np.array_equal(sp.to_dense(ce), ref),
              "tr", sp.trace(ce) == O.trace(oc), "stored", c.stored_leaf_count == oc.data.shape[0])
    s1 = sp.add_scaled(0.3, a, -1.7, a); s2 = O.add_scaled(0.3, oa, -1.7, oa)
    print("  add", np.array_equal(sp.to_dense(s1), O.to_dense(s2)))
h, nocc = water_cluster(30, 0)
f = sp.build_from_dense(h, 32); of = O.from_dense(h, 32)
b1 = sp.gershgorin_bounds(f); b2 = O.gershgorin_bounds(of)
print("gersh", (b1.eps_min, b1.eps_max) == b2, b1, b2)
t = time.time(); p, st = sp.sp2_solve(f, nocc, 1e-8, kernel="exact"); print("gpu sp2", time.time() - t, st.iteration)
t = time.time(); r = O.sp2_solve(of, nocc, 1e-8, threads=8); print("cpu sp2", time.time() - t, r.iterations)
print("sp2 bitwise", np.array_equal(sp.to_dense(p), O.to_dense(r.x)), st.branch_history == r.branches)
p2, st2 = sp.sp2_solve(f, nocc, 1e-8)
print("sp2 dmma rel", np.linalg.norm(sp.to_dense(p2) - O.to_dense(r.x)) / np.linalg.norm(O.to_dense(r.x)), st2.iteration)
