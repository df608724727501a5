"""Census of the config-5-generator matrix at depth 7: dense cull vs tier walk
vs per-range tier walks (diagnostic for shard counting)."""
import ctypes, sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200 import _native as nat
from paper_1403_7458_b200.parallel import even_cuts
from paper_1403_7458_b200.synth import cluster_sites, device_cluster
cs = cluster_sites(64, seed=3)
w = device_cluster(cs, 16)
g = w.n_blocks
lib = nat.load()
def census_range(m, tau, lo, hi):
    st = nat.Stats()
    work = torch.zeros(g * g, dtype=torch.int32, device="cuda")
    nat.check(lib.spamm_census_range(m._h, m._h, tau, lo, hi, work.data_ptr(), nat.current_stream(), ctypes.byref(st)))
    return st.leaf_products, st.symmetric, int(work.sum())
for tau in (1e-5, 1e-3):
    print("tau", tau, "dense", sp.convolution_census(w, w, tau).leaf_products)
    sp.set_dense_cull(False)
    print("  walk", sp.convolution_census(w, w, tau).leaf_products)
    sp.set_dense_cull(True)
    print("  range full", census_range(w, tau, 0, g * g))
    for n in (2, 3, 4):
        cuts = even_cuts(g * g, n)
        parts = [census_range(w, tau, cuts[r], cuts[r + 1]) for r in range(n)]
        print("  ", n, "shards", parts, "sum", sum(p[0] for p in parts))
    sp.set_symmetric_products(False)
    cuts = even_cuts(g * g, 3)
    parts = [census_range(w, tau, cuts[r], cuts[r + 1]) for r in range(3)]
    print("   nonsym 3 shards", parts, "sum", sum(p[0] for p in parts))
    sp.set_symmetric_products(True)
