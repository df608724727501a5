import ctypes, sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200 import _native as nat
from paper_1403_7458_b200.parallel import DeviceEngine, even_cuts, partition_work
from paper_1403_7458_b200.synth import cluster_sites, device_cluster
cs = cluster_sites(64, seed=3)
whole = device_cluster(cs, 16)
g = whole.n_blocks
lib = nat.load()
def census_range(m, tau, lo, hi):
    st = nat.Stats()
    nat.check(lib.spamm_census_range(m._h, m._h, tau, lo, hi, None, nat.current_stream(), ctypes.byref(st)))
    return st.leaf_products, st.symmetric
eng = DeviceEngine()
own = even_cuts(g * g, 3)
shards = [device_cluster(cs, 16, shard=(own[r], own[r + 1])) for r in range(3)]
leaf = sum(s.leaf_norms2_device() for s in shards)
for s in shards:
    s.set_global_pyramid(leaf, True)
tau = 1e-5
work, ok = eng.census_work(shards[0], tau)
cuts = partition_work(eng.to_numpy(work), 3)
print("cuts", cuts, "sym_ok", ok, "work sum", int(work.sum()))
for r, s in enumerate(shards):
    lo, hi = cuts[r], cuts[r + 1]
    print("shard", r, "census on shard", census_range(s, tau, lo, hi), "on whole", census_range(whole, tau, lo, hi))
    need = eng.needed_keys(s, tau, lo, hi)
    halo = need[~torch.isin(need, s.keys_device())]
    ks, bs = [], []
    for o in shards:
        hit = torch.isin(halo, o.keys_device())
        if bool(hit.any()):
            ks.append(halo[hit]); bs.append(eng.gather(o, halo[hit]))
    ext = eng.extend(s, torch.cat(ks), torch.cat(bs), leaf, True)
    print("   ext stored", ext.stored_leaf_count, "sym", ext.symmetric, "census ext", census_range(ext, tau, lo, hi),
          "pyr equal", torch.equal(ext.norms_device(), whole.norms_device()))
    c, lp, ex = eng.multiply_range(ext, tau, lo, hi)
    print("   multiply_range lp", lp, "exec", ex, "C blocks", c.stored_leaf_count)
