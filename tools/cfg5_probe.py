"""Feasibility probe: config 5 (4096 molecules, N=102400, Nb=64) on one B200."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import cluster_sites, device_cluster
from paper_1403_7458_b200.kernel import reserve_memory
t = time.time(); cs = cluster_sites(4096, seed=0); print("sites %.2fs" % (time.time() - t), len(cs.orig), flush=True)
torch.cuda.synchronize(); t = time.time()
h = device_cluster(cs, 64)
torch.cuda.synchronize(); print("device build %.2fs stored %d G %d" % (time.time() - t, h.stored_leaf_count, h.n_blocks), flush=True)
print("free GB", torch.cuda.mem_get_info()[0] / 1e9, flush=True)
for tau in (1e-4, 1e-6, 1e-8, 1e-10):
    st = sp.convolution_census(h, h, tau)
    print("tau", tau, "leaf", st.leaf_products, "frac %.4f" % (st.leaf_products / 1600**3), "census %.3fs" % st.wall_seconds, flush=True)
for tau in (1e-4, 1e-6, 1e-8):
    free = torch.cuda.mem_get_info()[0]
    torch.cuda.synchronize(); t = time.time()
    c, st = sp.multiply(h, h, tau, timed=True)
    torch.cuda.synchronize(); w = time.time() - t
    print("tau", tau, "C blocks", c.stored_leaf_count, "wall %.3fs cull %.1f ms leaf %.1f ms fin %.1f ms" % (w, st.ms_cull, st.ms_leaf, st.ms_finalize),
          "exec TF %.2f" % (st.executed_products * 2 * 64**3 / st.ms_leaf / 1e9), "ref-eq TF %.2f" % (st.flop_estimate / (w * 1e12)), flush=True)
    del c
    torch.cuda.synchronize()
