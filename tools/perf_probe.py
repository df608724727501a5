"""Quick device-timing probe of one config (not the bench; scratch tooling)."""
import sys, time, json, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import water_cluster, CONFIGS
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
t = time.time(); h, nocc = water_cluster(cfg.n_mol, 0); print("gen", time.time() - t, h.shape, flush=True)
f = sp.build_from_dense(h, cfg.block_size)
print("stored", f.stored_leaf_count)
x0 = sp.sp2_init(f, sp.gershgorin_bounds(f))
for kern in ("dmma", "exact"):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.time()
        c, st = sp.multiply(x0, x0, cfg.tau, kernel=kern, timed=True)
        torch.cuda.synchronize(); w = time.time() - t
        print(kern, "T", st.leaf_products, "C", st.c_blocks, "ms cull %.3f leaf %.3f fin %.3f wall %.3f" % (st.ms_cull, st.ms_leaf, st.ms_finalize, w * 1e3),
              "leaf TF %.2f" % (st.flop_estimate / st.ms_leaf / 1e9), flush=True)
for crit in ("trace", "fro"):
    torch.cuda.synchronize(); t = time.time()
    p, s = sp.sp2_solve(f, nocc, cfg.tau, criterion=crit, timed=True)
    torch.cuda.synchronize(); w = time.time() - t
    print(crit, "iters", s.iteration, "wall %.3f s" % w, "flops %.3e" % s.flops, "GF/s %.1f" % (s.flops / w / 1e9),
          "leaf TF %.2f" % (s.flops / s.ms_leaf / 1e9), "per-it ms %.2f" % (w / (s.iteration + 1) * 1e3), flush=True)
for i, st in enumerate(s.product_stats):
    print(i, st.leaf_products, st.c_blocks, "cull %.3f leaf %.3f fin %.3f wall %.3f TF %.2f" % (st.ms_cull, st.ms_leaf, st.ms_finalize, st.wall_seconds * 1e3, st.flop_estimate / max(st.ms_leaf, 1e-9) / 1e9))
