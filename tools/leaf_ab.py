"""A/B the leaf kernels on cfg3 (Nb=32) and cfg4 (Nb=64) X0^2; checks results agree."""
import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import water_cluster, CONFIGS
for ci in (4, 3):
    cfg = CONFIGS[ci]
    h, nocc = water_cluster(cfg.n_mol, 0)
    f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
    x0 = sp.sp2_init(f, sp.gershgorin_bounds(f))
    ref = None
    for kern in ("dmma", "dmma_cpasync", "exact"):
        ts = []
        for rep in range(6):
            c, st = sp.multiply(x0, x0, cfg.tau, kernel=kern, timed=True)
            ts.append(st.ms_leaf)
        d = sp.to_dense_device(c)
        if ref is None: ref = d
        err = (torch.linalg.norm(d - ref) / torch.linalg.norm(ref)).item()
        best = min(ts[2:])
        print(cfg.name, kern, "leaf ms", ["%.3f" % t for t in ts], "TF %.2f" % (st.flop_estimate / best / 1e9), "rel-vs-first %.2e" % err, flush=True)
