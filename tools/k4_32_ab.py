"""Bitwise A/B of the Nb=32 K4 configurations on cfg3's X0^2 (and repeats)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[3]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), 32)
x = sp.sp2_init(f, sp.gershgorin_bounds(f))
outs = []
for rep in range(4):
    c, st = sp.multiply(x, x, cfg.tau)
    outs.append(sp.to_dense(c))
ce, _ = sp.multiply(x, x, cfg.tau, kernel="exact")
e = sp.to_dense(ce)
print(os.environ.get("SPAMM_K4_32", "0"), [np.array_equal(outs[0], o) for o in outs[1:]],
      "rel vs exact %.3e" % (np.linalg.norm(outs[0] - e) / np.linalg.norm(e)),
      "max abs diff among reps %.3e" % max(np.abs(outs[0] - o).max() for o in outs[1:]))
np.save(f"/root/repo/gpurun_out/k4_32_{os.environ.get('SPAMM_K4_32','0')}.npy", outs[0])
