"""Repeat X*X on an SP2 iterate (cfg3) and compare the products bitwise."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(h, cfg.block_size)
x = sp.sp2_init(f, sp.gershgorin_bounds(f))
for _ in range(10):
    x, _ = sp.sp2_step(x, n_occ, cfg.tau, kernel="exact")
ref = None
bad = 0
for rep in range(int(os.environ.get("REPS", "30"))):
    c, st = sp.multiply(x, x, cfg.tau)
    d = c.blocks_device().clone()
    if ref is None:
        ref = d
        keys = c.keys_device().clone()
        continue
    if not torch.equal(d, ref):
        bad += 1
        diff = (d != ref).reshape(d.shape[0], -1).any(dim=1)
        idx = torch.nonzero(diff).flatten()
        print("rep", rep, "blocks differing", idx.numel(), "first keys", keys[idx[:5]].tolist(),
              "max abs", float((d - ref).abs().max()), flush=True)
print(os.environ.get("SPAMM_K4_32", "0"), "bad reps", bad, "of", int(os.environ.get("REPS", "30")) - 1)
