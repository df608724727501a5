"""Repeat one SP2 step on a fixed cfg3 iterate; compare the outputs bitwise."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[int(os.environ.get("CFG", "3"))]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(h, cfg.block_size)
x = sp.sp2_init(f, sp.gershgorin_bounds(f))
for _ in range(int(os.environ.get("PRE", "10"))):
    x, _ = sp.sp2_step(x, n_occ, cfg.tau, kernel="exact")
mode = sys.argv[1] if len(sys.argv) > 1 else "step"
ref, bad = None, 0
reps = int(os.environ.get("REPS", "60"))
for rep in range(reps):
    if mode == "step":
        y, br = sp.sp2_step(x, n_occ, cfg.tau)
    else:
        y, st = sp.multiply(x, x, cfg.tau, kernel=os.environ.get("KERNEL", "auto"))
    d = y.blocks_device().clone()
    k = y.keys_device().clone()
    if ref is None:
        ref = (k, d)
        continue
    if not (torch.equal(k, ref[0]) and torch.equal(d, ref[1])):
        bad += 1
print(mode, "bad", bad, "of", reps - 1, flush=True)
