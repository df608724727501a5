"""A short program for ncu captures: two cfg4 SP2 solves (the first warms
the pools and caches).  The 37 multiplies of a solve launch K4z 37 times, so
`-k regex:k_leaf_ozaki -s 40 -c 1` profiles iteration 3 of the second solve.
Usage: python tools/ncu_solve.py [config]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, water_cluster  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(2):
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
print(f"ncu_solve: {cfg.name} iterations {st.iteration}", flush=True)
