"""Host-side timeline of cfg4 SP2 solves (SPAMM_HTRACE=1 marks in csrc):
mean host time between consecutive marks; the last solve's dump is the
steady-state one."""
import os
import sys

os.environ.setdefault("SPAMM_HTRACE", "1")
import torch

sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(4):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
