"""Driver for an ncu capture of the Nb=32 K4 (cfg3 SP2)."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[3]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
