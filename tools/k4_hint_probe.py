"""A/B of the K4 L2 cache-policy bits (SPAMM_K4_HINT, read once per process):
cfg4 SP2 solve time and K4 TF/s.  Usage: SPAMM_K4_HINT=n python tools/k4_hint_probe.py"""
import os
import sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
flush = torch.empty(512 << 17, dtype=torch.float64, device="cuda")
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", timed=True)
s = torch.cuda.current_stream()
tot = leaf = 0.0
xf = 0
for _ in range(6):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", timed=True)
    e1.record(s)
    e1.synchronize()
    tot += e0.elapsed_time(e1)
    leaf += st.ms_leaf
    xf += st.executed_flops
print(f"hint={os.environ.get('SPAMM_K4_HINT', '0')} cfg{sys.argv[1] if len(sys.argv) > 1 else 4}: "
      f"{tot / 6:.2f} ms/solve  K4 {xf / (leaf * 1e-3) / 1e12:.2f} TF/s")
