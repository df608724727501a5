"""A/B timing of cfg4 SP2 solves: K4 (DMMA) vs K4z, ms per solve and K4 ms."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, seed=0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
kerns = sys.argv[2].split(",") if len(sys.argv) > 2 else ["dmma", "ozaki"]
for kern in kerns:
    sp.sp2_solve(f, n_occ, cfg.tau, kernel=kern, criterion="fro", fro_tol=1e-6)
    ts, ls = [], []
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p, st = sp.sp2_solve(f, n_occ, cfg.tau, kernel=kern, criterion="fro", fro_tol=1e-6,
                             timed=True)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        ls.append(st.ms_leaf)
    print(f"{cfg.name} {kern}: solve {min(ts):.2f} ms (median {sorted(ts)[2]:.2f}) "
          f"K4 {min(ls):.2f} ms iters {st.iteration} "
          f"executed {st.executed_flops / min(ls) / 1e9:.1f} TF/s", flush=True)
