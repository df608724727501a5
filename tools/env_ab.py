"""Interleaved A/B of cfg4 (or cfgN) SP2 solve time under environment settings.
Usage: python tools/env_ab.py CONFIG ROUNDS 'ENV=1 ENV2=x' '' ...
Each setting runs ROUNDS times in its own process (settings interleaved);
prints the median solve ms per setting."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1403_7458_b200 as sp
    from paper_1403_7458_b200.synth import CONFIGS, water_cluster
    cfg = CONFIGS[int(sys.argv[2])]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
    for _ in range(2):
        sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    ts = []
    for _ in range(7):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("RESULT", sorted(ts)[3], st.iteration, flush=True)
    sys.exit(0)

cfgn, rounds, settings = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
res = {s: [] for s in settings}
for _ in range(rounds):
    for s in settings:
        env = dict(os.environ)
        for kv in s.split():
            k, v = kv.split("=", 1)
            env[k] = v
        out = subprocess.run([sys.executable, __file__, "--child", cfgn], env=env,
                             capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("RESULT"):
                res[s].append(float(line.split()[1]))
for s, v in res.items():
    v = sorted(v)
    print(f"{s or '(default)':40s} median {v[len(v)//2]:.3f} ms  all {[round(x, 2) for x in v]}")
