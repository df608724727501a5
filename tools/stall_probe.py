"""Host stalls: cgroup CPU throttling / scheduling vs SP2 step time."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
def cg():
    try:
        return dict(l.split() for l in open("/sys/fs/cgroup/cpu.stat"))
    except OSError:
        return {}
print("cpu.max", open("/sys/fs/cgroup/cpu.max").read().strip() if os.path.exists("/sys/fs/cgroup/cpu.max") else None)
print("affinity", len(os.sched_getaffinity(0)), "torch threads", torch.get_num_threads())
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), 64)
for i in range(25):
    c0 = cg(); t = time.perf_counter(); r0 = time.process_time()
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t; cpu = time.process_time() - r0; c1 = cg()
    print(i, "wall %.1f ms cpu %.1f ms" % (dt * 1e3, cpu * 1e3), {k: int(c1[k]) - int(c0[k]) for k in c1 if k in c0 and int(c1[k]) != int(c0[k])}, flush=True)
