"""SP2 cfg4 step-time distribution (device events, L2 flushed) -- run once per
SPAMM_WAIT mode; also reports cgroup CPU throttling during the run."""
import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import bench
import paper_1403_7458_b200 as sp
cfg, h, n_occ = bench.workload(4)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
flush = torch.empty(bench.L2_FLUSH_BYTES // 8, dtype=torch.float64, device="cuda")
def cg():
    try:
        return {k: int(v) for k, v in (l.split() for l in open("/sys/fs/cgroup/cpu.stat"))}
    except OSError:
        return {}
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
c0 = cg()
out = []
for _ in range(40):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    e1.record()
    e1.synchronize()
    out.append(e0.elapsed_time(e1))
c1 = cg()
a = np.array(out)
print(os.environ.get("SPAMM_WAIT", "block"), f"median {np.median(a):.2f} mean {a.mean():.2f} p90 {np.percentile(a, 90):.2f} max {a.max():.2f}",
      {k: c1[k] - c0[k] for k in c1 if k in c0 and c1[k] != c0[k]}, "cpus", len(os.sched_getaffinity(0)))
