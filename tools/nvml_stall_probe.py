"""Does NVML polling (bench.py's ClockSampler) perturb SP2 step times?
Runs cfg4 solves with and without the sampler thread and prints step times."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1403_7458_b200 as sp  # noqa: E402

cfg, h, n_occ = bench.workload(4)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
flush = torch.empty(bench.L2_FLUSH_BYTES // 8, dtype=torch.float64, device="cuda")


def run(n):
    out = []
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6)
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return np.array(out)


run(3)
for rep in range(2):
    a = run(15)
    with bench.ClockSampler(0):
        b = run(15)
    print(f"no-sampler  median {np.median(a):.2f} max {a.max():.2f} :", np.round(a, 1).tolist())
    print(f"sampler     median {np.median(b):.2f} max {b.max():.2f} :", np.round(b, 1).tolist())
