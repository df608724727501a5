"""Why does the pipelined e2e cost more than device solves?  (a) fresh matrix
per solve (device-resident H), (b) device solves under concurrent H2D / D2H
traffic on a copy stream."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
h_pin = torch.from_numpy(h).pin_memory()
o_pin = torch.empty_like(h_pin).pin_memory()
hd = torch.from_numpy(h).cuda()
hd2 = hd.clone()
f = sp.build_from_dense(hd, cfg.block_size)
kw = dict(criterion="fro")
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, **kw)
s = torch.cuda.current_stream()
cs = torch.cuda.Stream()
K = 6


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / K


def same():
    for _ in range(K):
        sp.sp2_solve(f, n_occ, cfg.tau, **kw)


def fresh():
    for _ in range(K):
        ff = sp.build_from_dense(hd, cfg.block_size)
        sp.sp2_solve(ff, n_occ, cfg.tau, **kw)


def traffic(kind):
    def run():
        with torch.cuda.stream(cs):
            for _ in range(K * 12):
                if kind in ("h2d", "both"):
                    hd2.copy_(h_pin, non_blocking=True)
                if kind in ("d2h", "both"):
                    o_pin.copy_(hd2, non_blocking=True)
        same()
        s.wait_stream(cs)
    return run


print(f"same f      {timed(same):.2f} ms/solve")
print(f"fresh f     {timed(fresh):.2f} ms/solve")
for k in ("h2d", "d2h", "both"):
    print(f"same f + {k:4s} traffic {timed(traffic(k)):.2f} ms/solve (traffic may outlast)")
