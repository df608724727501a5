"""e2e pipeline cost split: sp2_solve_many over k problems (k = 1, 2, 5, 10)
vs k device-resident solves, CUDA events on the compute stream."""
import sys
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.pipeline import sp2_solve_many
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
h_pin = torch.from_numpy(h).pin_memory()
outs = [torch.empty_like(h_pin).pin_memory() for _ in range(10)]
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
kw = dict(criterion="fro")
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, **kw)
sp2_solve_many([h_pin] * 2, n_occ, cfg.tau, cfg.block_size, out=outs[:2], **kw)
s = torch.cuda.current_stream()


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    fn()
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1)


def dev(k):
    for _ in range(k):
        sp.sp2_solve(f, n_occ, cfg.tau, **kw)


def single_e2e(k):
    for i in range(k):
        hd = h_pin.to("cuda", non_blocking=True)
        ff = sp.build_from_dense(hd, cfg.block_size)
        p, _ = sp.sp2_solve(ff, n_occ, cfg.tau, **kw)
        outs[i].copy_(sp.to_dense_device(p), non_blocking=True)


for k in (1, 2, 5, 10):
    a = timed(lambda: dev(k))
    b = timed(lambda: sp2_solve_many([h_pin] * k, n_occ, cfg.tau, cfg.block_size, out=outs[:k], **kw))
    c = timed(lambda: single_e2e(k))
    d = timed(lambda: sp2_solve_many([h_pin] * k, n_occ, cfg.tau, cfg.block_size, out=outs[:k],
                                     solver=lambda ff, o: sp.sp2_solve(ff, o, cfg.tau, **kw)))
    print(f"k={k:2d}: device {a / k:7.2f} ms/solve  riding e2e {b / k:7.2f}  "
          f"plain-overlap e2e {d / k:7.2f}  serial e2e {c / k:7.2f}")
h2d = timed(lambda: h_pin.to("cuda", non_blocking=True))
hd = h_pin.to("cuda")
d2h = timed(lambda: outs[0].copy_(hd, non_blocking=True))
bld = timed(lambda: sp.build_from_dense(hd, cfg.block_size))
p, _ = sp.sp2_solve(f, n_occ, cfg.tau, **kw)
td = timed(lambda: sp.to_dense_device(p))
print(f"h2d {h2d:.2f} ms  d2h {d2h:.2f} ms  build {bld:.2f} ms  to_dense {td:.2f} ms")
