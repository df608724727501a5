"""Per-iteration cost of the sharded SP2 driver at world size 1 (one GPU):
the host/driver overhead the multi-GPU path adds on top of the native solve."""
import os, sys, time
import torch
import torch.distributed as dist
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.parallel import DeviceEngine, ShardedSP2
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
drv = ShardedSP2(DeviceEngine())
for _ in range(2):
    drv.solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
t = time.perf_counter()
res = drv.solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
dt = time.perf_counter() - t
t = time.perf_counter()
sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
dn = time.perf_counter() - t
print(f"sharded(world 1) {dt*1e3:.1f} ms ({res.iteration} it)  native {dn*1e3:.1f} ms")
dist.destroy_process_group()
