"""Per-solve cost of the sharded SP2 drivers at world size 1 (one GPU): the
host/driver overhead the multi-GPU paths add on top of the native solve."""
import os, sys, time
import torch
import torch.distributed as dist
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.parallel import DeviceEngine, NativeShardedSP2, ShardedSP2
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)


def timeit(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


print("native           %.1f ms" % timeit(lambda: sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")))
print("NativeShardedSP2 %.1f ms" % timeit(lambda: NativeShardedSP2().solve(f, n_occ, cfg.tau)))
print("ShardedSP2(eng)  %.1f ms" % timeit(lambda: ShardedSP2(DeviceEngine()).solve(f, n_occ, cfg.tau)))
dist.destroy_process_group()
