"""Phase timestamps (globaltimer) of the last k_finalize_small launch of a cfg4
SP2 solve (needs the FS_PROBE build of norms.cu)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200 import _native as nat
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
lib = nat.load()
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    lib.spamm_debug_fs_prof(buf)
    t = np.array(buf[:9], dtype=np.int64)
    print("phase us:", np.round(np.diff(t) / 1e3, 2).tolist(), "total", (t[8] - t[0]) / 1e3)
