"""Bitwise A/B of two builds: sha256 of the K4z products and SP2 densities on
cfg3/cfg4 and a dense decay pair (long task lists: > 128 tasks per C block).
Run once per build (SPAMM_LIB_PATH selects the library) and diff the output.
Usage: [SPAMM_LIB_PATH=...] python tools/ab_bitwise.py"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, decay_pair, water_cluster  # noqa: E402


def digest(m):
    return hashlib.sha256(m.blocks_device().cpu().numpy().tobytes()).hexdigest()[:16]


for c in (3, 4):
    cfg = CONFIGS[c]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    x2, _ = sp.multiply(x, x, cfg.tau, kernel="ozaki")
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, kernel="ozaki", criterion="fro")
    print(f"{cfg.name}: X0^2 {digest(x2)} P {digest(p)} iters {st.iteration}", flush=True)
for nb, n in ((32, 8192), (64, 12288)):  # G = 256 / 192 tasks per C block
    da, db = decay_pair(n, 0.002, (0, 1))
    a, b = sp.build_from_dense(da, nb), sp.build_from_dense(db, nb)
    c, _ = sp.multiply(a, b, 1e-12, kernel="ozaki")
    print(f"decay Nb={nb}: C {digest(c)}", flush=True)
