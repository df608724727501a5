"""Determinism probe: repeated SP2 solves must give identical histories."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
from conftest import golden
cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = CONFIGS[cfg_i]
gd = golden("cfg3_sp2" if cfg_i == 3 else "cfg4_sp2")
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(h, cfg.block_size)
ref = None
for rep in range(8):
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro", fro_tol=1e-6, kernel=sys.argv[2] if len(sys.argv) > 2 else "auto")
    tr = np.array(st.trace_history)
    idem = np.array(st.idempotency_history)
    relg = np.max(np.abs(tr - gd["traces"][: len(tr)]) / np.abs(gd["traces"][: len(tr)])) if len(tr) == len(gd["traces"]) else -1
    if ref is None:
        ref = (tr, idem, sp.to_dense(p))
    same = np.array_equal(tr, ref[0]) and np.array_equal(idem, ref[1]) and np.array_equal(sp.to_dense(p), ref[2])
    first = int(np.argmax(tr != ref[0])) if not np.array_equal(tr, ref[0]) else -1
    print(rep, "iters", st.iteration, "same as rep0", same, "first diff it", first, "max rel vs golden %.2e" % relg, flush=True)
