"""Per-step SP2 timing: timed vs untimed, device events vs wall."""
import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import water_cluster, CONFIGS
cfg = CONFIGS[4]
h, nocc = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
s = torch.cuda.current_stream()
for timed in (False, True, False, True, False):
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); w = time.perf_counter(); e0.record(s)
        p, st = sp.sp2_solve(f, nocc, cfg.tau, criterion="fro", timed=timed)
        e1.record(s); e1.synchronize(); w = time.perf_counter() - w
        comp = sum(x.ms_cull + x.ms_leaf + x.ms_finalize for x in st.product_stats)
        print("timed", timed, "dev %.1f ms wall %.1f ms  sum(cull+leaf+fin) %.1f  leaf %.1f  mults %d" % (e0.elapsed_time(e1), w * 1e3, comp, st.ms_leaf, len(st.product_stats)), flush=True)
