"""Variance probe: repeated X0^2 and an SP2 solve with NVML clocks per multiply."""
import sys, time, numpy as np, torch, pynvml
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import water_cluster, CONFIGS
pynvml.nvmlInit(); hd = pynvml.nvmlDeviceGetHandleByIndex(0)
def clk():
    return pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetCurrentClocksEventReasons(hd), pynvml.nvmlDeviceGetPowerUsage(hd) / 1000
cfg = CONFIGS[4]
h, nocc = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(h, cfg.block_size)
x0 = sp.sp2_init(f, sp.gershgorin_bounds(f))
for rep in range(30):
    c, st = sp.multiply(x0, x0, cfg.tau, timed=True)
    print("rep", rep, "leaf %.3f TF %.2f" % (st.ms_leaf, st.flop_estimate / st.ms_leaf / 1e9), clk(), flush=True)
p, s = sp.sp2_solve(f, nocc, cfg.tau, criterion="fro", timed=True)
for i, st in enumerate(s.product_stats):
    print(i, st.leaf_products, "leaf %.3f TF %.2f" % (st.ms_leaf, st.flop_estimate / max(st.ms_leaf, 1e-9) / 1e9))
# re-run multiplies of the slow-iteration style: take X after k SP2 steps and square repeatedly
x = x0
xs = []
for k in range(12):
    x, br = sp.sp2_step(x, nocc, cfg.tau)
    xs.append(x)
for k in (6, 7, 8, 10):
    for rep in range(5):
        c, st = sp.multiply(xs[k], xs[k], cfg.tau, timed=True)
        print("X%d^2" % (k + 1), rep, "leaf %.3f TF %.2f" % (st.ms_leaf, st.flop_estimate / st.ms_leaf / 1e9), clk(), flush=True)
