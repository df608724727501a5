"""Does NVML sampling (and at what period) perturb the SP2 step time?"""
import sys, time, numpy as np, torch, threading
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import water_cluster, CONFIGS
from bench import ClockSampler
cfg = CONFIGS[4]
h, nocc = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
s = torch.cuda.current_stream()
flush = torch.empty((512 << 20) // 8, dtype=torch.float64, device="cuda")
def run(tag, n=3, do_flush=False):
    for rep in range(n):
        if do_flush: flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        p, st = sp.sp2_solve(f, nocc, cfg.tau, criterion="fro", timed=True)
        e1.record(s); e1.synchronize()
        print(tag, "dev %.1f ms" % e0.elapsed_time(e1), flush=True)
run("plain")
run("flush", do_flush=True)
for period in (0.02, 0.1, 0.2):
    cs = ClockSampler(0)
    import bench
    orig = cs._run
    def _run(cs=cs, period=period):
        while not cs._stop.is_set():
            cs.samples.append(cs._nv.nvmlDeviceGetClockInfo(cs._h, cs._nv.NVML_CLOCK_SM))
            cs._nv.nvmlDeviceGetCurrentClocksEventReasons(cs._h)
            cs._stop.wait(period)
    cs._t = threading.Thread(target=_run, daemon=True)
    with cs:
        run("nvml%.2f" % period)
    print(cs.summary())
