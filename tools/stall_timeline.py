"""Where do the sporadic slow SP2 solves lose their time?  Profiles 15 cfg4
solves with torch.profiler (CUPTI), then for the slowest one prints its largest
individual GPU idle gaps and the activities that ran longer than the median
of the same name."""
import sys, json, collections, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
marks = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(15):
        with torch.profiler.record_function(f"solve{i}"):
            sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
            torch.cuda.synchronize()
prof.export_chrome_trace("/root/repo/gpurun_out/trace_stall.json")
ev = json.load(open("/root/repo/gpurun_out/trace_stall.json"))["traceEvents"]
solves = sorted([e for e in ev if str(e.get("name", "")).startswith("solve") and "dur" in e], key=lambda e: e["ts"])
print("solve wall ms:", [round(e["dur"] / 1e3, 1) for e in solves])
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e], key=lambda e: e["ts"])
cpu = [e for e in ev if e.get("cat") in ("cuda_runtime", "cuda_driver") and "dur" in e]
med = collections.defaultdict(list)
for e in gpu:
    med[e["name"]].append(e["dur"])
med = {k: np.median(v) for k, v in med.items()}
for s in sorted(solves, key=lambda e: -e["dur"])[:3]:
    a0, a1 = s["ts"], s["ts"] + s["dur"]
    g = [e for e in gpu if a0 <= e["ts"] <= a1]
    gaps = []
    for x, y in zip(g, g[1:]):
        gap = y["ts"] - (x["ts"] + x["dur"])
        gaps.append((gap, x["name"][:50], y["name"][:50], x["ts"] - a0))
    gaps.sort(key=lambda t: -t[0])
    print(f"\n== {s['name']} {s['dur']/1e3:.1f} ms: {len(g)} GPU activities, busy {sum(e['dur'] for e in g)/1e3:.1f} ms")
    for gap, x, y, t in gaps[:8]:
        print(f"  gap {gap/1e3:7.2f} ms at +{t/1e3:6.1f} ms  {x} -> {y}")
    slow = sorted(((e["dur"] - med[e["name"]], e["dur"], e["name"][:60]) for e in g), reverse=True)[:5]
    for d, dur, n in slow:
        print(f"  slow +{d/1e3:.2f} ms ({dur/1e3:.2f} ms)  {n}")
    c = sorted([e for e in cpu if a0 <= e["ts"] <= a1], key=lambda e: -e["dur"])[:8]
    for e in c:
        print(f"  host {e['name'][:40]:40s} {e['dur']/1e3:7.2f} ms at +{(e['ts']-a0)/1e3:6.1f}")
