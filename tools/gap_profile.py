"""GPU idle time inside cfg4 SP2 solves, aggregated by (kernel before the gap
-> kernel after the gap): where the host syncs and launch latencies cost.
Usage: python tools/gap_profile.py [config]  (torch.profiler / CUPTI)."""
import collections
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile

NS = 5
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for i in range(NS):
        with torch.profiler.record_function(f"solve{i}"):
            sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
            torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace_gap.json")
ev = json.load(open("/tmp/trace_gap.json"))["traceEvents"]
solves = sorted([e for e in ev if str(e.get("name", "")).startswith("solve") and "dur" in e
                 and e.get("cat") == "user_annotation"],
                key=lambda e: e["ts"])
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e],
             key=lambda e: e["ts"])


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("spamm::", "")
    return n.split("(")[0][:40]


pairs = collections.defaultdict(lambda: [0, 0.0])
busy_by = collections.defaultdict(float)
tot_wall = tot_busy = 0.0
for s in solves:
    a0, a1 = s["ts"], s["ts"] + s["dur"]
    g = [e for e in gpu if a0 <= e["ts"] <= a1]
    tot_wall += (g[-1]["ts"] + g[-1]["dur"] - g[0]["ts"])
    for e in g:
        tot_busy += e["dur"]
        busy_by[short(e["name"])] += e["dur"]
    for x, y in zip(g, g[1:]):
        gap = y["ts"] - (x["ts"] + x["dur"])
        k = (short(x["name"]), short(y["name"]))
        pairs[k][0] += 1
        pairs[k][1] += gap
print(f"per solve: GPU span {tot_wall / NS / 1e3:.2f} ms, busy {tot_busy / NS / 1e3:.2f} ms, "
      f"idle {(tot_wall - tot_busy) / NS / 1e3:.2f} ms")
print("busy by kernel (ms/solve):")
for k, v in sorted(busy_by.items(), key=lambda t: -t[1])[:16]:
    print(f"  {v / NS / 1e3:7.3f}  {k}")
print("idle by transition (ms/solve, count/solve, mean us):")
for k, (n, t) in sorted(pairs.items(), key=lambda t: -t[1][1])[:20]:
    print(f"  {t / NS / 1e3:7.3f} {n / NS:6.1f} {t / n:7.1f}  {k[0]} -> {k[1]}")

# host runtime calls issued inside the largest gap classes (what the host did)
cpu = sorted([e for e in ev if e.get("cat") in ("cuda_runtime", "cuda_driver") and "dur" in e],
             key=lambda e: e["ts"])
top = sorted(pairs.items(), key=lambda t: -t[1][1])[:3]
for (xa, ya), _ in top:
    agg = collections.defaultdict(lambda: [0, 0.0])
    span = nwin = 0
    for s in solves:
        a0, a1 = s["ts"], s["ts"] + s["dur"]
        g = [e for e in gpu if a0 <= e["ts"] <= a1]
        for x, y in zip(g, g[1:]):
            if (short(x["name"]), short(y["name"])) != (xa, ya):
                continue
            w0, w1 = x["ts"] + x["dur"], y["ts"]
            nwin += 1
            span += w1 - w0
            for c in cpu:
                if w0 - 5 <= c["ts"] <= w1:
                    agg[c["name"]][0] += 1
                    agg[c["name"]][1] += c["dur"]
    print(f"\nhost calls in gaps {xa} -> {ya} ({nwin} gaps, mean {span / max(nwin, 1):.1f} us):")
    for k, (n, t) in sorted(agg.items(), key=lambda t: -t[1][1])[:12]:
        print(f"  {n / max(nwin, 1):5.1f} calls/gap {t / max(nwin, 1):7.1f} us/gap  {k}")
