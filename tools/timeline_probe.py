"""GPU timeline of one SP2 solve via torch.profiler (CUPTI sees the library's
kernels too): busy time per kernel family and idle gaps between activities."""
import sys, json, collections, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    torch.cuda.synchronize()
prof.export_chrome_trace("/root/repo/gpurun_out/trace.json")
ev = json.load(open("/root/repo/gpurun_out/trace.json"))["traceEvents"]
gpu = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
gpu.sort(key=lambda e: e["ts"])
t0, t1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
busy = collections.defaultdict(float)
cnt = collections.Counter()
for e in gpu:
    name = e["name"].split("(")[0].replace("void ", "").replace("spamm::", "").replace("(anonymous namespace)::", "")[:50]
    busy[name] += e["dur"]; cnt[name] += 1
gaps = []
end = gpu[0]["ts"] + gpu[0]["dur"]
for a, b in zip(gpu, gpu[1:]):
    g = b["ts"] - max(end, a["ts"] + a["dur"])
    end = max(end, a["ts"] + a["dur"])
    if g > 0:
        gaps.append((g, a["name"][:40], b["name"][:40]))
tot = t1 - t0
print("span %.1f us, busy %.1f us, idle %.1f us, activities %d" % (tot, sum(busy.values()), sum(g for g, *_ in gaps), len(gpu)))
for k, v in sorted(busy.items(), key=lambda x: -x[1])[:22]:
    print("%10.1f us  n=%4d  %s" % (v, cnt[k], k))
pairs = collections.defaultdict(lambda: [0, 0.0])
for g, a, b in gaps:
    key = (a.split("(")[0][-30:], b.split("(")[0][-30:])
    pairs[key][0] += 1; pairs[key][1] += g
print("largest idle-gap transitions (count, total us):")
for k, v in sorted(pairs.items(), key=lambda x: -x[1][1])[:15]:
    print("%8.1f us n=%3d  %s -> %s" % (v[1], v[0], k[0], k[1]))
