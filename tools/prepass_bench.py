"""Per-kernel device time of K4z's operand pre-passes (and K4z) over repeated
cfg4 H*H products, pre-passes on the caller's stream (SPAMM_OZ_SIDE=0 is set
here) so no other kernel overlaps them.  torch.profiler / CUPTI."""
import collections, json, os, sys
os.environ["SPAMM_OZ_SIDE"] = "0"
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_7458_b200 as sp
from paper_1403_7458_b200.synth import CONFIGS, water_cluster
cfg = CONFIGS[4]
h, _ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(3):
    sp.multiply(f, f, cfg.tau, kernel="ozaki")
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile
N = 20
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(N):
        sp.multiply(f, f, cfg.tau, kernel="ozaki")
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace_pre.json")
ev = json.load(open("/tmp/trace_pre.json"))["traceEvents"]
agg = collections.defaultdict(float)
for e in ev:
    if e.get("cat") == "kernel" and "oz" in e["name"]:
        agg[e["name"].replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")[:40]] += e["dur"]
for k, v in sorted(agg.items(), key=lambda t: -t[1]):
    print(f"{v / N:8.1f} us  {k}")
