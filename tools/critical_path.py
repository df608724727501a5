"""Where the time between two K4z launches goes in cfg4 SP2 solves: for every
iteration, each kernel's start / end relative to the end of the previous K4z
launch, by stream, averaged over iterations of the same shape (the kernel
sequence), plus how long each K4z launch waited after the main stream's last
kernel (exposed side-stream pre-passes).  torch.profiler / CUPTI timeline.
Usage: python tools/critical_path.py [config]"""
import collections
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, water_cluster  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
h, n_occ = water_cluster(cfg.n_mol, 0)
f = sp.build_from_dense(torch.from_numpy(h).cuda(), cfg.block_size)
for _ in range(3):
    sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
        torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace_cp.json")
ev = json.load(open("/tmp/trace_cp.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e],
             key=lambda e: e["ts"])


def short(n):
    n = n.replace("(anonymous namespace)::", "").replace("void ", "").replace("spamm::", "")
    return n.split("(")[0].replace("unnamed>::", "")[:32]


k4 = [i for i, e in enumerate(gpu) if "k_leaf_ozaki" in e["name"] or "k_leaf_dmma" in e["name"]]
main_stream = gpu[k4[0]]["args"].get("stream", gpu[k4[0]].get("tid"))
shapes = collections.defaultdict(list)
waits = []
for a, b in zip(k4, k4[1:]):
    t0 = gpu[a]["ts"] + gpu[a]["dur"]
    seg = gpu[a + 1:b]
    if not seg or gpu[b]["ts"] - t0 > 5000:  # between solves
        continue
    rows = []
    for e in seg:
        st = e["args"].get("stream", e.get("tid"))
        rows.append((short(e["name"]), "main" if st == main_stream else "side",
                     e["ts"] - t0, e["ts"] + e["dur"] - t0))
    main_end = max([r[3] for r in rows if r[1] == "main"], default=0.0)
    side_end = max([r[3] for r in rows if r[1] == "side"], default=0.0)
    k4_start = gpu[b]["ts"] - t0
    waits.append((k4_start, main_end, side_end))
    shapes[tuple((r[0], r[1]) for r in rows)].append(rows)
print(f"{len(waits)} iterations; mean K4z-end -> next K4z start {sum(w[0] for w in waits) / len(waits):.1f} us;"
      f" main stream done at {sum(w[1] for w in waits) / len(waits):.1f}, side at "
      f"{sum(w[2] for w in waits) / len(waits):.1f} us")
print(f"K4z start after the main stream's last kernel: "
      f"{sum(w[0] - w[1] for w in waits) / len(waits):.1f} us mean")
for shape, its in sorted(shapes.items(), key=lambda kv: -len(kv[1]))[:4]:
    print(f"\n-- {len(its)} iterations with this sequence (us from the K4z end):")
    for j, (name, stream) in enumerate(shape):
        s0 = sum(r[j][2] for r in its) / len(its)
        s1 = sum(r[j][3] for r in its) / len(its)
        print(f"  {stream:4s} {name:32s} {s0:7.1f} -> {s1:7.1f}  ({s1 - s0:5.1f})")
