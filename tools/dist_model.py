"""Per-iteration time model of the distributed SP2 (dist.py) at N GPUs, from
one GPU: the census-balanced cut of X0 * X0 under the symmetric ownership,
then per rank the executed leaf products, the owned blocks and the operand
halo its tasks read from other ranks (exact, from the range task lists).

    T(N) = max_r exec_r * t_product            (leaf products, K4z / DMMA rate)
         + max_r halo_r * Nb^2 * 8 B / B_link  (all-to-all of the halo, NVLink 5)
         + t_rest / N + t_collectives          (norms, finalisation, update, syncs)

t_product and t_rest come from the measured single-GPU solve (bench line:
K4 time per executed product; step time minus K4 time); B_link = 700 GB/s per
GPU inbound (NVLink 5 / NVSwitch, 900 GB/s nominal per direction);
t_collectives: 4 all-reduces / all-to-alls of <= 32 MB per iteration, ~60 us.

Usage: python tools/dist_model.py cfg4|cfg5 [tau ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.dist import DeviceShardEngine, UPPER, owners, partition_work  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, cluster_sites, device_cluster, water_cluster  # noqa: E402


def main():
    which = sys.argv[1]
    taus = [float(t) for t in sys.argv[2:]] or [CONFIGS[4 if which == "cfg4" else 5].tau]
    if which == "cfg4":
        cfg = CONFIGS[4]
        h, _ = water_cluster(cfg.n_mol, seed=0)
        f = sp.build_from_dense(h, cfg.block_size)
    else:
        cfg = CONFIGS[5]
        f = device_cluster(cluster_sites(cfg.n_mol, seed=0), cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    del f
    torch.cuda.empty_cache()
    eng = DeviceShardEngine()
    g, nb = x.n_blocks, x.block_size
    keys = x.keys_device()
    rows = []
    for tau in taus:
        work = eng.census_work(x, tau, True)
        w = work.cpu().numpy()
        for world in (1, 2, 4, 8):
            cuts = partition_work(w, world)
            own = owners(keys, g, cuts, UPPER)
            per = []
            for r in range(world):
                ti, tk, tj = eng.tasks(x, tau, cuts[r], cuts[r + 1], True)
                need = torch.unique(torch.cat([ti * g + tk, tk * g + tj, tj * g + tk]))
                pos = torch.searchsorted(torch.sort(keys).values, need)
                order = torch.argsort(keys)
                owner_of = own[order[pos.clamp(max=keys.numel() - 1)]]
                halo = int((owner_of != r).sum())
                per.append({"rank": r, "executed": int(ti.numel()),
                            "owned_blocks": int((own == r).sum()), "halo_blocks": halo,
                            "halo_GB": halo * nb * nb * 8 / 1e9})
                del ti, tk, tj, need
            ex = [p["executed"] for p in per]
            rows.append({"tau": tau, "world": world, "cuts": cuts[1:-1],
                         "executed_max": max(ex), "executed_mean": float(np.mean(ex)),
                         "imbalance": max(ex) / max(np.mean(ex), 1),
                         "halo_GB_max": max(p["halo_GB"] for p in per),
                         "owned_blocks_max": max(p["owned_blocks"] for p in per),
                         "ranks": per})
            print(json.dumps({k: v for k, v in rows[-1].items() if k != "ranks"}), flush=True)
    out = {"workload": cfg.name + "-X0^2", "G": g, "block_size": nb,
           "stored_blocks": int(x.stored_leaf_count), "rows": rows}
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/dist_model_{which}.json", "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
