"""Device side of the multi-GPU path on one GPU: shard multiplies
(spamm_multiply_range) must tile the full product exactly, and the sharded
SP2 driver with the device engine must reproduce sp2_solve bitwise."""

import numpy as np
import pytest
import torch

from conftest import pyramid_flat

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.parallel import DeviceEngine, ShardedSP2, even_cuts, partition_work  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, water_cluster  # noqa: E402


@pytest.mark.parametrize("symmetric", [True, False])
def test_shards_tile_the_full_product(rng, symmetric):
    n, nb = 300, 16
    d = rng.standard_normal((n, n)) * np.exp(-0.02 * np.abs(np.subtract.outer(np.arange(n),
                                                                              np.arange(n))))
    if symmetric:
        d = np.triu(d) + np.triu(d, 1).T
    x = sp.build_from_dense(d, nb)
    assert x.symmetric == symmetric
    tau = 1e-3
    full, st = sp.multiply(x, x, tau)
    eng = DeviceEngine()
    g = x.n_blocks
    for world in (1, 3, 5):
        keys, blocks, leaf, execd = [], [], 0, 0
        work_tot = torch.zeros(g * g, dtype=torch.int64, device="cuda")
        for r, (lo, hi) in enumerate(zip(even_cuts(g * g, world), even_cuts(g * g, world)[1:])):
            k, b, w, n_exec, n_full = eng.multiply_shard(x, tau, lo, hi)
            keys.append(k)
            blocks.append(b)
            work_tot += w
            leaf += n_full
            execd += n_exec
        keys = torch.cat(keys)
        assert keys.numel() == torch.unique(keys).numel()            # no block twice
        c = eng.assemble(x, keys, torch.cat(blocks))
        assert np.array_equal(sp.to_dense(c), sp.to_dense(full))
        assert np.array_equal(pyramid_flat(c._tier_norms), pyramid_flat(full._tier_norms))
        assert leaf == st.leaf_products and execd == st.executed_products
        assert int(work_tot.sum()) == st.executed_products


def test_device_engine_sharded_solve_world1_matches_sp2_solve():
    cfg = CONFIGS[3]
    h, n_occ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    p, st = sp.sp2_solve(f, n_occ, cfg.tau, criterion="fro")
    res = ShardedSP2(DeviceEngine()).solve(f, n_occ, cfg.tau, criterion="fro")
    assert res.iteration == st.iteration and res.converged
    assert res.trace_history == st.trace_history
    assert res.idempotency_history == st.idempotency_history
    assert np.array_equal(sp.to_dense(res.x), sp.to_dense(p))
    assert res.leaf_products == list(st.leaf_products)


def test_persistence_cuts_balance_cfg4_work():
    """Cuts from one iteration's measured task counts balance the next one."""
    cfg = CONFIGS[4]
    h, _ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    eng = DeviceEngine()
    g = x.n_blocks
    _, _, work, n_exec, _ = eng.multiply_shard(x, cfg.tau, 0, g * g)
    w = work.cpu().numpy()
    for world in (2, 4, 8):
        cuts = partition_work(w, world)
        parts = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
        assert max(parts) / (n_exec / world) < 1.05, parts
