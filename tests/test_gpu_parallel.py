"""Device side of the multi-GPU paths on one GPU: range multiplies (the
dense cull over a Morton range, spamm_multiply_range) must tile the full
product exactly, their work vectors balance the next cut, and the
distributed-operand pieces (ShardedMultiply, config 5) reproduce the
single-GPU product bitwise -- with the K4z row scales all-reduced."""

import numpy as np
import pytest
import torch

from conftest import pyramid_flat

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.dist import DeviceShardEngine, owners  # noqa: E402
from paper_1403_7458_b200.parallel import DeviceEngine, even_cuts, partition_work  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, water_cluster  # noqa: E402


@pytest.mark.parametrize("symmetric", [True, False])
@pytest.mark.parametrize("nb", [16, 64])
def test_range_products_tile_the_full_product(rng, symmetric, nb):
    n = 300 if nb == 16 else 1000
    d = rng.standard_normal((n, n)) * np.exp(-0.02 * np.abs(np.subtract.outer(np.arange(n),
                                                                              np.arange(n))))
    if symmetric:
        d = np.triu(d) + np.triu(d, 1).T
    x = sp.build_from_dense(d, nb)
    assert x.symmetric == symmetric
    tau = 1e-3
    full, st = sp.multiply(x, x, tau)
    eng = DeviceShardEngine()
    g = x.n_blocks
    mode = "upper" if symmetric else "pos"
    for world in (1, 3, 5):
        keys, blocks, leaf, execd = [], [], 0, 0
        work_tot = torch.zeros(g * g, dtype=torch.int64, device="cuda")
        cuts = even_cuts(g * g, world)
        for r in range(world):
            c, w, n_full, n_exec = eng.multiply_range(x, tau, cuts[r], cuts[r + 1], symmetric)
            k = c.keys_device().clone()
            assert bool((owners(k, g, cuts, mode) == r).all())    # exactly the owned blocks
            keys.append(k)
            blocks.append(c.blocks_device().clone())
            work_tot += w.to(torch.int64)
            leaf += n_full
            execd += n_exec
        keys = torch.cat(keys)
        assert keys.numel() == torch.unique(keys).numel()            # no block twice
        c = eng.assemble(x, keys, torch.cat(blocks))
        assert np.array_equal(sp.to_dense(c), sp.to_dense(full))
        assert np.array_equal(pyramid_flat(c._tier_norms), pyramid_flat(full._tier_norms))
        assert leaf == st.leaf_products and execd == st.executed_products
        assert int(work_tot.sum()) == st.executed_products


def test_persistence_cuts_balance_cfg4_work():
    """Cuts from one iteration's measured task counts balance the next one."""
    cfg = CONFIGS[4]
    h, _ = water_cluster(cfg.n_mol, seed=0)
    f = sp.build_from_dense(h, cfg.block_size)
    x = sp.sp2_init(f, sp.gershgorin_bounds(f))
    eng = DeviceShardEngine()
    g = x.n_blocks
    _, work, _, n_exec = eng.multiply_range(x, cfg.tau, 0, g * g, True)
    w = work.cpu().numpy()
    for world in (2, 4, 8):
        cuts = partition_work(w, world)
        parts = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
        assert max(parts) / (n_exec / world) < 1.05, parts


# -- distributed operand (ShardedMultiply) device pieces -----------------------

def _shard_run(full, shards, tau, sym, leaf=None):
    """Drive DeviceEngine's shard methods for every shard in turn (one
    process; the exchange is a direct gather from the owner's shard).
    ``leaf``: the global leaf tier, if the shards already hold it."""
    import torch
    from paper_1403_7458_b200.parallel import DeviceEngine, morton_positions, partition_work
    eng = DeviceEngine()
    g = full.n_blocks
    if leaf is None:
        leaf = sum(eng.leaf_norms2(s) for s in shards)
    for s in shards:
        eng.set_pyramid(s, leaf, sym)
    ex = None
    if eng.oz_exponents(shards[0]) is not None:     # K4z: the whole matrix's row scales
        exs = [eng.oz_exponents(s) for s in shards]
        ex = tuple(torch.stack([e[i] for e in exs]).max(0).values for i in range(2))
    work, sym_ok = eng.census_work(shards[0], tau)
    cuts = partition_work(eng.to_numpy(work), len(shards))
    if sym and not sym_ok:           # a mirror ulp tie somewhere: every shard runs the full path
        sym = False
        for s in shards:
            eng.set_pyramid(s, leaf, False)
    out_k, out_b, leaf_total = [], [], 0
    for r, s in enumerate(shards):
        need = eng.needed_keys(s, tau, cuts[r], cuts[r + 1])
        own = torch.isin(need, s.keys_device())
        halo = need[~own]
        blocks = []
        for o in shards:                 # fetch each halo block from its owner
            hit = torch.isin(halo, o.keys_device())
            if bool(hit.any()):
                blocks.append((halo[hit], eng.gather(o, halo[hit])))
        hk = torch.cat([k for k, _ in blocks]) if blocks else halo
        nb = full.block_size
        hb = torch.cat([b for _, b in blocks]) if blocks else torch.empty((0, nb, nb),
                                                                          dtype=torch.float64,
                                                                          device="cuda")
        assert hk.numel() == halo.numel()
        ext = eng.extend(s, hk, hb, leaf, sym)
        if ex is not None:
            eng.install_exponents(ext, *ex)
        c, lp, _ = eng.multiply_range(ext, tau, cuts[r], cuts[r + 1])
        out_k.append(c.keys_device().clone())
        out_b.append(c.blocks_device().clone())
        leaf_total += lp
    return torch.cat(out_k), torch.cat(out_b), leaf_total


@pytest.mark.parametrize("nshards,nb", [(2, 16), (3, 16), (3, 64)])
def test_distributed_operand_shards_reproduce_product(nshards, nb):
    """nb = 64 runs K4z: bitwise only because the shards' row scales are
    the whole matrix's (the halo alone would give other exponents)."""
    import torch
    from paper_1403_7458_b200.parallel import even_cuts, morton_positions
    from paper_1403_7458_b200.synth import water_cluster
    h, _ = water_cluster(20 if nb == 16 else 60, seed=6)
    full = sp.build_from_dense(h, nb)
    assert full.symmetric
    tau = 1e-6
    ref, st = sp.multiply(full, full, tau)
    g = full.n_blocks
    keys, blocks = full.keys_device(), full.blocks_device()
    mk = morton_positions(keys, g)
    own_cuts = even_cuts(g * g, nshards)
    shards = []
    for r in range(nshards):
        m = (mk >= own_cuts[r]) & (mk < own_cuts[r + 1])
        shards.append(sp.QuadTreeMatrix.from_blocks(full.n_native, nb, full.chunk_size,
                                                    keys[m], blocks[m], full.depth))
    ck, cb, lp = _shard_run(full, shards, tau, True)
    assert lp == st.leaf_products
    order = torch.argsort(ck)
    rk = ref.keys_device()
    rorder = torch.argsort(rk)
    assert torch.equal(ck[order], rk[rorder])
    assert torch.equal(cb[order], ref.blocks_device()[rorder])    # bitwise: same K4 per block


def test_cluster_shards_match_whole_matrix():
    import torch
    from paper_1403_7458_b200.parallel import even_cuts
    from paper_1403_7458_b200.synth import cluster_sites, device_cluster
    cs = cluster_sites(64, seed=3)
    whole = device_cluster(cs, 16)
    g = whole.n_blocks
    cuts = even_cuts(g * g, 3)
    shards = [device_cluster(cs, 16, shard=(cuts[r], cuts[r + 1])) for r in range(3)]
    assert sum(s.stored_leaf_count for s in shards) == whole.stored_leaf_count
    assert not any(s.symmetric for s in shards)           # until the global pyramid is set
    k = torch.cat([s.keys_device() for s in shards])
    b = torch.cat([s.blocks_device() for s in shards])
    wk = whole.keys_device()
    assert torch.equal(k, wk) and torch.equal(b, whole.blocks_device())   # Morton order kept
    leaf = sum(s.leaf_norms2_device() for s in shards)
    assert torch.equal(leaf, whole.leaf_norms2_device())
    for s in shards:
        s.set_global_pyramid(leaf, True)
        assert s.symmetric
        assert torch.equal(s.norms_device(), whole.norms_device())
    ck, cb, lp = _shard_run(whole, shards, 1e-5, True, leaf=leaf)
    ref, st = sp.multiply(whole, whole, 1e-5)
    assert lp == st.leaf_products
    o, ro = torch.argsort(ck), torch.argsort(ref.keys_device())
    assert torch.equal(cb[o], ref.blocks_device()[ro])
