"""BASELINE config 5 at full size (4096 molecules, N=102400 -> 131072, Nb=64,
2.56 M blocks, 84 GB of H generated in HBM) at all four tau of the sweep --
the SURVEY 8(c) cfg5 procedure.  The reference cannot hold the dense matrix,
so parity is checked piece by piece against the oracle's restatements:

(a) >= 1,024 sampled leaf blocks: their norm^2 recomputed on the host with
    the reference's einsum recipe (oracle.leaf_norms2_recipe), bitwise;
(b) the whole norm pyramid rebuilt by the oracle (pyramid_from_leaf_norms2,
    quadtree.py:188-192) from the gathered leaf tier, bitwise;
(c) per tau, the per-tier visited / culled counters of _sweep
    (kernel.py:96-122) by per-k counting on the oracle's pyramid (a triple
    survives iff its own product passes, since parents' norms dominate:
    SURVEY 0-2) -- tiers 0-9 in numpy on the host, tiers 10-11 with the same
    IEEE product in torch on the device;
(d) per tau, exact leaf task sets for 8 sampled k slices:
    {(i, j) : nA[i,k] nB[k,j] > tau} against the product's own task list;
(e) per tau, >= 1,024 sampled C blocks recomputed from their task lists in
    FP64 (torch, cuBLAS DGEMM; rel-Fro <= 1e-12) and, at tau = 1e-4, 16 of
    them with the oracle's reference-order leaf kernel against the exact
    kernel, bitwise."""

import numpy as np
import pytest
import torch

from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, cluster_sites, device_cluster  # noqa: E402

TAUS = (1e-4, 1e-6, 1e-8, 1e-10)


@pytest.fixture(scope="module")
def h():
    cfg = CONFIGS[5]
    m = device_cluster(cluster_sites(cfg.n_mol, seed=0), cfg.block_size)
    assert m.stored_leaf_count == 1600 * 1600 and m.n_blocks == 2048 and m.symmetric
    return m


@pytest.fixture(scope="module")
def oracle_tiers(h):
    g = h.n_blocks
    leaf2 = h.leaf_norms2_device().cpu().numpy().reshape(g, g)
    return O.pyramid_from_leaf_norms2(leaf2)


def test_cfg5_leaf_norms_and_pyramid_bitwise(h, oracle_tiers):
    g, nb = h.n_blocks, h.block_size
    rng = np.random.default_rng(11)
    pick = torch.as_tensor(np.sort(rng.choice(h.stored_leaf_count, 1024, replace=False)),
                           device="cuda")
    blocks = h.blocks_device()[pick].cpu().numpy()
    keys = h.keys_device()[pick].cpu().numpy()
    leaf2 = h.leaf_norms2_device().cpu().numpy()
    assert np.array_equal(O.leaf_norms2_recipe(blocks), leaf2[keys])          # (a)
    dev = h.norms_device().cpu().numpy()
    assert np.array_equal(dev, np.concatenate([t.ravel() for t in oracle_tiers]))   # (b)
    del nb


def _count_tier(t, tau, tiers):
    """#{(i,k,j) : fl(n[t][i,k] * n[t][k,j]) > tau} (per-k counting)."""
    a = tiers[t]
    w = a.shape[0]
    if t <= 9:
        return int(sum(np.count_nonzero(a[:, k][:, None] * a[k, :][None, :] > tau)
                       for k in range(w)))
    d = torch.as_tensor(a, device="cuda")
    cnt = 0
    for k0 in range(0, w, 64):
        blk = d[:, k0:k0 + 64].T[:, :, None] * d[k0:k0 + 64, :][:, None, :]
        cnt += int((blk > tau).sum())
    return cnt


@pytest.mark.parametrize("tau", TAUS)
def test_cfg5_tau_sweep_parity(h, oracle_tiers, tau):
    g, nb = h.n_blocks, h.block_size
    st = sp.convolution_census(h, h, tau)
    # (c) per-tier counters of the reference sweep
    visited = [_count_tier(t, tau, oracle_tiers) for t in range(len(oracle_tiers))]
    culled = [1 - visited[0]] + [8 * visited[t - 1] - visited[t] for t in range(1, len(visited))]
    assert st.visited == tuple(visited)
    assert st.culled == tuple(culled)
    # (d) exact k slices of the leaf task set
    lib_tasks = [torch.empty(st.leaf_products, dtype=torch.int32, device="cuda")
                 for _ in range(3)]
    import ctypes

    from paper_1403_7458_b200 import _native as nat
    n = ctypes.c_int64()
    nat.check(nat.load().spamm_tasks(h._h, h._h, float(tau), lib_tasks[0].data_ptr(),
                                     lib_tasks[1].data_ptr(), lib_tasks[2].data_ptr(),
                                     st.leaf_products, ctypes.byref(n), nat.current_stream()))
    assert n.value == st.leaf_products
    ti, tk, tj = lib_tasks
    leaf = torch.as_tensor(oracle_tiers[-1], device="cuda")
    rng = np.random.default_rng(int(-np.log10(tau)))
    for k in rng.choice(1600, 8, replace=False).tolist():
        sel = tk == k
        got = torch.sort(ti[sel].to(torch.int64) * g + tj[sel].to(torch.int64)).values
        pred = leaf[:, k][:, None] * leaf[k, :][None, :] > tau
        want = torch.nonzero(pred.reshape(-1)).reshape(-1)
        assert torch.equal(got, want), k
    del ti, tk, tj, lib_tasks, sel, got, pred, want
    torch.cuda.empty_cache()
    # (e) sampled C blocks: FP64 recomputation from the task lists
    c, stm = sp.multiply(h, h, tau)
    assert stm.counts_equal(st)
    ck = c.keys_device()
    n_sample = 1024 if tau in (1e-4, 1e-8) else 256
    pick = torch.as_tensor(np.sort(rng.choice(ck.numel(), n_sample, replace=False)),
                           device="cuda")
    keys = h.keys_device()
    order = torch.argsort(keys)
    skeys = keys[order]
    hb = h.blocks_device()
    cb = c.blocks_device()
    worst = 0.0
    for p in pick.tolist():
        key = int(ck[p])
        i, j = divmod(key, g)
        ks = torch.nonzero(leaf[i, :] * leaf[:, j] > tau).reshape(-1)
        ak = order[torch.searchsorted(skeys, i * g + ks)]
        bk = order[torch.searchsorted(skeys, ks * g + j)]
        ref = torch.bmm(hb[ak], hb[bk]).sum(0)
        err = float(torch.linalg.norm(cb[p] - ref) / torch.linalg.norm(ref))
        worst = max(worst, err)
    assert worst <= 1e-12, worst
    if tau == 1e-4:      # the exact kernel against the reference-order oracle kernel
        del c, cb
        ce, _ = sp.multiply(h, h, tau, kernel="exact")
        cek = ce.keys_device()
        for p in pick[:16].tolist():
            key = int(cek[p])
            i, j = divmod(key, g)
            ks = np.flatnonzero(oracle_tiers[-1][i, :] * oracle_tiers[-1][:, j] > tau)
            ak = order[torch.searchsorted(skeys, torch.as_tensor(i * g + ks, device="cuda"))]
            bk = order[torch.searchsorted(skeys, torch.as_tensor(ks * g + j, device="cuda"))]
            a_blk, b_blk = hb[ak].cpu().numpy(), hb[bk].cpu().numpy()
            ref = np.zeros((1, nb, nb))
            t = np.arange(len(ks))
            O.gemm_batch(t, t, np.zeros(len(ks), dtype=np.int64), a_blk, b_blk, ref, threads=8)
            assert np.array_equal(ce.blocks_device()[p].cpu().numpy(), ref[0])
