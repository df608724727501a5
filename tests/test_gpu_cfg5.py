"""BASELINE config 5 at full size (4096 molecules, N=102400 -> 131072, Nb=64,
84 GB of H generated in HBM): the SURVEY 8(c) cfg5 procedure -- the reference
cannot hold the dense matrix, so parity is checked through (i) the leaf
survivor count recomputed independently from the gathered leaf norms (leaf
predicate theorem) and (ii) sampled C blocks recomputed on the
host with the oracle's reference-order leaf kernel."""

import numpy as np
import pytest
import torch

from oracle import spamm_oracle as O

pytestmark = pytest.mark.gpu

import paper_1403_7458_b200 as sp  # noqa: E402
from paper_1403_7458_b200.synth import CONFIGS, cluster_sites, device_cluster  # noqa: E402


def _leaf_norms(x):
    g, d = x.n_blocks, x.depth
    off = ((1 << (2 * d)) - 1) // 3
    return x.norms_device()[off:off + g * g].reshape(g, g)


def test_cfg5_full_size_counts_and_sampled_blocks():
    cfg = CONFIGS[5]
    cs = cluster_sites(cfg.n_mol, seed=0)
    h = device_cluster(cs, cfg.block_size)
    assert h.stored_leaf_count == 1600 * 1600 and h.n_blocks == 2048 and h.symmetric
    tau = 1e-4
    c, st = sp.multiply(h, h, tau)
    assert st.symmetric
    # (i) independent survivor count: #{(i,k,j): fl(n_ik * n_kj) > tau} on the native grid
    L = _leaf_norms(h)[:1600, :1600].contiguous()
    cnt = 0
    for k0 in range(0, 1600, 64):
        a = L[:, k0:k0 + 64]                     # (i, k)
        b = L[k0:k0 + 64, :]                     # (k, j)
        cnt += int((a.T[:, :, None] * b[:, None, :] > tau).sum())
    assert cnt == st.leaf_products
    # (ii) sampled C blocks vs the reference-order leaf kernel on the host
    ce, ste = sp.multiply(h, h, tau, kernel="exact")
    assert ste.counts_equal(st)
    keys = h.keys_device()
    order = torch.argsort(keys)
    skeys = keys[order]
    ck = c.keys_device()
    ck_sorted, ck_order = torch.sort(ck)
    cek = ce.keys_device()
    g = h.n_blocks
    rng = np.random.default_rng(1)
    Lh = L.cpu().numpy()
    blocks_h = h.blocks_device()
    for idx in rng.choice(ck.numel(), size=24, replace=False):
        key = int(ck[idx])
        i, j = divmod(key, g)
        ks = np.flatnonzero(Lh[i, :] * Lh[:, j] > tau)
        assert len(ks) > 0
        ak = torch.as_tensor(i * g + ks, device="cuda")
        bk = torch.as_tensor(ks * g + j, device="cuda")
        apos = order[torch.searchsorted(skeys, ak)]
        bpos = order[torch.searchsorted(skeys, bk)]
        a_blk = blocks_h[apos].cpu().numpy()
        b_blk = blocks_h[bpos].cpu().numpy()
        ref = np.zeros((1, 64, 64))
        t = np.arange(len(ks))
        O.gemm_batch(t, t, np.zeros(len(ks), dtype=np.int64), a_blk, b_blk, ref, threads=4)
        got = c.blocks_device()[idx].cpu().numpy()
        assert np.linalg.norm(got - ref[0]) <= 1e-12 * np.linalg.norm(ref[0])
        pe = int(torch.nonzero(cek == key)[0])
        assert np.array_equal(ce.blocks_device()[pe].cpu().numpy(), ref[0])   # exact kernel: bitwise
