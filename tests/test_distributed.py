"""Multi-GPU host logic (paper_1403_7458_b200/parallel.py) on CPU: gloo,
world size 2, with an oracle-backed engine standing in for the GPUs.
The sharded SP2 must reproduce the single-process trajectory bitwise."""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import spamm_oracle as O
from paper_1403_7458_b200.parallel import ShardedSP2, even_cuts, partition_work
from paper_1403_7458_b200.synth import water_cluster
from paper_1403_7458_b200.synth_morton import morton_decode, morton_keys


class OracleEngine:
    """CPU stand-in for DeviceEngine with the same shard semantics:
    owned = C blocks with Morton position in [lo, hi) (upper triangle only
    when X is symmetric, plus their mirrors)."""

    def grid(self, x):
        return x.n_blocks

    def init_x0(self, f):
        return O.sp2_init(f, O.gershgorin_bounds(f))

    def trace(self, x):
        return O.trace(x)

    def multiply_shard(self, x, tau, lo, hi):
        g, nb = x.n_blocks, x.block_size
        d = O.to_dense(x)
        sym = np.array_equal(d, d.T)
        c, _, (ti, tk, tj) = O.multiply(x, x, tau)
        mt = morton_keys(ti, tj)
        own_t = (mt >= lo) & (mt < hi) & ((ti <= tj) if sym else True)
        work = np.zeros(g * g, dtype=np.int64)
        np.add.at(work, mt[own_t], 1)
        n_exec = int(own_t.sum())
        n_full = 2 * n_exec - int((own_t & (ti == tj)).sum()) if sym else n_exec
        ci, cj = c.keys // g, c.keys % g
        mc = morton_keys(ci, cj)
        own_c = (mc >= lo) & (mc < hi) & ((ci <= cj) if sym else True)
        keys = [c.keys[own_c]]
        blocks = [c.data[own_c]]
        if sym:
            mir = own_c & (ci != cj)
            mkeys = cj[mir] * g + ci[mir]
            pos = np.searchsorted(c.keys, mkeys)
            keys.append(c.keys[pos])
            blocks.append(c.data[pos])
        keys = np.concatenate(keys).astype(np.int64)
        blocks = np.concatenate(blocks).reshape(-1, nb, nb)
        return (torch.from_numpy(keys), torch.from_numpy(np.ascontiguousarray(blocks)),
                torch.from_numpy(work), n_exec, n_full)

    def assemble(self, x, keys, blocks):
        keys = keys.numpy()
        order = np.argsort(keys)
        return O.from_blocks(x.n_native, x.block_size, x.chunk_size, keys[order],
                             blocks.numpy()[order], x.depth)

    def finish(self, x, x2, n_occ, want_idem):
        t_x, t_sq = O.trace(x), O.trace(x2)
        square = abs(t_sq - n_occ) <= abs(2.0 * t_x - t_sq - n_occ)
        idem = O.add_scaled(1.0, x2, -1.0, x).norm() if want_idem else None
        if square:
            return x2, O.SQUARE, t_x, t_sq, idem
        return O.add_scaled(2.0, x, -1.0, x2), O.EXPAND, t_x, t_sq, idem

    def scalar_tensor(self, v, like):
        return torch.tensor([int(v)], dtype=torch.int64)

    def to_numpy(self, t):
        return t.numpy()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, h, n_occ, nb, tau, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f = O.from_dense(h, nb)
        res = ShardedSP2(OracleEngine()).solve(f, n_occ, tau, criterion="fro")
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), p=O.to_dense(res.x),
                 traces=np.array(res.trace_history), iters=res.iteration,
                 idem=np.array(res.idempotency_history),
                 cuts=np.array(res.cuts_history), work=np.array(res.local_work),
                 leaf=np.array(res.leaf_products))
    finally:
        dist.destroy_process_group()


def test_partition_work_properties():
    rng = np.random.default_rng(0)
    w = rng.integers(0, 50, 256)
    for world in (1, 2, 3, 8):
        cuts = partition_work(w, world)
        assert cuts[0] == 0 and cuts[-1] == 256 and len(cuts) == world + 1
        assert all(a <= b for a, b in zip(cuts, cuts[1:]))
        parts = [w[a:b].sum() for a, b in zip(cuts, cuts[1:])]
        assert sum(parts) == w.sum()
        assert max(parts) - w.sum() / world <= w.max()       # balanced to one block
    assert partition_work(np.zeros(64, dtype=np.int64), 4) == even_cuts(64, 4)


def test_morton_helpers_roundtrip():
    i, j = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    m = morton_keys(i.ravel(), j.ravel())
    assert sorted(m.tolist()) == list(range(256))
    ii, jj = morton_decode(m)
    assert np.array_equal(ii, i.ravel()) and np.array_equal(jj, j.ravel())
    assert morton_keys(1, 0) == 2 and morton_keys(0, 1) == 1   # row bit above column bit


def test_sharded_sp2_gloo_world2_matches_single_process(tmp_path):
    h, n_occ = water_cluster(8, seed=5)
    nb, tau = 16, 1e-9
    ref = O.sp2_solve(O.from_dense(h, nb), n_occ, tau, criterion="fro")
    port = _free_port()
    torch.multiprocessing.spawn(_worker, args=(2, port, h, n_occ, nb, tau, str(tmp_path)),
                                nprocs=2, join=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    for o in outs:
        assert int(o["iters"]) == ref.iterations
        assert np.array_equal(o["traces"], np.array(ref.trace_history))
        assert np.array_equal(o["idem"], np.array(ref.idem_history))
        assert np.array_equal(o["p"], O.to_dense(ref.x))
        assert list(o["leaf"]) == ref.leaf_products           # full counts = sum of shards
    # both ranks computed work, the cut moved with the measured work (persistence LB)
    w0, w1 = outs[0]["work"], outs[1]["work"]
    assert w0.sum() > 0 and w1.sum() > 0
    cuts = outs[0]["cuts"]
    assert np.array_equal(cuts, outs[1]["cuts"])
    assert any(not np.array_equal(cuts[0], c) for c in cuts[1:])
    tot = w0 + w1
    assert np.max(np.abs(w0[1:] - w1[1:]) / tot[1:]) < 0.5
