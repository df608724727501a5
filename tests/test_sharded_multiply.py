"""Distributed-operand SpAMM (parallel.ShardedMultiply) on CPU: gloo, world
size 2, an oracle-backed engine standing in for the GPUs.  The operand is
split by Morton segments (no rank holds all of it); every rank's C blocks
must equal the single-process product bitwise, and the halo exchange must
deliver exactly the blocks the shard's tasks read."""

import os
import socket
from dataclasses import dataclass

import numpy as np
import torch

from oracle import spamm_oracle as O
from paper_1403_7458_b200.parallel import ShardedMultiply, even_cuts, morton_positions
from paper_1403_7458_b200.synth import water_cluster


@dataclass
class Shard:
    n_native: int
    block_size: int
    chunk_size: int
    depth: int
    keys: np.ndarray
    data: np.ndarray
    tier_norms: list = None
    sym: bool = False

    @property
    def n_blocks(self):
        return 1 << self.depth


class OracleShardEngine:
    """CPU stand-in for DeviceEngine's shard methods (same semantics: the
    symmetric path runs the upper C blocks in range and writes mirrors)."""

    def grid(self, m):
        return m.n_blocks

    def block_size(self, m):
        return m.block_size

    def to_numpy(self, t):
        return t.numpy()

    def leaf_norms2(self, m):
        g = m.n_blocks
        leaf = np.zeros(g * g)
        if len(m.keys):
            leaf[m.keys] = O.leaf_norms2_recipe(m.data)
        return torch.from_numpy(leaf)

    def is_symmetric(self, m):
        return m.sym

    def set_pyramid(self, m, leaf, symmetric):
        g = m.n_blocks
        m.tier_norms = O.pyramid_from_leaf_norms2(leaf.numpy().reshape(g, g))
        m.sym = bool(symmetric)

    def _own_tasks(self, m, tau, lo, hi):
        _, _, ti, tk, tj = O.sweep(m.tier_norms, m.tier_norms, tau)
        mt = morton_positions(ti * m.n_blocks + tj, m.n_blocks)
        own = (mt >= lo) & (mt < hi)
        if m.sym:
            own &= ti <= tj
        return ti[own], tk[own], tj[own]

    def census_work(self, m, tau):
        g = m.n_blocks
        ti, _, tj = self._own_tasks(m, tau, 0, g * g)
        work = np.zeros(g * g, dtype=np.int64)
        np.add.at(work, morton_positions(ti * g + tj, g), 1)
        _, _, a, k, b = O.sweep(m.tier_norms, m.tier_norms, tau)
        fwd = np.sort((a * g + k) * g + b)
        sym_ok = np.array_equal(fwd, np.sort((b * g + k) * g + a))   # mirror-closed task set
        return torch.from_numpy(work), sym_ok

    def needed_keys(self, m, tau, lo, hi):
        g = m.n_blocks
        ti, tk, tj = self._own_tasks(m, tau, lo, hi)
        return torch.from_numpy(np.unique(np.concatenate([ti * g + tk, tk * g + tj])))

    def gather(self, m, keys):
        keys = keys.numpy()
        pos = np.searchsorted(m.keys, keys)
        assert np.array_equal(m.keys[np.minimum(pos, len(m.keys) - 1)], keys), "not owned"
        return torch.from_numpy(np.ascontiguousarray(m.data[pos]))

    def extend(self, m, keys, blocks, leaf, symmetric):
        k = np.concatenate([m.keys, keys.numpy()])
        d = np.concatenate([m.data, blocks.numpy().reshape(-1, m.block_size, m.block_size)])
        order = np.argsort(k)
        ext = Shard(m.n_native, m.block_size, m.chunk_size, m.depth, k[order], d[order])
        self.set_pyramid(ext, leaf, symmetric)
        return ext

    def multiply_range(self, m, tau, lo, hi):
        g, nb = m.n_blocks, m.block_size
        ti, tk, tj = self._own_tasks(m, tau, lo, hi)
        a_pos = np.searchsorted(m.keys, ti * g + tk)
        b_pos = np.searchsorted(m.keys, tk * g + tj)
        assert np.array_equal(m.keys[a_pos], ti * g + tk), "halo incomplete (A)"
        assert np.array_equal(m.keys[b_pos], tk * g + tj), "halo incomplete (B)"
        ckeys, c_pos = np.unique(ti * g + tj, return_inverse=True)
        c = np.zeros((len(ckeys), nb, nb))
        order = np.lexsort((tk, c_pos))          # C block, then k ascending (reference order)
        O.gemm_batch(a_pos[order], b_pos[order], c_pos[order], m.data, m.data, c)
        executed = len(ti)
        keys, data = [ckeys], [c]
        full = executed
        if m.sym:
            ci, cj = ckeys // g, ckeys % g
            mir = ci != cj
            keys.append(cj[mir] * g + ci[mir])
            data.append(np.transpose(c[mir], (0, 2, 1)))
            full = 2 * executed - int((ti == tj).sum())
        return (np.concatenate(keys), np.concatenate(data)), full, executed


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, h, nb, tau, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = O.from_dense(h, nb)
        g = full.n_blocks
        own_cuts = even_cuts(g * g, world)
        mk = morton_positions(full.keys, g)
        mine = (mk >= own_cuts[rank]) & (mk < own_cuts[rank + 1])
        local = Shard(full.n_native, nb, full.chunk_size, full.depth, full.keys[mine],
                      full.data[mine])
        sm = ShardedMultiply(OracleShardEngine())
        leaf = sm.globalize(local, symmetric=True)
        cuts, sym_ok = sm.balance(local, tau)
        prod = sm.multiply(local, own_cuts, cuts, tau, leaf, symmetric=sym_ok)
        (keys, data) = prod.c
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), keys=keys, data=data,
                 leaf=prod.leaf_products, executed=prod.executed_products,
                 halo=prod.halo_blocks, sent=prod.sent_blocks, cuts=np.array(cuts),
                 own=int(mine.sum()), pyramid=np.concatenate([t.ravel() for t in local.tier_norms]))
    finally:
        dist.destroy_process_group()


def test_sharded_multiply_gloo_world2_bitwise(tmp_path):
    h, _ = water_cluster(12, seed=4)
    nb, tau = 16, 1e-5
    full = O.from_dense(h, nb)
    ref, stats, _ = O.multiply(full, full, tau)
    port = _free_port()
    torch.multiprocessing.spawn(_worker, args=(2, port, h, nb, tau, str(tmp_path)), nprocs=2,
                                join=True)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    # the global pyramid every rank installed is the whole matrix's, bitwise
    want = np.concatenate([t.ravel() for t in full.tier_norms])
    for o in outs:
        assert np.array_equal(o["pyramid"], want)
        assert int(o["own"]) < len(full.keys)            # nobody holds the whole operand
    keys = np.concatenate([o["keys"] for o in outs])
    data = np.concatenate([o["data"] for o in outs])
    assert len(np.unique(keys)) == len(keys)             # every C block computed once
    order = np.argsort(keys)
    assert np.array_equal(keys[order], ref.keys)
    assert np.array_equal(data[order], ref.data)         # bitwise: same k order per block
    assert sum(int(o["leaf"]) for o in outs) == stats["leaf_products"]
    assert sum(int(o["halo"]) for o in outs) == sum(int(o["sent"]) for o in outs) > 0
    assert np.array_equal(outs[0]["cuts"], outs[1]["cuts"])
    e0, e1 = int(outs[0]["executed"]), int(outs[1]["executed"])
    assert abs(e0 - e1) <= 0.2 * (e0 + e1)                # census-balanced shards
