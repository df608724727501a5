"""Distributed-operand SpAMM for BASELINE config 5: H is split by
Morton segments of the block grid and no rank holds all of it.

Reference semantics: the paper's over-decomposition of the (i, k, j)
convolution space over PEs with a measured-cost balance (PAPER.md:505-512,
812-833), which the reference only simulates (chare_sim.py:180-328).  The SP2
driver over the same primitives -- X, X^2 and the update sharded, persistence
load balancing -- is ``dist.py``.  ``engine`` isolates device work:
:class:`DeviceEngine` calls the sm_100a library; the CPU tests supply an
oracle-backed engine and run the same logic under gloo.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .synth_morton import morton_keys

__all__ = ["partition_work", "even_cuts", "DeviceEngine", "ShardedMultiply", "ShardProduct",
           "morton_positions"]


from .dist import even_cuts, partition_work  # noqa: E402  (shared host logic)


def morton_positions(keys, g: int):
    """Morton position (row bit above column bit) of keys bi*G+bj; numpy or
    torch int64 (device tensors stay on the device)."""
    def spread(x):
        x = (x | (x << 16)) & 0x0000FFFF0000FFFF
        x = (x | (x << 8)) & 0x00FF00FF00FF00FF
        x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0F
        x = (x | (x << 2)) & 0x3333333333333333
        return (x | (x << 1)) & 0x5555555555555555
    return (spread(keys // g) << 1) | spread(keys % g)


@dataclass
class ShardProduct:
    c: object                      # this rank's C blocks (range, + mirrors on the symmetric path)
    leaf_products: int = 0         # reference-equivalent survivors of the rank's range
    executed_products: int = 0
    halo_blocks: int = 0           # operand blocks received from other ranks
    sent_blocks: int = 0
    seconds: dict = field(default_factory=dict)


class ShardedMultiply:
    """C = A*A with A distributed over ranks by Morton segments of the block
    grid (BASELINE config 5): no rank holds the whole operand.

    * ``globalize``: every rank's leaf tier of norm^2 is summed (one
      all-reduce of G*G doubles, 32 MB at config 5; each position has one
      owner, so the sum is exact) and installed as the shard's pyramid -- the
      tier sums are the whole matrix's, so every rank culls exactly as a
      single GPU would;
    * ``balance``: per-C-block task counts from a census on the global
      pyramid (identical on every rank) are cut into equal-work Morton
      segments (``partition_work``; SP2 replaces this with the previous
      iteration's counts, persistence load balancing);
    * ``multiply``: the rank lists the operand blocks its tasks read, requests
      the ones it does not own from their owners (all-to-all of counts, keys,
      then blocks: NCCL over NVLink on GPUs, gloo in the CPU tests), builds
      its extended operand (own + received blocks, global pyramid) and runs
      the range multiply.  C stays distributed; on the symmetric path a rank
      also writes the mirrors of its upper blocks.
    """

    def __init__(self, engine, group=None):
        import torch.distributed as dist
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def globalize(self, local, symmetric: bool):
        """All-reduce the leaf tier of norm^2 (and, for the INT8-sliced leaf
        kernel, the row / column scale exponents with MAX) and install the
        whole matrix's pyramid on the shard."""
        import torch.distributed as dist
        leaf = self.engine.leaf_norms2(local)
        if self.world > 1:
            dist.all_reduce(leaf, group=self.group)
        self.engine.set_pyramid(local, leaf, symmetric)
        self.ex = None
        ex = getattr(self.engine, "oz_exponents", lambda m: None)(local)
        if ex is not None:
            if self.world > 1:
                for e in ex:
                    dist.all_reduce(e, op=dist.ReduceOp.MAX, group=self.group)
            self.ex = ex
        return leaf

    def balance(self, local, tau: float):
        """(cuts, symmetric_ok): equal-work C segments from a census on the
        global pyramid (identical on every rank), and whether the symmetric
        path holds on the whole grid -- if a mirror ulp tie breaks it anywhere,
        every rank must run the full path (``multiply(..., symmetric=False)``)."""
        work, sym_ok = self.engine.census_work(local, tau)
        return partition_work(self.engine.to_numpy(work), self.world), sym_ok

    def _all_to_all(self, send, send_counts, recv_counts, row: int = 1):
        """Variable all-to-all of the rows of ``send`` (grouped by destination)."""
        import torch
        import torch.distributed as dist
        recv = torch.empty((int(sum(recv_counts)) * row,), dtype=send.dtype, device=send.device)
        if self.world == 1:
            recv.copy_(send.reshape(-1))
            return recv
        dist.all_to_all_single(recv, send.reshape(-1).contiguous(),
                               output_split_sizes=[int(c) * row for c in recv_counts],
                               input_split_sizes=[int(c) * row for c in send_counts],
                               group=self.group)
        return recv

    def multiply(self, local, owner_cuts: list, cuts: list, tau: float, leaf,
                 symmetric: bool) -> ShardProduct:
        import torch
        eng = self.engine
        t = {}
        t0 = time.perf_counter()
        if eng.is_symmetric(local) != bool(symmetric):
            eng.set_pyramid(local, leaf, symmetric)
        lo, hi = cuts[self.rank], cuts[self.rank + 1]
        g = eng.grid(local)
        need = eng.needed_keys(local, tau, lo, hi)
        bounds = torch.as_tensor(owner_cuts[1:-1], dtype=torch.int64, device=need.device)
        owner = torch.searchsorted(bounds, morton_positions(need, g), right=True)
        remote = owner != self.rank
        req_keys, req_owner = need[remote], owner[remote]
        order = torch.argsort(req_owner, stable=True)
        req_keys, req_owner = req_keys[order], req_owner[order]
        send_counts = torch.bincount(req_owner, minlength=self.world).to(torch.int64)
        recv_counts = self._all_to_all(send_counts, [1] * self.world, [1] * self.world)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        wanted = self._all_to_all(req_keys, sc, rc)              # keys others need from me
        t["plan"] = time.perf_counter() - t0
        blocks_out = eng.gather(local, wanted)
        nb = eng.block_size(local)
        blocks_in = self._all_to_all(blocks_out, rc, sc, row=nb * nb).reshape(-1, nb, nb)
        t["exchange"] = time.perf_counter() - t0 - t["plan"]
        ext = eng.extend(local, req_keys, blocks_in, leaf, symmetric)
        if getattr(self, "ex", None) is not None:   # the whole matrix's K4z row scales
            eng.install_exponents(ext, *self.ex)
        c, leaf_products, executed = eng.multiply_range(ext, tau, lo, hi)
        t["total"] = time.perf_counter() - t0
        return ShardProduct(c=c, leaf_products=leaf_products, executed_products=executed,
                            halo_blocks=int(req_keys.numel()), sent_blocks=int(wanted.numel()),
                            seconds=t)


class DeviceEngine:
    """Engine over libspamm_b200 (one GPU per rank)."""

    def __init__(self, kernel: str = "auto"):
        self.kernel = kernel

    def grid(self, x):
        return x.n_blocks

    def to_numpy(self, t):
        return t.cpu().numpy()

    # -- Morton-shard operands (ShardedMultiply) -------------------------------
    def block_size(self, m):
        return m.block_size

    def leaf_norms2(self, m):
        return m.leaf_norms2_device()

    def set_pyramid(self, m, leaf, symmetric):
        m.set_global_pyramid(leaf, symmetric)

    def is_symmetric(self, m):
        return bool(m.symmetric)

    def census_work(self, m, tau):
        import ctypes

        import torch

        from . import _native as nat
        g = m.n_blocks
        work = torch.zeros(g * g, dtype=torch.int32, device="cuda")
        st = nat.Stats()
        nat.check(nat.load().spamm_census_range(m._h, m._h, float(tau), 0, g * g,
                                                work.data_ptr(), nat.current_stream(),
                                                ctypes.byref(st)))
        return work.to(torch.int64), bool(st.symmetric) or not m.symmetric

    def needed_keys(self, m, tau, lo, hi):
        """Sorted unique keys of the operand blocks the shard's tasks read."""
        import ctypes

        import torch

        from . import _native as nat
        lib, stream = nat.load(), nat.current_stream()
        n = ctypes.c_int64()
        nat.check(lib.spamm_tasks_range(m._h, m._h, float(tau), int(lo), int(hi), None, None,
                                        None, 0, ctypes.byref(n), stream))
        cap = int(n.value)
        if cap == 0:
            return torch.empty(0, dtype=torch.int64, device="cuda")
        t = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(3)]
        nat.check(lib.spamm_tasks_range(m._h, m._h, float(tau), int(lo), int(hi),
                                        t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(), cap,
                                        ctypes.byref(n), stream))
        g = m.n_blocks
        ti, tk, tj = (x.to(torch.int64) for x in t)
        parts = [ti * g + tk, tk * g + tj]
        if m.symmetric:                 # K4z's B operand on the symmetric path: X_jk^T
            parts.append(tj * g + tk)
        return torch.unique(torch.cat(parts))

    def gather(self, m, keys):
        import torch
        nb = m.block_size
        if keys.numel() == 0:
            return torch.empty((0, nb, nb), dtype=torch.float64, device="cuda")
        own = m.keys_device()
        order = torch.argsort(own)
        pos = torch.searchsorted(own[order], keys)
        pos = order[pos.clamp(max=own.numel() - 1)]
        if not bool((own[pos] == keys).all()):
            raise RuntimeError("ShardedMultiply: a requested block is not owned by this rank")
        return m.blocks_device()[pos].contiguous()

    def extend(self, m, keys, blocks, leaf, symmetric):
        import torch

        from .quadtree import QuadTreeMatrix
        all_keys = torch.cat([m.keys_device(), keys.to(torch.int64)])
        all_blocks = torch.cat([m.blocks_device(), blocks.reshape(-1, m.block_size,
                                                                  m.block_size)])
        ext = QuadTreeMatrix.from_blocks(m.n_native, m.block_size, m.chunk_size, all_keys,
                                         all_blocks, m.depth)
        ext.set_global_pyramid(leaf, symmetric)
        return ext

    def oz_exponents(self, m):
        """K4z row / column exponents of the shard (None unless K4z applies)."""
        import torch

        from . import _native as nat
        if self.kernel not in ("auto", "ozaki") or m.block_size not in (32, 64):
            return None
        out = []
        for by_col in (0, 1):
            ex = torch.empty(m.n_blocks * m.block_size, dtype=torch.int32, device="cuda")
            nat.check(nat.load().spamm_mat_oz_exponents(m._h, by_col, ex.data_ptr(),
                                                        nat.current_stream()))
            out.append(ex)
        return tuple(out)

    def install_exponents(self, m, row, col):
        from . import _native as nat
        nat.check(nat.load().spamm_mat_set_oz_exponents(m._h, row.data_ptr(), col.data_ptr(),
                                                        nat.current_stream()))

    def multiply_range(self, m, tau, lo, hi):
        import ctypes

        from . import _native as nat
        from .kernel import _leaf_kernel
        from .quadtree import QuadTreeMatrix
        st = nat.Stats()
        out = ctypes.c_void_p()
        stream = nat.current_stream()
        nat.check(nat.load().spamm_multiply_range(m._h, m._h, float(tau),
                                                  _leaf_kernel(self.kernel), int(lo), int(hi),
                                                  None, stream, ctypes.byref(out),
                                                  ctypes.byref(st)))
        return QuadTreeMatrix(out, stream), int(st.leaf_products), int(st.executed_products)
