"""Multi-GPU SP2: the C-block Morton curve sharded across ranks.

Reference semantics: the paper's over-decomposition of the (i, k, j)
convolution space with persistence-based load balancing (PAPER.md:505-512,
812-833), which the reference only *simulates* (chare_sim.py:180-328:
``build_chare_graph``, ``greedy_comm_balance`` using the previous measured
cost).  Here it is executed, one process per GPU:

* every rank holds X (replicated; cfg4 X is 114 MB) and its norm pyramid;
* the C grid, in the storage's Morton order, is cut into ``world`` contiguous
  segments of equal predicted work -- the per-C-block task counts of the
  previous iteration (persistence); the first iteration splits evenly;
* each rank runs the multiply on its segment only (``spamm_multiply_range``:
  the cull prunes every quadtree node whose Morton subtree misses the
  segment), on the symmetric path the upper blocks in range plus mirrors;
* the computed blocks are all-gathered (NCCL over NVLink on GPUs, gloo in the
  CPU tests) and X^2 is re-assembled identically on every rank;
* the rest of the iteration (traces, branch, fused update, idempotency) runs
  redundantly on the replicated X^2, so the trajectory is bitwise the
  single-GPU one and no scalar reduction is needed.

The engine argument isolates device work: :class:`DeviceEngine` calls the
sm_100a library; ``tests/test_distributed.py`` supplies a CPU engine backed
by the oracle to exercise this host logic with gloo (world size 2).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from .synth_morton import morton_keys

__all__ = ["partition_work", "even_cuts", "ShardedSP2", "DeviceEngine", "ShardedResult",
           "ShardedMultiply", "ShardProduct", "morton_positions", "NativeShardedSP2",
           "exchange_blocks", "block_owners"]


def even_cuts(n_pos: int, world: int) -> list:
    """Equal-length Morton segments [cuts[r], cuts[r+1])."""
    return [(n_pos * r) // world for r in range(world + 1)]


def partition_work(work: np.ndarray, world: int) -> list:
    """Cut the Morton-indexed work vector into ``world`` contiguous segments of
    (nearly) equal total work: cut r is the first position whose inclusive
    prefix sum reaches r/world of the total (deterministic on every rank)."""
    work = np.asarray(work, dtype=np.int64).reshape(-1)
    n = len(work)
    total = int(work.sum())
    if total == 0 or world == 1:
        return even_cuts(n, world)
    csum = np.cumsum(work)
    cuts = [0]
    for r in range(1, world):
        target = (total * r + world - 1) // world
        pos = int(np.searchsorted(csum, target, side="left")) + 1
        cuts.append(min(max(pos, cuts[-1]), n))
    cuts.append(n)
    return cuts


@dataclass
class ShardedResult:
    x: object
    iteration: int = 0
    converged: bool = False
    trace_history: list = field(default_factory=list)
    branch_history: list = field(default_factory=list)
    idempotency_history: list = field(default_factory=list)
    cuts_history: list = field(default_factory=list)
    local_work: list = field(default_factory=list)      # tasks this rank ran, per iteration
    leaf_products: list = field(default_factory=list)   # full (all ranks) per iteration
    seconds_per_iteration: list = field(default_factory=list)


class ShardedSP2:
    """SP2 with the multiply sharded over a torch.distributed process group."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist
        self.engine = engine
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    # -- collectives ---------------------------------------------------------
    def _allgather_blocks(self, keys, blocks):
        """Variable-size all-gather of (keys int64 [m], blocks f64 [m, nb, nb])."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return keys, blocks
        dev = blocks.device
        m = torch.tensor([keys.numel()], dtype=torch.int64, device=dev)
        sizes = [torch.zeros_like(m) for _ in range(self.world)]
        dist.all_gather(sizes, m, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        mx = max(sizes)
        nb = blocks.shape[-1]
        kp = torch.full((mx,), -1, dtype=torch.int64, device=dev)
        bp = torch.zeros((mx, nb, nb), dtype=blocks.dtype, device=dev)
        if keys.numel():
            kp[: keys.numel()] = keys
            bp[: keys.numel()] = blocks
        kl = [torch.empty_like(kp) for _ in range(self.world)]
        bl = [torch.empty_like(bp) for _ in range(self.world)]
        dist.all_gather(kl, kp, group=self.group)
        dist.all_gather(bl, bp, group=self.group)
        keys = torch.cat([k[:s] for k, s in zip(kl, sizes)])
        blocks = torch.cat([b[:s] for b, s in zip(bl, sizes)])
        return keys, blocks

    def _consistent_shard(self, x, tau, lo, hi):
        """Shard multiply with one symmetric-path decision for all ranks: a
        rank whose range meets a mirror ulp tie falls back to the full path, and
        then every rank must (else mirrors and full-range blocks overlap)."""
        import torch
        import torch.distributed as dist
        out = self.engine.multiply_shard(x, tau, lo, hi)
        sym = getattr(self.engine, "last_symmetric", None)
        if self.world == 1 or sym is None:
            return out
        flags = torch.tensor([1 if sym else 0, 1 if sym else 0], dtype=torch.int64,
                             device=out[2].device)
        flags[1] = -flags[1]
        dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=self.group)
        any_full, all_full = int(flags[0]) == 0, int(-flags[1]) == 0
        if any_full and not all_full:
            out = self.engine.multiply_shard(x, tau, lo, hi, symmetric=False)
        return out

    def _allreduce_sum(self, t):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t

    # -- solve ---------------------------------------------------------------
    def solve(self, f, n_occ: int, tau: float, max_iter: int = 100, criterion: str = "fro",
              fro_tol: float = 1e-6, idem_tol: float = 1e-9) -> ShardedResult:
        eng = self.engine
        x = eng.init_x0(f)
        n_pos = eng.grid(x) ** 2
        cuts = even_cuts(n_pos, self.world)
        res = ShardedResult(x=x)
        res.trace_history.append(eng.trace(x))
        want_idem = criterion == "fro"
        for _ in range(max_iter):
            t0 = time.perf_counter()
            res.cuts_history.append(list(cuts))
            lo, hi = cuts[self.rank], cuts[self.rank + 1]
            keys, blocks, work, n_exec, n_full = self._consistent_shard(x, tau, lo, hi)
            res.local_work.append(int(n_exec))
            keys, blocks = self._allgather_blocks(keys, blocks)
            x2 = eng.assemble(x, keys, blocks)
            work = self._allreduce_sum(work)
            counts = self._allreduce_sum(eng.scalar_tensor(n_full, like=work))
            res.leaf_products.append(int(counts.item()))
            # persistence load balancing: next cut from this iteration's tasks
            cuts = partition_work(eng.to_numpy(work), self.world)
            x_next, branch, t_x, t_sq, idem = eng.finish(x, x2, n_occ, want_idem)
            if want_idem:
                res.idempotency_history.append(idem)
                done = idem < fro_tol
            else:
                done = abs(t_sq - t_x) < idem_tol and abs(t_x - n_occ) < 1e-6 * n_occ
            if done:
                res.converged = True
                res.seconds_per_iteration.append(time.perf_counter() - t0)
                break
            x = x_next
            res.iteration += 1
            res.trace_history.append(eng.trace(x))
            res.branch_history.append(branch)
            res.seconds_per_iteration.append(time.perf_counter() - t0)
        res.x = x
        return res


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
        import torch.distributed as dist
        leaf = self.engine.leaf_norms2(local)
        if self.world > 1:
            dist.all_reduce(leaf, group=self.group)
        self.engine.set_pyramid(local, leaf, symmetric)
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

    def init_x0(self, f):
        from .sp2 import _reserve_for, gershgorin_bounds, sp2_init
        _reserve_for(f)
        return sp2_init(f, gershgorin_bounds(f))

    def trace(self, x):
        from .quadtree import trace
        return trace(x)

    def multiply_shard(self, x, tau, lo, hi, symmetric=True):
        import ctypes

        import torch

        from . import _native as nat
        from .kernel import _check_tau, _leaf_kernel
        from .quadtree import QuadTreeMatrix
        tau = _check_tau(tau)
        g = x.n_blocks
        work = torch.zeros(g * g, dtype=torch.int32, device="cuda")
        st = nat.Stats()
        out = ctypes.c_void_p()
        stream = nat.current_stream()
        lib = nat.load()
        if not symmetric:
            lib.spamm_set_symmetric_products(0)
        try:
            nat.check(lib.spamm_multiply_range(x._h, x._h, tau, _leaf_kernel(self.kernel),
                                               int(lo), int(hi), work.data_ptr(), stream,
                                               ctypes.byref(out), ctypes.byref(st)))
        finally:
            if not symmetric:
                lib.spamm_set_symmetric_products(1)
        self.last_symmetric = bool(st.symmetric) or not x.symmetric
        c = QuadTreeMatrix(out, stream)
        keys = c.keys_device().clone()
        blocks = c.blocks_device().clone()
        return keys, blocks, work.to(torch.int64), int(st.executed_products), int(st.leaf_products)

    def assemble(self, x, keys, blocks):
        from .quadtree import QuadTreeMatrix
        return QuadTreeMatrix.from_blocks(x.n_native, x.block_size, x.chunk_size, keys, blocks,
                                          x.depth)

    def finish(self, x, x2, n_occ, want_idem):
        import ctypes

        from . import _native as nat
        from .quadtree import QuadTreeMatrix
        from .sp2 import EXPAND, SQUARE
        stream = nat.current_stream()
        br = ctypes.c_int32()
        t_x, t_sq, idem = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        e = ctypes.c_void_p()
        nat.check(nat.load().spamm_sp2_finish(x._h, x2._h, float(n_occ), int(want_idem), stream,
                                              ctypes.byref(br), ctypes.byref(t_x),
                                              ctypes.byref(t_sq), ctypes.byref(idem),
                                              ctypes.byref(e)))
        if br.value == 0:
            return x2, SQUARE, t_x.value, t_sq.value, (idem.value if want_idem else None)
        return (QuadTreeMatrix(e, stream), EXPAND, t_x.value, t_sq.value,
                idem.value if want_idem else None)

    def scalar_tensor(self, v, like):
        import torch
        return torch.tensor([int(v)], dtype=torch.int64, device=like.device)

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
        return torch.unique(torch.cat([ti * g + tk, tk * g + tj]))

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


def morton_of_keys(keys: np.ndarray, g: int) -> np.ndarray:
    """Morton position (row bit above column bit) of reference keys bi*G+bj."""
    return morton_keys(np.asarray(keys) // g, np.asarray(keys) % g)


# ---------------------------------------------------------------------------
# Native sharded SP2 (the device path for N > 1)
# ---------------------------------------------------------------------------

def block_owners(keys, g: int, cut_pos) -> "torch.Tensor":
    """Owner rank of every C block in a sharded SP2 product: the rank whose
    Morton range holds the block's upper-triangle position (a rank computes
    its upper blocks and writes their mirrors)."""
    import torch
    i, j = keys // g, keys % g
    upper = torch.minimum(i, j) * g + torch.maximum(i, j)
    inner = torch.as_tensor(list(cut_pos[1:-1]), dtype=torch.int64, device=keys.device)
    return torch.searchsorted(inner, morton_positions(upper, g), right=True)


def exchange_blocks(keys, blocks, g: int, cut_pos, group=None) -> dict:
    """In-place all-gather of a sharded product's blocks: afterwards every
    rank's ``blocks`` (storage order, same layout on every rank) holds every
    rank's computed blocks.  One all_gather (NCCL on GPUs) of the owned blocks,
    padded to the largest share."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1 or blocks.shape[0] == 0:
        return {"sent_blocks": 0, "received_blocks": 0}
    rank = dist.get_rank(group)
    owner = block_owners(keys, g, cut_pos)
    counts = torch.bincount(owner, minlength=world).tolist()
    mx = max(counts)
    nb = blocks.shape[-1]
    mine = owner == rank
    send = torch.zeros((mx, nb, nb), dtype=blocks.dtype, device=blocks.device)
    send[: counts[rank]] = blocks[mine]
    out = torch.empty((world * mx, nb, nb), dtype=blocks.dtype, device=blocks.device)
    dist.all_gather_into_tensor(out, send, group=group)
    for r in range(world):
        if r != rank and counts[r]:
            blocks[owner == r] = out[r * mx: r * mx + counts[r]]
    return {"sent_blocks": counts[rank], "received_blocks": sum(counts) - counts[rank]}


class NativeShardedSP2:
    """SP2 on N GPUs (one process per GPU), X replicated: per iteration every
    rank runs the same dense cull (``spamm_sp2_multiply_shard``), computes the
    leaf products of its contiguous run of C nodes -- cut by the current
    iteration's task counts, so every rank gets the same work -- the owned
    blocks are all-gathered (``exchange_blocks``), and the rest of the
    iteration runs on every rank (``spamm_sp2_shard_finish``: traces, fused
    residual, branch, update).  The trajectory is bitwise the single-GPU
    ``sp2_solve``'s; at world size 1 it is that solve."""

    def __init__(self, kernel: str = "auto", group=None):
        import torch.distributed as dist
        self.kernel = kernel
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1

    def multiply_shard(self, x, tau: float, rank: int | None = None, world: int | None = None):
        import ctypes

        from . import _native as nat
        from .kernel import _check_tau, _leaf_kernel
        from .quadtree import QuadTreeMatrix
        rank = self.rank if rank is None else rank
        world = self.world if world is None else world
        st = nat.Stats()
        out = ctypes.c_void_p()
        cuts = (ctypes.c_int64 * (world + 1))()
        stream = nat.current_stream()
        nat.check(nat.load().spamm_sp2_multiply_shard(x._h, _check_tau(tau),
                                                      _leaf_kernel(self.kernel), int(rank),
                                                      int(world), stream, ctypes.byref(out),
                                                      ctypes.cast(cuts, ctypes.c_void_p),
                                                      ctypes.byref(st)))
        self.last_executed = int(st.executed_products)   # the whole product's (all ranks)
        return QuadTreeMatrix(out, stream), list(cuts), int(st.leaf_products)

    def finish(self, x, c, n_occ: float, want_idem: bool):
        import ctypes

        from . import _native as nat
        from .quadtree import QuadTreeMatrix
        stream = nat.current_stream()
        br = ctypes.c_int32()
        t_x, t_sq, idem = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        e = ctypes.c_void_p()
        nat.check(nat.load().spamm_sp2_shard_finish(x._h, c._h, float(n_occ), int(want_idem),
                                                    stream, ctypes.byref(br), ctypes.byref(t_x),
                                                    ctypes.byref(t_sq), ctypes.byref(idem),
                                                    ctypes.byref(e)))
        from .sp2 import EXPAND, SQUARE
        c._refresh()
        nxt = QuadTreeMatrix(e, stream) if e.value else c
        return (nxt, SQUARE if br.value == 0 else EXPAND, t_x.value, t_sq.value,
                idem.value if want_idem else None)

    def solve(self, f, n_occ: int, tau: float, max_iter: int = 100, criterion: str = "fro",
              fro_tol: float = 1e-6, idem_tol: float = 1e-9) -> ShardedResult:
        from .quadtree import trace
        from .sp2 import _reserve_for, gershgorin_bounds, sp2_init
        _reserve_for(f)
        x = sp2_init(f, gershgorin_bounds(f))
        g = x.n_blocks
        res = ShardedResult(x=x)
        res.trace_history.append(trace(x))
        want_idem = criterion == "fro"
        pending = False
        for _ in range(max_iter):
            t0 = time.perf_counter()
            c, cuts, leaf = self.multiply_shard(x, tau)
            res.cuts_history.append(cuts)
            res.leaf_products.append(leaf)
            # cuts give every rank an equal share of the executed products
            res.local_work.append(self.last_executed // self.world)
            exchange_blocks(c.keys_device(), c.blocks_device(), g, cuts, self.group)
            nxt, branch, t_x, t_sq, idem = self.finish(x, c, n_occ, want_idem)
            if pending:
                res.trace_history.append(t_x)
                pending = False
            if want_idem:
                res.idempotency_history.append(idem)
                done = idem < fro_tol
            else:
                done = abs(t_sq - t_x) < idem_tol and abs(t_x - n_occ) < 1e-6 * n_occ
            res.seconds_per_iteration.append(time.perf_counter() - t0)
            if done:
                res.converged = True
                break
            x = nxt
            res.iteration += 1
            res.branch_history.append(branch)
            pending = True
        if pending:
            res.trace_history.append(trace(x))
        res.x = x
        return res
