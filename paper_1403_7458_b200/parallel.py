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

__all__ = ["partition_work", "even_cuts", "ShardedSP2", "DeviceEngine", "ShardedResult"]


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
            keys, blocks, work, n_exec, n_full = eng.multiply_shard(x, tau, lo, hi)
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

    def multiply_shard(self, x, tau, lo, hi):
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
        nat.check(nat.load().spamm_multiply_range(x._h, x._h, tau, _leaf_kernel(self.kernel),
                                                  int(lo), int(hi), work.data_ptr(), stream,
                                                  ctypes.byref(out), ctypes.byref(st)))
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


def morton_of_keys(keys: np.ndarray, g: int) -> np.ndarray:
    """Morton position (row bit above column bit) of reference keys bi*G+bj."""
    return morton_keys(np.asarray(keys) // g, np.asarray(keys) % g)
