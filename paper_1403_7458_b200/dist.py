"""Distributed SP2: X, X^2 and the update sharded along the Morton curve,
one process per GPU (BASELINE north_star "Multi-GPU sharding").

Reference semantics: the paper over-decomposes the (i, k, j) convolution
space and rebalances from the previous iteration's measured work
(persistence load balancing), which the reference
only simulates (chare_sim.py:249-328 ``greedy_comm_balance``, with the prior
measured cost at :272).  Here it runs:

* **Ownership.**  The G x G block grid in the storage's Morton order is cut
  into ``world`` contiguous segments ``cuts``.  Block (i, j) belongs to the
  rank whose segment holds its Morton position -- or, while X is exactly
  symmetric (the symmetric SpAMM path), the position of its upper-triangle
  twin (min(i, j), max(i, j)), so a rank owns a block and its mirror.  X,
  X^2 and 2X - X^2 share one ownership, so every elementwise step is local.
* **Global structure, no replicated data.**  Each rank holds only its own
  blocks.  The leaf tier of norm^2 (G^2 doubles: 32 KB at cfg4, 32 MB at
  cfg5; one owner per position, so the sum is exact) is all-reduced and the
  same tier sums as ``_from_blocks`` (quadtree.py:188-192) give every rank
  the whole matrix's pyramid, so every rank culls exactly like one GPU would.
  The K4z row scales are all-reduced with MAX for the same reason.
* **Cull and gather.**  A rank culls only its own C segment (the upper
  blocks of it on the symmetric path; a mirror ulp tie anywhere makes every
  rank take the full path, as one GPU would), lists the operand blocks its
  tasks read, and fetches the ones it does not own from their owners: an
  all-to-all of counts, keys and blocks (NCCL over NVLink on GPUs).
* **Multiply, reduce four kinds of scalars.**  The leaf products of the
  segment run locally with no C reduction across GPUs.  tr X, tr X^2 (per
  diagonal block, summed in block order) and the idempotency residual (leaf
  tier of ||X^2 - X||^2, its root taken in the pyramid's order) are one
  all-reduce, so the branch and convergence decisions are bitwise the single
  GPU's.
* **Persistence load balancing.**  The per-C-block task counts of this
  iteration (all-reduced) cut the next iteration's segments; blocks whose
  owner changed move with one all-to-all.

The result is bitwise the single-GPU ``sp2_solve`` (same task sets, same
per-block products and reductions).  ``engine`` isolates the device work:
:class:`DeviceShardEngine` calls the sm_100a library; the CPU tests supply
an oracle-backed engine and run the same driver under gloo.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

__all__ = ["Comm", "owners", "pyramid_root2", "seq_sum", "DistributedSP2", "DistResult",
           "DeviceShardEngine", "partition_work", "even_cuts"]

UPPER, POS = "upper", "pos"


# ---------------------------------------------------------------------------
# helpers (host logic shared with parallel.py)
# ---------------------------------------------------------------------------

def even_cuts(n_pos: int, world: int) -> list:
    """Equal-length Morton segments [cuts[r], cuts[r+1])."""
    return [(n_pos * r) // world for r in range(world + 1)]


def partition_work(work, world: int) -> list:
    """Cut a Morton-indexed work vector into ``world`` contiguous segments of
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


def _spread(x):
    x = (x | (x << 16)) & 0x0000FFFF0000FFFF
    x = (x | (x << 8)) & 0x00FF00FF00FF00FF
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0F
    x = (x | (x << 2)) & 0x3333333333333333
    return (x | (x << 1)) & 0x5555555555555555


def owners(keys, g: int, cuts, mode: str):
    """Owner rank of the blocks ``keys`` (bi * G + bj; torch int64, any
    device): the segment holding the Morton position of (bi, bj) (``POS``)
    or of (min, max) (``UPPER``: a block and its mirror share an owner)."""
    import torch
    i, j = keys // g, keys % g
    if mode == UPPER:
        i, j = torch.minimum(i, j), torch.maximum(i, j)
    pos = (_spread(i) << 1) | _spread(j)
    inner = torch.as_tensor(list(cuts[1:-1]), dtype=torch.int64, device=keys.device)
    return torch.searchsorted(inner, pos, right=True)


def seq_sum(v) -> float:
    """Sequential sum in index order (trace: quadtree.py:305's block order)."""
    t = 0.0
    for x in np.asarray(v, dtype=np.float64).tolist():
        t = t + x
    return t


def pyramid_root2(leaf) -> float:
    """Root norm^2 of a pyramid built from a G x G leaf tier of norm^2 with
    the tier sums of _from_blocks (quadtree.py:188-192): (c00 + c01) +
    (c10 + c11), the root as ((c00 + c01) + c10) + c11 (numpy's contiguous
    run)."""
    a = np.asarray(leaf, dtype=np.float64)
    g = int(round(np.sqrt(a.size)))
    a = a.reshape(g, g)
    while a.shape[0] > 1:
        h = a.shape[0] // 2
        q = a.reshape(h, 2, h, 2)
        if h == 1:
            a = ((q[:, 0, :, 0] + q[:, 0, :, 1]) + q[:, 1, :, 0]) + q[:, 1, :, 1]
        else:
            a = (q[:, 0, :, 0] + q[:, 0, :, 1]) + (q[:, 1, :, 0] + q[:, 1, :, 1])
    return float(a[0, 0])


class Comm:
    """torch.distributed collectives with the world-size-1 shortcuts.  With
    the gloo backend (the CPU tests, and one-GPU multi-process tests) device
    tensors travel through host memory; with NCCL host tensors travel through
    the device.  ``calls`` / ``bytes`` count what went over the wire."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.gloo = self.on and dist.get_backend(group) == "gloo"
        self.calls = 0
        self.bytes = 0

    def _io(self, t):
        """(tensor on the backend's device, device to return to or None)."""
        import torch
        if self.gloo and t.is_cuda:
            return t.cpu(), t.device
        if not self.gloo and not t.is_cuda:
            return t.to(torch.device("cuda", torch.cuda.current_device())), t.device
        return t, None

    @staticmethod
    def _back(t, dev):
        return t.to(dev) if dev is not None else t

    def _reduce(self, t, op):
        import torch.distributed as dist
        if self.world == 1:
            return t
        self.calls += 1
        self.bytes += t.numel() * t.element_size()
        x, dev = self._io(t.contiguous())
        dist.all_reduce(x, op=op, group=self.group)
        return self._back(x, dev)

    def all_sum(self, t):
        import torch.distributed as dist
        return self._reduce(t, dist.ReduceOp.SUM)

    def all_max(self, t):
        import torch.distributed as dist
        return self._reduce(t, dist.ReduceOp.MAX)

    def all_min(self, t):
        import torch.distributed as dist
        return self._reduce(t, dist.ReduceOp.MIN)

    def all_to_all_rows(self, send, send_counts):
        """Rows of ``send`` grouped by destination rank (``send_counts`` per
        rank, a python list) -> (the rows every rank sent here, by source
        rank; the per-source counts)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return send, list(send_counts)
        shape = tuple(send.shape[1:])
        row = int(np.prod(shape)) if shape else 1
        flat, dev = self._io(send.reshape(-1).contiguous())
        sc = torch.tensor([int(c) for c in send_counts], dtype=torch.int64, device=flat.device)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(v) for v in rc.tolist()]
        out = torch.empty(sum(recv_counts) * row, dtype=send.dtype, device=flat.device)
        dist.all_to_all_single(out, flat, output_split_sizes=[c * row for c in recv_counts],
                               input_split_sizes=[int(c) * row for c in send_counts],
                               group=self.group)
        self.calls += 2
        self.bytes += flat.numel() * flat.element_size()
        return self._back(out, dev).reshape((-1,) + shape), recv_counts

    def all_gather_rows(self, t):
        """Concatenate every rank's rows (variable counts), rank order."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return t
        x, dev = self._io(t.contiguous())
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=x.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n, group=self.group)
        sizes = [int(v) for v in sizes]
        pad = torch.zeros((max(sizes),) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        pad[: x.shape[0]] = x
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        return self._back(torch.cat([p[:v] for p, v in zip(parts, sizes)]), dev)


# ---------------------------------------------------------------------------
# the driver
# ---------------------------------------------------------------------------

@dataclass
class DistResult:
    x: object                       # this rank's blocks of P
    iteration: int = 0
    converged: bool = False
    trace_history: list = field(default_factory=list)
    branch_history: list = field(default_factory=list)
    idempotency_history: list = field(default_factory=list)
    branch_margins: list = field(default_factory=list)
    leaf_products: list = field(default_factory=list)    # whole product, per multiply
    local_executed: list = field(default_factory=list)   # leaf products this rank ran
    cuts_history: list = field(default_factory=list)
    mode_history: list = field(default_factory=list)
    halo_blocks: list = field(default_factory=list)      # operand blocks fetched per multiply
    moved_blocks: list = field(default_factory=list)     # blocks re-homed by the rebalance
    owned_blocks: list = field(default_factory=list)
    seconds_per_iteration: list = field(default_factory=list)
    cuts: list = field(default_factory=list)
    mode: str = POS
    symmetric: bool = False
    leaf: object = None             # global leaf tier of norm^2 of x


class DistributedSP2:
    """SP2 with X, X^2 and 2X - X^2 Morton-sharded over a process group."""

    def __init__(self, engine, group=None):
        self.engine = engine
        self.comm = Comm(group)
        self.rank, self.world = self.comm.rank, self.comm.world

    # -- data movement -------------------------------------------------------
    def redistribute(self, m, g: int, cuts, mode: str):
        """Move every block of the local matrix ``m`` to its owner under
        (cuts, mode); returns the new local matrix and the blocks sent."""
        import torch
        eng = self.engine
        keys = eng.keys(m)
        dest = owners(keys, g, cuts, mode)
        stay = dest == self.rank
        if self.world == 1:
            return m, 0
        go = ~stay
        order = torch.argsort(dest[go], stable=True)
        sk = keys[go][order]
        sb = eng.blocks(m)[go][order]
        counts = torch.bincount(dest[go], minlength=self.world).tolist()
        rk, _ = self.comm.all_to_all_rows(sk, counts)
        rb, _ = self.comm.all_to_all_rows(sb, counts)
        out = eng.rebuild(m, keys[stay], eng.blocks(m)[stay], rk, rb)
        return out, int(go.sum())

    def _globalize(self, x, sym: bool):
        """All-reduce the leaf tier (and the K4z row scales) and install them
        on the shard (its operand copies them)."""
        eng = self.engine
        leaf = self.comm.all_sum(eng.leaf_norms2(x))
        eng.install_pyramid(x, leaf, sym)
        ex = eng.oz_exponents(x)
        if ex is not None:
            ex = tuple(self.comm.all_max(e) if e is not None else None for e in ex)
            eng.install_exponents(x, ex)
        return leaf, ex

    def _plan(self, x, g, cuts, mode, tau, lo, hi, sym):
        """The symmetric-path decision for the whole grid (a mirror ulp tie on
        any rank sends every rank down the full path, as on one GPU) and the
        operand keys this rank must fetch, grouped by owner (one native cull)."""
        import torch
        eng, comm = self.engine, self.comm
        ok, req, counts = eng.plan(x, tau, lo, hi, sym, self.rank, self.world, cuts, mode)
        sym_eff = sym
        if sym:
            sym_eff = bool(comm.all_min(torch.tensor([1 if ok else 0], dtype=torch.int64)).item())
            if ok and not sym_eff:
                _, req, counts = eng.plan(x, tau, lo, hi, False, self.rank, self.world, cuts,
                                          mode)
        return sym_eff, req, counts

    def _halo(self, x, req, counts):
        """Fetch the planned operand blocks from their owners (all-to-all of
        the keys, then of the blocks)."""
        wanted, rc = self.comm.all_to_all_rows(req, counts)     # keys others need from me
        blocks = self.engine.gather(x, wanted)
        got, _ = self.comm.all_to_all_rows(blocks, rc)
        return got

    # -- solve ---------------------------------------------------------------
    def solve(self, f, n_occ, tau: float, max_iter: int = 100, criterion: str = "fro",
              fro_tol: float = 1e-6, idem_tol: float = 1e-9, balance: str = "persistence"):
        """``f`` replicated on every rank (Gershgorin bounds and X0 bitwise
        the single GPU's, then each rank keeps its own blocks of X0)."""
        eng = self.engine
        g = eng.grid(f)
        bounds = eng.gershgorin(f)
        x0 = eng.sp2_init(f, bounds)
        sym = bool(eng.symmetric(x0))
        mode = UPPER if sym else POS
        # iteration 0 cut from a census of X0 * X0 (identical on every rank)
        work0 = eng.census_work(x0, tau, sym)
        cuts = partition_work(eng.to_numpy(work0), self.world) if balance != "even" else \
            even_cuts(g * g, self.world)
        x = eng.select(x0, owners(eng.keys(x0), g, cuts, mode) == self.rank)
        del x0
        return self._loop(x, g, cuts, mode, sym, n_occ, tau, max_iter, criterion, fro_tol,
                          idem_tol, balance)

    def solve_cluster(self, cs, block_size: int, tau: float, max_iter: int = 100,
                      criterion: str = "fro", fro_tol: float = 1e-6, idem_tol: float = 1e-9,
                      balance: str = "persistence"):
        """Config 5: SP2 of the counter-based cluster H (synth.cluster_sites)
        with no rank ever holding H or X.  Each rank generates its Morton share
        of H in HBM, the Gershgorin bounds come from a row range per rank
        evaluated on the fly (min / max over ranks: bitwise the single-GPU
        bounds), X0 = (eps_max I - H) / (eps_max - eps_min) is formed on the
        shard, and the first cut comes from a census of X0 * X0 on the
        all-reduced pyramid."""
        import torch
        eng, comm = self.engine, self.comm
        n = len(cs.orig)
        g = 1
        while g * block_size < n:
            g *= 2
        cuts0 = even_cuts(g * g, self.world)
        f = eng.cluster_shard(cs, block_size, cuts0[self.rank], cuts0[self.rank + 1])
        rows = even_cuts(n, self.world)
        lo, hi = eng.cluster_gershgorin(cs, rows[self.rank], rows[self.rank + 1])
        lo = float(comm.all_min(torch.tensor([lo], dtype=torch.float64)).item())
        hi = float(comm.all_max(torch.tensor([hi], dtype=torch.float64)).item())
        if not hi > lo:
            raise ValueError("degenerate spectral bounds: eps_max equals eps_min")
        x = eng.shard_init(f, lo, hi, owners(eng.keys(eng.identity_like(f)), g, cuts0, POS)
                           == self.rank)
        del f
        # census-balanced first cut on the whole matrix's pyramid, then re-home
        # X0 to its symmetric ownership
        leaf = comm.all_sum(eng.leaf_norms2(x))
        eng.install_pyramid(x, leaf, True)
        work = eng.census_work(x, tau, True)
        work = comm.all_max(work)       # identical on every rank (a safety net)
        cuts = partition_work(eng.to_numpy(work), self.world) if balance != "even" else cuts0
        x, _ = self.redistribute(x, g, cuts, UPPER)
        return self._loop(x, g, cuts, UPPER, True, cs.n_occ, tau, max_iter, criterion,
                          fro_tol, idem_tol, balance)

    def solve_sharded(self, x, g: int, cuts, mode: str, sym: bool, n_occ, tau: float,
                      max_iter: int = 100, criterion: str = "fro", fro_tol: float = 1e-6,
                      idem_tol: float = 1e-9, balance: str = "persistence"):
        """Start from a local shard of X0 (owned under (cuts, mode)) -- the
        path for operands no GPU can hold (config 5)."""
        return self._loop(x, g, cuts, mode, sym, n_occ, tau, max_iter, criterion, fro_tol,
                          idem_tol, balance)

    def _loop(self, x, g, cuts, mode, sym, n_occ, tau, max_iter, criterion, fro_tol,
              idem_tol, balance):
        import torch
        eng, comm = self.engine, self.comm
        want_idem = criterion == "fro"
        multi = self.world > 1
        res = DistResult(x=x)
        # one rank: the shard is the whole matrix (its own pyramid and K4z
        # scales are the global ones) and no collective runs
        leaf, ex = self._globalize(x, sym) if multi else (None, None)
        tr_pending = False
        for it in range(max_iter):
            t0 = time.perf_counter()
            res.cuts_history.append(list(cuts))
            res.mode_history.append(mode)
            if multi:       # (reading the count settles a lazily pruned shard: a sync)
                res.owned_blocks.append(eng.count(x))
            lo, hi = (cuts[self.rank], cuts[self.rank + 1]) if multi else (0, -1)
            sym_eff = sym
            ext = x
            if multi:
                # one symmetric-path decision for the whole grid (a mirror ulp
                # tie anywhere sends every rank down the full path, as on one GPU)
                sym_eff, req, counts = self._plan(x, g, cuts, mode, tau, lo, hi, sym)
                got = self._halo(x, req, counts)
                res.halo_blocks.append(int(req.numel()))
                ext = eng.extend(x, req, got, leaf, sym_eff, ex)
                mode_c = UPPER if sym_eff else POS
                if mode != mode_c:                  # symmetry lost: re-home X by position
                    x, _ = self.redistribute(x, g, cuts, mode_c)
                    mode = mode_c
            else:
                res.halo_blocks.append(0)
            # the rank's C segment, the whole-matrix scalars (one all-reduce
            # inside the step), the branch and the update on the shard
            (x_next, square, t_x, t_sq, idem, work, leaf_r,
             exec_r) = eng.sp2_step(ext, x, n_occ, tau, lo, hi, want_idem, sym_eff,
                                    comm if multi else None)
            del ext
            res.local_executed.append(int(exec_r))
            cnt = int(comm.all_sum(torch.tensor([int(leaf_r)], dtype=torch.int64)).item()) \
                if multi else int(leaf_r)
            res.leaf_products.append(cnt)
            if it == 0 or tr_pending:           # tr of X0, then of every accepted X
                res.trace_history.append(t_x)
                tr_pending = False
            t_ex = 2.0 * t_x - t_sq
            res.branch_margins.append(abs(t_ex - n_occ) - abs(t_sq - n_occ))
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
            sym = sym_eff
            res.iteration += 1
            res.branch_history.append("SQUARE" if square else "EXPAND")
            tr_pending = True
            if multi:
                # persistence load balancing: next cut from this iteration's counts
                if balance == "persistence":
                    w = comm.all_sum(work.to(torch.int64))
                    new_cuts = partition_work(eng.to_numpy(w), self.world)
                    if new_cuts != cuts:
                        x, moved = self.redistribute(x, g, new_cuts, mode)
                        res.moved_blocks.append(moved)
                        cuts = new_cuts
                leaf, ex = self._globalize(x, sym)
            res.seconds_per_iteration.append(time.perf_counter() - t0)
        if tr_pending:
            if multi:
                vec = eng.to_numpy(comm.all_sum(eng.diag_traces(x).to(torch.float64)))
                res.trace_history.append(seq_sum(vec[:g]))
            else:
                res.trace_history.append(eng.trace(x))
        res.x, res.cuts, res.mode, res.symmetric, res.leaf = x, cuts, mode, sym, leaf
        return res

    def gather(self, res):
        """The whole P on every rank (tests / small problems)."""
        eng = self.engine
        keys = self.comm.all_gather_rows(eng.keys(res.x))
        blocks = self.comm.all_gather_rows(eng.blocks(res.x))
        return eng.assemble(res.x, keys, blocks)


# ---------------------------------------------------------------------------
# device engine (libspamm_b200)
# ---------------------------------------------------------------------------

class DeviceShardEngine:
    """The driver's device work on one GPU per rank (libspamm_b200)."""

    def __init__(self, kernel: str = "auto"):
        self.kernel = kernel

    # -- access ---------------------------------------------------------------
    def grid(self, m):
        return m.n_blocks

    def count(self, m):
        return int(m.stored_leaf_count)

    def keys(self, m):
        return m.keys_device()

    def blocks(self, m):
        return m.blocks_device()

    def to_numpy(self, t):
        return t.detach().cpu().numpy()

    def _from_blocks(self, like, keys, blocks):
        import torch

        from .quadtree import QuadTreeMatrix
        nb = like.block_size
        return QuadTreeMatrix.from_blocks(like.n_native, nb, like.chunk_size,
                                          keys.to(torch.int64).contiguous(),
                                          blocks.reshape(-1, nb, nb).contiguous(), like.depth)

    def select(self, m, mask):
        return self._from_blocks(m, self.keys(m)[mask], self.blocks(m)[mask])

    def rebuild(self, m, keys, blocks, more_keys, more_blocks):
        import torch
        return self._from_blocks(m, torch.cat([keys, more_keys.to(keys.device)]),
                                 torch.cat([blocks, more_blocks.to(blocks.device)]))

    def assemble(self, like, keys, blocks):
        return self._from_blocks(like, keys, blocks)

    def gather(self, m, keys):
        """The stored blocks with the given keys (spamm_mat_gather_blocks)."""
        import torch

        from . import _native as nat
        nb = m.block_size
        keys = keys.to(device="cuda", dtype=torch.int64).contiguous()
        out = torch.empty((keys.numel(), nb, nb), dtype=torch.float64, device="cuda")
        if keys.numel():
            nat.check(nat.load().spamm_mat_gather_blocks(m._h, keys.data_ptr(), keys.numel(),
                                                         out.data_ptr(), nat.current_stream()))
        return out

    def plan(self, m, tau, lo, hi, sym, rank, world, cuts, mode):
        """spamm_shard_plan: (symmetric path held on the range, the remote
        operand keys grouped by owner, per-owner counts)."""
        import ctypes

        import torch

        from . import _native as nat
        g = m.n_blocks
        keys = torch.empty(g * g, dtype=torch.int64, device="cuda")
        cuts_h = (ctypes.c_int64 * (world + 1))(*[int(c) for c in cuts])
        counts = (ctypes.c_int64 * (world + 1))()
        ok = ctypes.c_int32()
        n_tasks = ctypes.c_int64()
        nat.check(nat.load().spamm_shard_plan(
            m._h, float(tau), int(lo), int(hi), int(bool(sym)), int(rank), int(world),
            ctypes.cast(cuts_h, ctypes.c_void_p), int(mode == UPPER), keys.data_ptr(),
            ctypes.cast(counts, ctypes.c_void_p), ctypes.byref(ok), ctypes.byref(n_tasks),
            nat.current_stream()))
        per = [int(counts[r]) for r in range(world)]
        return bool(ok.value), keys[: int(counts[world])], per

    def install_exponents(self, m, ex):
        from . import _native as nat
        row, col = ex
        nat.check(nat.load().spamm_mat_set_oz_exponents(
            m._h, row.data_ptr(), col.data_ptr() if col is not None else None,
            nat.current_stream()))

    # -- replicated start ------------------------------------------------------
    def gershgorin(self, f):
        from .sp2 import _reserve_for, gershgorin_bounds
        _reserve_for(f)
        return gershgorin_bounds(f)

    def sp2_init(self, f, bounds):
        from .sp2 import sp2_init
        return sp2_init(f, bounds)

    def symmetric(self, m):
        return bool(m.symmetric)

    # -- config 5: sharded start ---------------------------------------------------
    def cluster_shard(self, cs, block_size, lo, hi):
        from .synth import device_cluster
        return device_cluster(cs, block_size, shard=(lo, hi))

    def cluster_gershgorin(self, cs, row0, row1):
        import ctypes

        import torch

        from . import _native as nat
        pos = torch.from_numpy(np.ascontiguousarray(cs.pos, dtype=np.float64)).cuda()
        orig = torch.from_numpy(np.ascontiguousarray(cs.orig, dtype=np.int64)).cuda()
        diag = torch.from_numpy(np.ascontiguousarray(cs.diag, dtype=np.float64)).cuda()
        lo, hi = ctypes.c_double(), ctypes.c_double()
        nat.check(nat.load().spamm_cluster_gershgorin(
            pos.data_ptr(), orig.data_ptr(), diag.data_ptr(), len(cs.orig), float(cs.amp),
            float(cs.decay), int(cs.seed), int(row0), int(row1), nat.current_stream(),
            ctypes.byref(lo), ctypes.byref(hi)))
        return float(lo.value), float(hi.value)

    def identity_like(self, m):
        from .quadtree import identity
        return identity(m.n_native, m.block_size, m.chunk_size)

    def shard_init(self, f, lo, hi, eye_mask):
        """X0's share: (eps_max I - F) / (eps_max - eps_min) (sp2.py:79-89) on
        the shard (the identity's owned diagonal blocks, add_scaled)."""
        from .quadtree import add_scaled
        spread = hi - lo
        eye = self.select(self.identity_like(f), eye_mask)
        return add_scaled(hi / spread, eye, -1.0 / spread, f)

    # -- global structure --------------------------------------------------------
    def leaf_norms2(self, m):
        return m.leaf_norms2_device()

    def install_pyramid(self, m, leaf, sym):
        m.set_global_pyramid(leaf, sym)

    def _ozaki(self, m):
        return self.kernel in ("auto", "ozaki") and m.block_size in (32, 64)

    def oz_exponents(self, m):
        """K4z row exponents (and column ones; equal for a symmetric X but
        computed anyway -- the product may leave the symmetric path)."""
        import torch

        from . import _native as nat
        if not self._ozaki(m):
            return None
        out = []
        for by_col in (0, 1):
            ex = torch.empty(m.n_blocks * m.block_size, dtype=torch.int32, device="cuda")
            nat.check(nat.load().spamm_mat_oz_exponents(m._h, by_col, ex.data_ptr(),
                                                        nat.current_stream()))
            out.append(ex)
        return tuple(out)

    def _set_sym(self, on: bool):
        from . import _native as nat
        nat.check(nat.load().spamm_set_symmetric_products(1 if on else 0))

    # -- products ----------------------------------------------------------------
    def census_work(self, m, tau, sym):
        import ctypes

        import torch

        from . import _native as nat
        g = m.n_blocks
        work = torch.zeros(g * g, dtype=torch.int32, device="cuda")
        st = nat.Stats()
        self._set_sym(sym)
        try:
            nat.check(nat.load().spamm_census_range(m._h, m._h, float(tau), 0, g * g,
                                                    work.data_ptr(), nat.current_stream(),
                                                    ctypes.byref(st)))
        finally:
            self._set_sym(True)
        return work.to(torch.int64)

    def tasks(self, m, tau, lo, hi, sym):
        import ctypes

        import torch

        from . import _native as nat
        lib, stream = nat.load(), nat.current_stream()
        empty = torch.empty(0, dtype=torch.int64, device="cuda")
        if hi <= lo:
            return empty, empty, empty
        n = ctypes.c_int64()
        self._set_sym(sym)
        try:
            nat.check(lib.spamm_tasks_range(m._h, m._h, float(tau), int(lo), int(hi), None, None,
                                            None, 0, ctypes.byref(n), stream))
            cap = int(n.value)
            if cap == 0:
                return empty, empty, empty
            t = [torch.empty(cap, dtype=torch.int32, device="cuda") for _ in range(3)]
            nat.check(lib.spamm_tasks_range(m._h, m._h, float(tau), int(lo), int(hi),
                                            t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(),
                                            cap, ctypes.byref(n), stream))
        finally:
            self._set_sym(True)
        return tuple(x.to(torch.int64) for x in t)

    def extend(self, m, keys, blocks, leaf, sym, ex):
        """The rank's operand: its own blocks plus the fetched ones
        (spamm_shard_extend: Morton order, the shard's installed pyramid,
        symmetry flag and K4z scales -- the whole matrix's)."""
        import ctypes

        import torch

        from . import _native as nat
        from .quadtree import QuadTreeMatrix
        if keys.numel() == 0:
            return m
        keys = keys.to(device="cuda", dtype=torch.int64).contiguous()
        blocks = blocks.to(device="cuda", dtype=torch.float64).contiguous()
        out = ctypes.c_void_p()
        stream = nat.current_stream()
        nat.check(nat.load().spamm_shard_extend(m._h, keys.data_ptr(), blocks.data_ptr(),
                                                keys.numel(), stream, ctypes.byref(out)))
        return QuadTreeMatrix(out, stream)

    def multiply_range(self, m, tau, lo, hi, sym):
        import ctypes

        import torch

        from . import _native as nat
        from .kernel import _leaf_kernel
        from .quadtree import QuadTreeMatrix
        g = m.n_blocks
        work = torch.zeros(g * g, dtype=torch.int32, device="cuda")
        st = nat.Stats()
        out = ctypes.c_void_p()
        stream = nat.current_stream()
        self._set_sym(sym)
        try:
            nat.check(nat.load().spamm_multiply_range(m._h, m._h, float(tau),
                                                      _leaf_kernel(self.kernel), int(lo),
                                                      int(hi), work.data_ptr(), stream,
                                                      ctypes.byref(out), ctypes.byref(st)))
        finally:
            self._set_sym(True)
        c = QuadTreeMatrix(out, stream)
        return c, work, int(st.leaf_products), int(st.executed_products)

    # -- SP2 pieces -------------------------------------------------------------
    def sp2_step(self, ext, x, n_occ, tau, lo, hi, want_idem, sym, comm):
        """spamm_shard_sp2_step: the rank's C segment of X^2 from its operand
        ``ext``, the scalars of the whole matrices (``comm`` all-reduces one
        vector from inside the step; None on one rank), the branch and the
        fused update on the shard."""
        import ctypes

        import torch

        from . import _native as nat
        from .kernel import _leaf_kernel, _check_tau
        from .quadtree import QuadTreeMatrix
        g = x.n_blocks
        work = torch.zeros(g * g, dtype=torch.int32, device="cuda") if hi >= 0 else None
        st = nat.Stats()
        out = ctypes.c_void_p()
        br = ctypes.c_int32()
        t_x, t_sq, idem = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        stream = nat.current_stream()
        cb = nat.ALLREDUCE_FN()          # NULL: one rank, no collective
        if comm is not None:
            def _allreduce(_ctx, ptr, n, _stream):
                try:
                    t = torch.as_tensor(_DevArray(ptr, n, "<f8"), device="cuda")
                    t.copy_(comm.all_sum(t.clone()))
                    return 0
                except Exception:  # noqa: BLE001 - reported to the library as a failure
                    import traceback
                    traceback.print_exc()
                    return 1
            cb = nat.ALLREDUCE_FN(_allreduce)
        self._set_sym(sym)
        try:
            nat.check(nat.load().spamm_shard_sp2_step(
                ext._h, x._h, float(n_occ), _check_tau(tau), _leaf_kernel(self.kernel),
                int(lo), int(hi), work.data_ptr() if work is not None else None, int(want_idem),
                cb, None, stream, ctypes.byref(out), ctypes.byref(br), ctypes.byref(t_x),
                ctypes.byref(t_sq), ctypes.byref(idem), ctypes.byref(st)))
        finally:
            self._set_sym(True)
        return (QuadTreeMatrix(out, stream), br.value == 0, float(t_x.value), float(t_sq.value),
                float(idem.value) if want_idem else None, work, int(st.leaf_products),
                int(st.executed_products))

    def trace(self, m):
        from .quadtree import trace
        return trace(m)

    def diag_traces(self, m):
        import torch

        from . import _native as nat
        out = torch.empty(m.n_blocks, dtype=torch.float64, device="cuda")
        nat.check(nat.load().spamm_mat_diag_traces(m._h, out.data_ptr(), nat.current_stream()))
        return out


class _DevArray:
    """A raw device buffer seen by torch without a copy (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}
