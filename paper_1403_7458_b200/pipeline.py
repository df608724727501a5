"""Host <-> device pipelined SP2 over a stream of Hamiltonians.

The reference solves one host matrix at a time (cli.py:134-150: read F,
``sp2_solve``, write P).  Fed a sequence of host Hamiltonians, this driver
keeps the GPU on the SP2 loop while the PCIe copy engines move the data:
problem k+1's H is uploaded and problem k-1's P downloaded on a separate copy
stream while problem k solves, through two device slots for H and two for P
(events order slot reuse).  Each problem is the single-problem path
(``build_from_dense`` -> ``sp2_solve`` -> ``to_dense``), so every P is bitwise
what the one-at-a-time calls return.

    ps, states = sp2_solve_many([h0, h1, ...], n_occ, tau, block_size=64)
"""

from __future__ import annotations

from . import _native as nat

__all__ = ["sp2_solve_many"]


def _pinned_host(x):
    import numpy as np
    import torch
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            raise ValueError("sp2_solve_many takes host matrices")
        t = x.to(torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
    return t if t.is_pinned() else t.pin_memory()


def sp2_solve_many(hamiltonians, n_occ, tau: float, block_size: int = 16, *, solver=None,
                   out=None, before_each=None, **solve_kw):
    """Solve a sequence of host Hamiltonians, overlapping transfers with compute.

    ``n_occ``: one occupation for all problems or one per problem.  ``solver``:
    ``f -> (p, state)`` on the current stream (default ``sp2_solve(f, n_occ_k,
    tau, **solve_kw)``; e.g. a multi-GPU ``NativeShardedSP2`` solve).
    ``out``: optional pinned host tensors for the densities.  ``before_each``:
    optional ``k -> None`` hook run on the compute stream before problem k.
    Returns ``(densities, states)``; densities are pinned host tensors (native
    size), complete when this returns.  All copies are ordered after work
    already queued on the current stream, and the current stream is made to
    wait for the last download, so CUDA events around the call bracket the
    whole job.
    """
    import torch

    from .quadtree import build_from_dense
    from .sp2 import sp2_solve

    hs = list(hamiltonians)
    if not hs:
        return [], []
    n = hs[0].shape[0]
    for h in hs:
        if len(h.shape) != 2 or tuple(h.shape) != (n, n):
            raise ValueError(f"all Hamiltonians must be {n}x{n}, got {tuple(h.shape)}")
    occ = list(n_occ) if hasattr(n_occ, "__len__") else [n_occ] * len(hs)
    if len(occ) != len(hs):
        raise ValueError("n_occ: one value or one per Hamiltonian")
    if out is not None and len(out) != len(hs):
        raise ValueError("out: one tensor per Hamiltonian")
    hs = [_pinned_host(h) for h in hs]
    riding = solver is None
    if not riding:
        user_solver = solver

        def solver(f, k):
            return user_solver(f, occ[k])
    if out is None:
        out = [torch.empty((n, n), dtype=torch.float64).pin_memory() for _ in hs]

    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    copy.wait_stream(comp)              # copies start after the caller's queued work
    nslot = min(2, len(hs))
    d_in = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(nslot)]
    d_out = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(nslot)]
    # the slot buffers are used on both streams: keep the caching allocator
    # from recycling them under a pending copy
    for t in d_in + d_out:
        t.record_stream(copy)
    lib = nat.load()

    def on_copy(fn):
        """Run fn on the copy stream; returns an event marking its end."""
        with torch.cuda.stream(copy):
            fn()
            ev = torch.cuda.Event()
            ev.record(copy)
        return ev

    def after(ev):
        if ev is not None:
            comp.wait_event(ev)

    def to_dense(p, slot):
        nat.check(lib.spamm_mat_to_dense(p._h, d_out[slot].data_ptr(), n, nat.current_stream()))

    states = []
    in_ready = [None] * nslot
    in_ready[0] = on_copy(lambda: d_in[0].copy_(hs[0], non_blocking=True))
    if riding:
        # The bulk copies of the neighbours ride this solve's K4 windows
        # (spamm_sp2_solve_ex): H_{k+1} up, P_{k-1} down.  Slot reuse is
        # ordered by construction: the chunks are issued after this solve's
        # first cull, i.e. after build(k-1) and to_dense(k-1) on the compute
        # stream, and to_dense(k+1) waits for this solve's copies.
        prev_done = None
        for k in range(len(hs)):
            s = k % nslot
            if before_each is not None:
                before_each(k)
            after(in_ready[s])
            f = build_from_dense(d_in[s], block_size)
            items = []
            if k + 1 < len(hs):
                items.append(nat.Transfer(d_in[(k + 1) % nslot].data_ptr(), hs[k + 1].data_ptr(),
                                          hs[k + 1].numel() * 8))
            if k > 0:
                items.append(nat.Transfer(out[k - 1].data_ptr(), d_out[(k - 1) % nslot].data_ptr(),
                                          n * n * 8))
            side = None
            if items:
                arr = (nat.Transfer * len(items))(*items)
                side = nat.SideCopies(copy.cuda_stream, arr, len(items), 0)
            p, state = sp2_solve(f, occ[k], tau, _side=side, **solve_kw)
            done = on_copy(lambda: None) if items else None
            if k + 1 < len(hs):
                in_ready[(k + 1) % nslot] = done
            after(prev_done)            # d_out[s]'s last reader: P_{k-2}, rode solve k-1
            to_dense(p, s)
            prev_done = done
            states.append(state)
        last = len(hs) - 1
        ev = torch.cuda.Event()
        ev.record(comp)
        with torch.cuda.stream(copy):
            copy.wait_event(ev)
            out[last].copy_(d_out[last % nslot], non_blocking=True)
    else:
        # custom solver: plain double buffering (uploads / downloads overlap
        # the neighbouring solves, not aligned to its kernels)
        out_free = [None] * nslot
        for k in range(len(hs)):
            s = k % nslot
            if k + 1 < len(hs):
                nxt = k + 1
                build_ev = torch.cuda.Event()
                build_ev.record(comp)   # builds of earlier problems are queued before here

                def up(nxt=nxt, build_ev=build_ev):
                    copy.wait_event(build_ev)
                    d_in[nxt % nslot].copy_(hs[nxt], non_blocking=True)
                in_ready[nxt % nslot] = on_copy(up)
            if before_each is not None:
                before_each(k)
            after(in_ready[s])
            f = build_from_dense(d_in[s], block_size)
            p, state = solver(f, k)
            after(out_free[s])
            to_dense(p, s)
            ev = torch.cuda.Event()
            ev.record(comp)

            def down(k=k, s=s, ev=ev):
                copy.wait_event(ev)
                out[k].copy_(d_out[s], non_blocking=True)
            out_free[s] = on_copy(down)
            states.append(state)
    comp.wait_stream(copy)
    torch.cuda.current_stream().synchronize()
    return out, states
