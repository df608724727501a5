"""SpAMM on device-resident quadtree matrices (host mirror of ``spamm.kernel``).

``multiply(a, b, tau, mode, deterministic, workers)`` keeps the reference
signature and validation (kernel.py:157-173) and returns ``(C, ProductStats)``
with identical counters.  Everything between the arguments and the result
runs in ``libspamm_b200``:

* K2/K3 tiered cull + in-order compaction (replaces ``_sweep`` kernel.py:96-122
  and the sort/searchsorted block kernel.py:189-204),
* K4 leaf products with a task-sorted segmented reduction (replaces
  ``_gemm_batch`` kernel.py:64-77): K4z (FP64 products as exact int8 digit
  products on the tcgen05 tensor cores) for Nb in {32, 64}, DMMA otherwise,
* K1 finalisation of C (``_from_blocks`` kernel.py:219-220).

``mode``/``workers``/``deterministic`` are accepted for drop-in compatibility;
the GPU schedule is deterministic for every setting (one CTA owns one C block
and reduces its k-ascending segment in registers).  Extra keyword
``kernel``: "auto" (K4z for Nb in {32, 64} when the digit slices fit, DMMA
for Nb in {8, 16} and as the fallback), "ozaki" (force K4z; C elements in a
row / column holding Inf or NaN are recomputed in FP64 in the reference's
order), "dmma", or "exact"
(CUDA-core, the reference's exact rounding order: bitwise-identical C).
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .quadtree import QuadTreeMatrix, _check_conformable

__all__ = ["ProductStats", "multiply", "convolution_census", "leaf_gemm", "gemm_batch",
           "leaf_tasks", "set_symmetric_products", "set_dense_cull", "set_near_tau_ulps",
           "WORKERS_ENV_VAR"]

WORKERS_ENV_VAR = "SPAMM_WORKERS"


@dataclass
class ProductStats:
    """Per-tier occlusion counters for one multiply (kernel.py:38-61)."""

    tau: float
    visited: tuple
    culled: tuple
    leaf_products: int
    flop_estimate: int
    wall_seconds: float = 0.0
    # device timings (CUDA events), filled when multiply(..., timed=True)
    ms_cull: float = 0.0
    ms_leaf: float = 0.0
    ms_finalize: float = 0.0
    c_blocks: int = 0
    # symmetric SpAMM (X*X, X == X^T): leaf products actually executed
    executed_products: int = 0
    symmetric: bool = False
    # near-tau report (the parity contract's "documented ties", kernel.py:108):
    # per tier, tested products within near_tau_ulps ulp(tau) of tau, and the
    # smallest relative distance |p - tau| / tau of a tested product (inf when
    # none lies within tau * 2**-20, or tau == 0)
    near_tau: tuple = ()
    tau_margin: float = math.inf
    near_tau_ulps: int = 64

    def to_json_dict(self) -> dict:
        return {
            "tau": self.tau,
            "tiers": [{"t": t, "visited": int(v), "culled": int(c)}
                      for t, (v, c) in enumerate(zip(self.visited, self.culled))],
            "leaf_products": int(self.leaf_products),
            "flop_estimate": int(self.flop_estimate),
            "wall_seconds": self.wall_seconds,
        }

    def counts_equal(self, other: "ProductStats") -> bool:
        return (self.visited == other.visited and self.culled == other.culled
                and self.leaf_products == other.leaf_products)


def _resolve_workers(mode: str, workers) -> int:
    """kernel.py:125-135 (validation only; the GPU schedule ignores it)."""
    if mode == "serial":
        return 1
    if workers is not None:
        if workers < 1:
            raise ValueError(f"workers must be >= 1, got {workers}")
        return int(workers)
    env = os.environ.get(WORKERS_ENV_VAR)
    if env:
        return max(1, int(env))
    return os.cpu_count() or 1


def _check_tau(tau) -> float:
    tau = float(tau)
    if not math.isfinite(tau) or tau < 0:
        raise ValueError(f"tau must be finite and >= 0, got {tau}")
    return tau


def _leaf_kernel(kernel: str) -> int:
    try:
        return nat.LEAF_KERNELS[kernel]
    except KeyError:
        raise ValueError(f"kernel must be one of {sorted(nat.LEAF_KERNELS)}, got {kernel!r}")


def _stats_from(st: nat.Stats, block_size: int, wall: float) -> ProductStats:
    n = int(st.n_tiers)
    return ProductStats(
        tau=float(st.tau),
        visited=tuple(int(st.visited[t]) for t in range(n)),
        culled=tuple(int(st.culled[t]) for t in range(n)),
        leaf_products=int(st.leaf_products),
        flop_estimate=int(st.leaf_products) * 2 * block_size ** 3,
        wall_seconds=float(wall),
        ms_cull=float(st.ms_cull), ms_leaf=float(st.ms_leaf),
        ms_finalize=float(st.ms_finalize), c_blocks=int(st.c_blocks),
        executed_products=int(st.executed_products), symmetric=bool(st.symmetric),
        near_tau=tuple(int(st.near_tau[t]) for t in range(n)),
        tau_margin=float(st.tau_margin), near_tau_ulps=int(st.near_tau_ulps),
    )


def set_symmetric_products(enabled: bool) -> None:
    """Toggle the symmetric SpAMM path (on by default; results are bitwise
    identical either way -- the switch exists for A/B measurements)."""
    nat.check(nat.load().spamm_set_symmetric_products(1 if enabled else 0))


def set_near_tau_ulps(ulps: int) -> None:
    """Width of the near-tau band reported in ``ProductStats.near_tau`` (ulps
    of tau; default 64, the operand-norm error of the DMMA / K4z kernels
    against the reference; 1 suits the bitwise exact kernel)."""
    nat.check(nat.load().spamm_set_near_tau_ulps(int(ulps)))


def set_dense_cull(enabled: bool) -> None:
    """Toggle the dense cull for trees of depth <= 8 (on by default; task sets,
    order and counters are identical to the tier walk -- A/B switch)."""
    nat.check(nat.load().spamm_set_dense_cull(1 if enabled else 0))


def multiply(a: QuadTreeMatrix, b: QuadTreeMatrix, tau: float, mode: str = "serial",
             deterministic: bool = True, workers: int | None = None, *,
             kernel: str = "auto", timed: bool = False):
    """SpAMM C = A*B under occlusion tolerance ``tau`` (kernel.py:157-223)."""
    _check_conformable(a, b)
    tau = _check_tau(tau)
    if mode not in ("serial", "tasked"):
        raise ValueError(f"mode must be 'serial' or 'tasked', got {mode!r}")
    _resolve_workers(mode, workers)
    kid = _leaf_kernel(kernel)
    stream = nat.current_stream()
    t0 = time.perf_counter()
    st = nat.Stats()
    out = ctypes.c_void_p()
    nat.check(nat.load().spamm_multiply(a._h, b._h, tau, kid, 1 if timed else 0, stream,
                                        ctypes.byref(out), ctypes.byref(st)))
    c = QuadTreeMatrix(out, stream)
    return c, _stats_from(st, a.block_size, time.perf_counter() - t0)


def convolution_census(a: QuadTreeMatrix, b: QuadTreeMatrix, tau: float) -> ProductStats:
    """Counts only (kernel.py:226-239); identical to multiply's counters."""
    _check_conformable(a, b)
    tau = _check_tau(tau)
    t0 = time.perf_counter()
    st = nat.Stats()
    nat.check(nat.load().spamm_census(a._h, b._h, tau, nat.current_stream(), ctypes.byref(st)))
    return _stats_from(st, a.block_size, time.perf_counter() - t0)


def leaf_tasks(a: QuadTreeMatrix, b: QuadTreeMatrix, tau: float):
    """Surviving leaf triples as int64 host arrays (ti, tk, tj), grouped by C
    block along the Morton curve with k ascending.  The *set* equals the
    reference ``_sweep`` output (kernel.py:96-122); parity tests sort both."""
    import torch
    _check_conformable(a, b)
    tau = _check_tau(tau)
    lib = nat.load()
    stream = nat.current_stream()
    n = ctypes.c_int64()
    st = nat.Stats()
    nat.check(lib.spamm_census(a._h, b._h, tau, stream, ctypes.byref(st)))
    cap = int(st.leaf_products)
    bufs = [torch.empty(max(cap, 1), dtype=torch.int32, device="cuda") for _ in range(3)]
    nat.check(lib.spamm_tasks(a._h, b._h, tau, bufs[0].data_ptr(), bufs[1].data_ptr(),
                              bufs[2].data_ptr(), cap, ctypes.byref(n), stream))
    if n.value != cap:
        raise RuntimeError("task count changed between census and task listing")
    return tuple(x[:cap].cpu().numpy().astype(np.int64) for x in bufs)


def gemm_batch(a_pos, b_pos, c_pos, a_data, b_data, c_data, kernel: str = "auto") -> None:
    """The compiled seam ``_gemm_batch`` (kernel.py:74-77) on CUDA tensors:
    ``c_data[c_pos[t]] += a_data[a_pos[t]] @ b_data[b_pos[t]]`` in task order.
    Tasks of one C block must be contiguous (the reference sorts by C)."""
    import torch
    for name, t in (("a_pos", a_pos), ("b_pos", b_pos), ("c_pos", c_pos)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int64
                and t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous int64 CUDA tensor")
    for name, t in (("a_data", a_data), ("b_data", b_data), ("c_data", c_data)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64
                and t.is_contiguous() and t.dim() == 3 and t.shape[1] == t.shape[2]):
            raise ValueError(f"{name} must be a contiguous (m, Nb, Nb) float64 CUDA tensor")
    nb = int(c_data.shape[1])
    if not (a_data.shape[1] == b_data.shape[1] == nb):
        raise ValueError("leaf blocks must share one square shape")
    n = int(a_pos.numel())
    if not (b_pos.numel() == c_pos.numel() == n):
        raise ValueError("position arrays must have equal length")
    nat.check(nat.load().spamm_gemm_batch(a_pos.data_ptr(), b_pos.data_ptr(), c_pos.data_ptr(),
                                          n, a_data.data_ptr(), int(a_data.shape[0]),
                                          b_data.data_ptr(), int(b_data.shape[0]),
                                          c_data.data_ptr(), nb, _leaf_kernel(kernel),
                                          nat.current_stream()))


def leaf_gemm(a: np.ndarray, b: np.ndarray, c: np.ndarray) -> np.ndarray:
    """``c += a @ b`` for one block (kernel.py:80-93), in place, through the
    exact leaf kernel (i-k-j, k ascending, unfused: bitwise the reference)."""
    import torch
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if not (a.shape == b.shape == c.shape) or a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"leaf blocks must share one square shape, got "
                         f"{a.shape}, {b.shape}, {c.shape}")
    nb = a.shape[0]
    dev = "cuda"
    ad = torch.from_numpy(np.ascontiguousarray(a)).to(dev).reshape(1, nb, nb)
    bd = torch.from_numpy(np.ascontiguousarray(b)).to(dev).reshape(1, nb, nb)
    cd = torch.from_numpy(np.ascontiguousarray(c, dtype=np.float64)).to(dev).reshape(1, nb, nb)
    z = torch.zeros(1, dtype=torch.int64, device=dev)
    gemm_batch(z, z, z, ad, bd, cd, kernel="exact")
    c[...] = cd.reshape(nb, nb).cpu().numpy()
    return c


def reserve_memory(nbytes: int) -> None:
    """Pre-grow the library's device memory pool (kept mapped) so steady-state
    allocations never block on new mappings; e.g. a few x the matrix size."""
    nat.check(nat.load().spamm_reserve_pool(int(nbytes), nat.current_stream()))
