"""CPU oracle for the SpAMM / SP2 hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
``paper_1403_7458_b200`` never imports anything under ``oracle/`` and fails
loudly when its CUDA library is missing.

It restates, array-in / array-out, the reference package ``spamm`` 0.1.0
(``/root/reference/pkg/src/spamm``), citing file:line for every function.
The arithmetic that defines the results lives in numpy / numba call sites
of the reference (no lock file; pyproject.toml:10-14 pins numpy>=1.24,
numba>=0.58; this image has numpy 2.3.5 and numba 0.65.0):

* leaf norm^2 ``np.einsum("tij,tij->t")`` (quadtree.py:186-187): numpy's
  ``sum_of_products_contig_contig_outstride0_two`` with the SSE2 build
  baseline = two lanes (even / odd element), each an unfused ``acc += x*x``
  over 8-element chunks in pair order (6,7),(4,5),(2,3),(0,1), then
  ``lane0 + lane1``.  :func:`leaf_norms2_recipe` restates that order and
  :func:`self_check_numpy` verifies numpy still follows it at start-up;
* tier sums ``reshape(h,2,h,2).sum(axis=(1,3))`` == ``(c00+c01)+(c10+c11)``;
* ``np.sqrt`` per tier (IEEE correctly rounded);
* leaf products: numba ``_gemm_acc`` i-k-j, unfused ``c += a*b``
  (kernel.py:64-71) -> ``oracle/leafgemm.c`` built with -ffp-contract=off;
* trace ``np.einsum("tii->")`` == sequential per diagonal block, then a
  sequential sum over blocks in key order (quadtree.py:305);
* Gershgorin row sums: numpy ``pairwise_sum`` (block 128, 8 accumulators),
  restated in :func:`pairwise_sum`.

Parity is pinned two ways: (1) tests/test_oracle_vs_reference.py runs the
real reference (importable in the build container) against this module;
(2) tests/golden/*.npz fixtures produced by tests/golden/make_golden.py from
the reference itself are checked by tests/test_oracle_golden.py, which also
runs on machines without /root/reference.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

NORM_REL_TOL = 1e-12
SQUARE = "SQUARE"
EXPAND = "EXPAND"

_HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------------------
# numeric recipes
# ---------------------------------------------------------------------------

def leaf_norms2_recipe(blocks: np.ndarray) -> np.ndarray:
    """Restated einsum("tij,tij->t") order (quadtree.py:186-187), vectorised over t.

    Two lanes; per 8-element chunk the products of pairs (6,7),(4,5),(2,3),(0,1)
    are added (unfused) to lanes (even, odd); a tail of <8 elements is
    consumed two at a time (odd tail element paired with 0); result lane0+lane1.
    """
    t = blocks.shape[0]
    x = np.ascontiguousarray(blocks, dtype=np.float64).reshape(t, -1)
    n = x.shape[1]
    l0 = np.zeros(t)
    l1 = np.zeros(t)
    i = 0
    while n - i >= 8:
        for p in (6, 4, 2, 0):
            a = x[:, i + p]
            b = x[:, i + p + 1]
            l0 = l0 + a * a
            l1 = l1 + b * b
        i += 8
    while i < n:
        a = x[:, i]
        l0 = l0 + a * a
        if i + 1 < n:
            b = x[:, i + 1]
            l1 = l1 + b * b
        i += 2
    return l0 + l1


def self_check_numpy() -> None:
    """Fail loudly if this numpy's einsum no longer follows the restated order."""
    rng = np.random.default_rng(7)
    for nb in (1, 2, 4, 32):
        blk = rng.standard_normal((8, nb, nb)) * np.exp(rng.standard_normal((8, 1, 1)) * 4)
        ref = np.einsum("tij,tij->t", blk, blk)
        if not np.array_equal(ref, leaf_norms2_recipe(blk)):
            raise RuntimeError("numpy einsum summation order differs from the restated "
                               "2-lane recipe; the bit-exact norm parity contract is void "
                               "on this numpy build")


def contig_sum_recipe(x: np.ndarray) -> float:
    """einsum's sum_of_arr for a contiguous run (used by trace when Nb = 1: the
    (t,1,1) diagonal coalesces to one contiguous vector): two lanes, per
    8-element chunk ((x0+x2)+(x4+x6)) added to lane 0 (odd elements to lane 1),
    tail two at a time, then lane0 + lane1."""
    x = np.asarray(x, dtype=np.float64)
    n = len(x)
    l0 = l1 = 0.0
    i = 0
    while n - i >= 8:
        l0 = ((float(x[i]) + float(x[i + 2])) + (float(x[i + 4]) + float(x[i + 6]))) + l0
        l1 = ((float(x[i + 1]) + float(x[i + 3])) + (float(x[i + 5]) + float(x[i + 7]))) + l1
        i += 8
    while i < n:
        l0 = float(x[i]) + l0
        if i + 1 < n:
            l1 = float(x[i + 1]) + l1
        i += 2
    return l0 + l1


def pairwise_sum(a: np.ndarray) -> float:
    """numpy's pairwise summation (PW_BLOCKSIZE=128, 8 accumulators), scalar."""
    n = len(a)
    if n < 8:
        r = 0.0
        for i in range(n):
            r += float(a[i])
        return r
    if n <= 128:
        r = [float(a[j]) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


# ---------------------------------------------------------------------------
# storage (quadtree.py)
# ---------------------------------------------------------------------------

@dataclass
class OMatrix:
    """Array view of the reference ``QuadTreeMatrix`` fields (quadtree.py:85-94)."""

    n_native: int
    block_size: int
    chunk_size: int
    keys: np.ndarray          # sorted int64, bi * G + bj
    data: np.ndarray          # (m, Nb, Nb) float64
    tier_norms: list          # tier_norms[t] is (2^t, 2^t) float64 norms

    @property
    def depth(self) -> int:
        return len(self.tier_norms) - 1

    @property
    def n_blocks(self) -> int:
        return 1 << self.depth

    @property
    def n_padded(self) -> int:
        return self.block_size << self.depth

    def norm(self) -> float:
        return float(self.tier_norms[0][0, 0])


def padded_geometry(n: int, block_size: int):
    """quadtree.py:197-201."""
    depth = 0
    while (block_size << depth) < n:
        depth += 1
    return block_size << depth, depth


def default_chunk_size(n_padded: int, block_size: int) -> int:
    """quadtree.py:204-205."""
    return max(block_size, n_padded >> 3)


def pyramid_from_leaf_norms2(norms2: np.ndarray) -> list:
    """quadtree.py:188-192: sqrt per tier; reshape(h,2,h,2).sum(axis=(1,3)) is
    (c00+c01)+(c10+c11) for h >= 2, but for the root (h = 1) numpy coalesces
    the two reduced axes into one contiguous run of 4 and sums it
    sequentially: ((c00+c01)+c10)+c11."""
    tiers = [np.sqrt(norms2)]
    while norms2.shape[0] > 1:
        h = norms2.shape[0] // 2
        q = norms2.reshape(h, 2, h, 2)
        if h == 1:
            norms2 = ((q[:, 0, :, 0] + q[:, 0, :, 1]) + q[:, 1, :, 0]) + q[:, 1, :, 1]
        else:
            norms2 = (q[:, 0, :, 0] + q[:, 0, :, 1]) + (q[:, 1, :, 0] + q[:, 1, :, 1])
        tiers.insert(0, np.sqrt(norms2))
    return tiers


def from_blocks(n_native, block_size, chunk_size, keys, data, depth) -> OMatrix:
    """quadtree.py:170-194: prune exact-zero blocks, build the norm pyramid."""
    keys = np.asarray(keys, dtype=np.int64)
    data = np.ascontiguousarray(data, dtype=np.float64)
    if len(keys):
        nz = data.reshape(len(keys), -1).any(axis=1)
        keys, data = keys[nz], data[nz]
    if len(keys) == 0:
        data = np.zeros((0, block_size, block_size))
    g = 1 << depth
    norms2 = np.zeros((g, g))
    if len(keys):
        norms2.reshape(-1)[keys] = leaf_norms2_recipe(data)
    return OMatrix(int(n_native), int(block_size), int(chunk_size), keys, data,
                   pyramid_from_leaf_norms2(norms2))


def from_dense(dense, block_size=16, chunk_size=None) -> OMatrix:
    """quadtree.py:208-242 (validation trimmed to what the tests use)."""
    dense = np.asarray(dense, dtype=np.float64)
    n = dense.shape[0]
    n_padded, depth = padded_geometry(n, block_size)
    if chunk_size is None:
        chunk_size = default_chunk_size(n_padded, block_size)
    g = n_padded // block_size
    padded = np.zeros((n_padded, n_padded))
    padded[:n, :n] = dense
    flat = np.ascontiguousarray(
        padded.reshape(g, block_size, g, block_size).transpose(0, 2, 1, 3)
    ).reshape(g * g, block_size, block_size)
    keys = np.flatnonzero(flat.reshape(g * g, -1).any(axis=1)).astype(np.int64)
    return from_blocks(n, block_size, chunk_size, keys, flat[keys].copy(), depth)


def to_dense(m: OMatrix) -> np.ndarray:
    """quadtree.py:245-252."""
    g, nb = m.n_blocks, m.block_size
    full = np.zeros((g * g, nb, nb))
    full[m.keys] = m.data
    dense = full.reshape(g, g, nb, nb).transpose(0, 2, 1, 3).reshape(g * nb, g * nb)
    return dense[:m.n_native, :m.n_native].copy()


def identity(n, block_size=16, chunk_size=None) -> OMatrix:
    """quadtree.py:308-323."""
    n_padded, depth = padded_geometry(n, block_size)
    g = n_padded // block_size
    n_diag = (n + block_size - 1) // block_size
    keys = np.arange(n_diag, dtype=np.int64) * g + np.arange(n_diag)
    data = np.zeros((n_diag, block_size, block_size))
    for b in range(n_diag):
        fill = min(block_size, n - b * block_size)
        data[b, :fill, :fill] = np.eye(fill)
    if chunk_size is None:
        chunk_size = default_chunk_size(n_padded, block_size)
    return from_blocks(n, block_size, chunk_size, keys, data, depth)


def add_scaled(alpha, a: OMatrix, beta, b: OMatrix) -> OMatrix:
    """quadtree.py:281-293: fl(fl(alpha*a) + fl(beta*b)) over the key union."""
    keys = np.union1d(a.keys, b.keys)
    data = np.zeros((len(keys), a.block_size, a.block_size))
    data[np.searchsorted(keys, a.keys)] = alpha * a.data
    data[np.searchsorted(keys, b.keys)] += beta * b.data
    return from_blocks(a.n_native, a.block_size, a.chunk_size, keys, data, a.depth)


def trace(m: OMatrix) -> float:
    """quadtree.py:296-305: per-diagonal-block sequential sums, then sequential."""
    g = m.n_blocks
    diag = np.arange(g, dtype=np.int64) * (g + 1)
    hit = np.flatnonzero(np.isin(m.keys, diag))
    if m.block_size == 1:
        return contig_sum_recipe(m.data[hit].reshape(-1))
    total = 0.0
    for p in hit:                       # keys are sorted -> diagonal blocks in key order
        d = np.diagonal(m.data[p])
        s = 0.0
        for v in d:
            s += float(v)
        total += s
    return float(total)


def verify_norms(m: OMatrix, rel_tol=NORM_REL_TOL):
    """quadtree.py:255-278, bottom-up over the dense pyramid."""
    worst = 0.0
    g = m.n_blocks
    leaf2 = np.zeros((g, g))
    if len(m.keys):
        leaf2.reshape(-1)[m.keys] = np.einsum("tij,tij->t", m.data, m.data)
    rec2 = leaf2
    for t in range(m.depth, -1, -1):
        nrm2 = m.tier_norms[t] ** 2
        dev = np.abs(nrm2 - rec2) / np.maximum(1.0, nrm2)
        worst = max(worst, float(dev.max()))
        if t:
            h = nrm2.shape[0] // 2
            rec2 = nrm2.reshape(h, 2, h, 2).sum(axis=(1, 3))
    return worst <= rel_tol, worst


# ---------------------------------------------------------------------------
# SpAMM (kernel.py)
# ---------------------------------------------------------------------------

_CHILD = np.array([(di, dk, dj) for di in (0, 1) for dk in (0, 1) for dj in (0, 1)],
                  dtype=np.int64)


def sweep(tn_a: list, tn_b: list, tau: float):
    """kernel.py:96-122: breadth-first tiered culling, strict ``>``."""
    depth = len(tn_a) - 1
    i = np.zeros(1, dtype=np.int64)
    k = np.zeros(1, dtype=np.int64)
    j = np.zeros(1, dtype=np.int64)
    visited, culled = [], []
    for t in range(depth + 1):
        keep = tn_a[t][i, k] * tn_b[t][k, j] > tau
        nk = int(np.count_nonzero(keep))
        visited.append(nk)
        culled.append(len(keep) - nk)
        i, k, j = i[keep], k[keep], j[keep]
        if t < depth:
            if nk == 0:
                visited.extend([0] * (depth - t))
                culled.extend([0] * (depth - t))
                break
            i = ((2 * i)[:, None] + _CHILD[:, 0]).ravel()
            k = ((2 * k)[:, None] + _CHILD[:, 1]).ravel()
            j = ((2 * j)[:, None] + _CHILD[:, 2]).ravel()
    return visited, culled, i, k, j


def tie_log(tn_a: list, tn_b: list, tau: float, ulps: int = 64):
    """Near-tau diagnostic over the products ``_sweep`` tests (kernel.py:96-122:
    the root, then the 8 children of every survivor per tier; the strict
    ``>`` is kernel.py:108).  Returns (near, margin): per tier the number of
    tested products p with |p - tau| <= ulps * ulp(tau), and the smallest
    |p - tau| / tau over tested products with |p - tau| <= tau * 2**-20
    (inf if none, and for tau == 0 where nothing is probed).  Not a reference
    function: it documents how close the reference's decisions came to a tie
    (the parity contract's "norm ties within one ulp of tau")."""
    depth = len(tn_a) - 1
    near = [0] * (depth + 1)
    margin = math.inf
    if not (tau > 0.0 and math.isfinite(tau)):
        return near, margin
    band = ulps * (np.nextafter(tau, np.inf) - tau)
    wide = math.ldexp(tau, -20)
    i = np.zeros(1, dtype=np.int64)
    k = np.zeros(1, dtype=np.int64)
    j = np.zeros(1, dtype=np.int64)
    for t in range(depth + 1):
        p = tn_a[t][i, k] * tn_b[t][k, j]
        d = np.abs(p - tau)
        near[t] = int(np.count_nonzero(d <= band))
        w = d[d <= wide]
        if len(w):
            margin = min(margin, float((w / tau).min()))
        keep = p > tau
        i, k, j = i[keep], k[keep], j[keep]
        if t == depth or len(i) == 0:
            break
        i = ((2 * i)[:, None] + _CHILD[:, 0]).ravel()
        k = ((2 * k)[:, None] + _CHILD[:, 1]).ravel()
        j = ((2 * j)[:, None] + _CHILD[:, 2]).ravel()
    return near, margin


def task_order(ti, tk, tj, g, block_size, chunk_size):
    """kernel.py:189-196: sort key C-chunk-major, in-chunk row-major, then k."""
    cs = max(1, chunk_size // block_size)
    gc = g // cs
    key = ((((ti // cs) * gc + tj // cs) * cs + ti % cs) * cs + tj % cs) * g + tk
    return np.argsort(key, kind="stable")


class _LeafLib:
    _lib = None

    @classmethod
    def get(cls):
        if cls._lib is None:
            path = os.path.join(_HERE, "_build", _variant() + ".so")
            if not os.path.exists(path):
                build_c()
            lib = ctypes.CDLL(path)
            lib.oracle_gemm_batch.restype = ctypes.c_int
            lib.oracle_gemm_batch.argtypes = [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
            cls._lib = lib
        return cls._lib


def _variant() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
    except OSError:
        flags = ""
    if " avx512f" in flags:
        return "libleafgemm_avx512"
    if " avx2" in flags:
        return "libleafgemm_avx2"
    return "libleafgemm_x86_64"


def build_c() -> None:
    """Compile oracle/leafgemm.c (three ISA variants, all -ffp-contract=off)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def gemm_batch(a_pos, b_pos, c_pos, a_data, b_data, c_data, threads: int = 1):
    """kernel.py:64-77 (+ tasked slices kernel.py:138-147, 206-217), in C.

    Threads take contiguous slices cut on C-block boundaries, so every C block
    is accumulated by one thread in task order: bitwise independent of threads.
    """
    a_pos = np.ascontiguousarray(a_pos, dtype=np.int64)
    b_pos = np.ascontiguousarray(b_pos, dtype=np.int64)
    c_pos = np.ascontiguousarray(c_pos, dtype=np.int64)
    n = len(a_pos)
    if n == 0:
        return
    threads = max(1, int(threads))
    starts = np.concatenate(([0], np.flatnonzero(np.diff(c_pos)) + 1))
    targets = (np.arange(1, threads) * n) // threads
    cut = np.unique(starts[np.clip(np.searchsorted(starts, targets), 0, len(starts) - 1)])
    bounds = np.unique(np.concatenate(([0], cut, [n]))).astype(np.int64)
    assert c_data.flags.c_contiguous and a_data.flags.c_contiguous and b_data.flags.c_contiguous
    rc = _LeafLib.get().oracle_gemm_batch(
        a_pos.ctypes.data, b_pos.ctypes.data, c_pos.ctypes.data, n,
        a_data.ctypes.data, b_data.ctypes.data, c_data.ctypes.data,
        int(a_data.shape[1]), bounds.ctypes.data, len(bounds) - 1, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_gemm_batch failed ({rc})")


def leaf_gemm(a, b, c):
    """kernel.py:80-93 restated as a pure-Python loop (small blocks only)."""
    n = a.shape[0]
    for i in range(n):
        for k in range(n):
            aik = a[i, k]
            for j in range(n):
                c[i, j] += aik * b[k, j]
    return c


def multiply(a: OMatrix, b: OMatrix, tau: float, threads: int = 1):
    """kernel.py:157-223.  Returns (C, stats dict, (ti, tk, tj) sorted tasks)."""
    t0 = time.perf_counter()
    visited, culled, ti, tk, tj = sweep(a.tier_norms, b.tier_norms, tau)
    g = a.n_blocks
    if len(ti) == 0:
        c = from_blocks(a.n_native, a.block_size, a.chunk_size, np.zeros(0, np.int64),
                        np.zeros((0, a.block_size, a.block_size)), a.depth)
    else:
        order = task_order(ti, tk, tj, g, a.block_size, a.chunk_size)
        ti, tk, tj = ti[order], tk[order], tj[order]
        c_keys, c_pos = np.unique(ti * g + tj, return_inverse=True)
        a_pos = np.searchsorted(a.keys, ti * g + tk)
        b_pos = np.searchsorted(b.keys, tk * g + tj)
        c_data = np.zeros((len(c_keys), a.block_size, a.block_size))
        gemm_batch(a_pos, b_pos, c_pos, a.data, b.data, c_data, threads)
        c = from_blocks(a.n_native, a.block_size, a.chunk_size, c_keys, c_data, a.depth)
    stats = {
        "tau": float(tau), "visited": tuple(int(v) for v in visited),
        "culled": tuple(int(v) for v in culled), "leaf_products": int(len(ti)),
        "flop_estimate": int(len(ti)) * 2 * a.block_size ** 3,
        "wall_seconds": time.perf_counter() - t0,
    }
    return c, stats, (ti, tk, tj)


# ---------------------------------------------------------------------------
# SP2 (sp2.py)
# ---------------------------------------------------------------------------

def gershgorin_bounds(f: OMatrix, sym_tol=1e-10):
    """sp2.py:68-76 (numpy pairwise row sums via ndarray.sum)."""
    dense = to_dense(f)
    asym = float(np.abs(dense - dense.T).max())
    if asym > sym_tol:
        raise ValueError(f"matrix is not symmetric: max |F - F^T| = {asym:.3e}")
    diag = np.diag(dense)
    radius = np.abs(dense).sum(axis=1) - np.abs(diag)
    return float((diag - radius).min()), float((diag + radius).max())


def sp2_init(f: OMatrix, bounds) -> OMatrix:
    """sp2.py:79-89."""
    lo, hi = bounds
    spread = hi - lo
    eye = identity(f.n_native, f.block_size, f.chunk_size)
    return add_scaled(hi / spread, eye, -1.0 / spread, f)


@dataclass
class OSP2Result:
    x: OMatrix
    iterations: int
    converged: bool
    branches: list = field(default_factory=list)
    trace_history: list = field(default_factory=list)
    leaf_products: list = field(default_factory=list)
    idem_history: list = field(default_factory=list)
    wall_seconds_per_iteration: list = field(default_factory=list)
    # |t_ex - n_occ| - |t_sq - n_occ| per multiply (sp2.py:97-99; >= 0: SQUARE)
    branch_margins: list = field(default_factory=list)
    # record_tasks=True: per multiply, sha256 of the sorted task keys
    # ((i G + k) G + j, int64 little-endian) and tie_log's (near total, margin)
    task_sha256: list = field(default_factory=list)
    tie_logs: list = field(default_factory=list)


def task_sha256(ti, tk, tj, g) -> str:
    """sha256 of a leaf task set as sorted int64 keys (i G + k) G + j."""
    import hashlib
    keys = np.sort((np.asarray(ti, np.int64) * g + tk) * g + tj).astype("<i8")
    return hashlib.sha256(keys.tobytes()).hexdigest()


def sp2_step(x: OMatrix, n_occ, tau, threads=1):
    """sp2.py:92-101."""
    x_sq, stats, _ = multiply(x, x, tau, threads)
    t_x = trace(x)
    t_sq = trace(x_sq)
    t_ex = 2.0 * t_x - t_sq
    if abs(t_sq - n_occ) <= abs(t_ex - n_occ):
        return x_sq, SQUARE, t_x, t_sq, stats, x_sq
    return add_scaled(2.0, x, -1.0, x_sq), EXPAND, t_x, t_sq, stats, x_sq


def sp2_solve(f: OMatrix, n_occ, tau, max_iter=100, idem_tol=1e-9, threads=1,
              criterion="trace", fro_tol=1e-6, record_tasks=False) -> OSP2Result:
    """sp2.py:115-143.  ``criterion="fro"`` is BASELINE cfg3's ||X^2-X||_F < tol,
    evaluated from reference primitives (add_scaled(1, X^2, -1, X).norm()) on
    the same X^2 the step computed, before the step is accepted."""
    x = sp2_init(f, gershgorin_bounds(f))
    res = OSP2Result(x=x, iterations=0, converged=False)
    res.trace_history.append(trace(x))
    for _ in range(max_iter):
        t0 = time.perf_counter()
        if record_tasks:
            _, _, ti, tk, tj = sweep(x.tier_norms, x.tier_norms, tau)
            res.task_sha256.append(task_sha256(ti, tk, tj, x.n_blocks))
            near, margin = tie_log(x.tier_norms, x.tier_norms, tau)
            res.tie_logs.append((int(sum(near)), margin))
        x_next, branch, t_x, t_sq, stats, x_sq = sp2_step(x, n_occ, tau, threads)
        res.leaf_products.append(stats["leaf_products"])
        res.branch_margins.append(abs((2.0 * t_x - t_sq) - n_occ) - abs(t_sq - n_occ))
        if criterion == "trace":
            done = abs(t_sq - t_x) < idem_tol and abs(t_x - n_occ) < 1e-6 * n_occ
        else:
            idem = add_scaled(1.0, x_sq, -1.0, x).norm()
            res.idem_history.append(idem)
            done = idem < fro_tol
        if done:
            res.converged = True
            res.wall_seconds_per_iteration.append(time.perf_counter() - t0)
            break
        x = x_next
        res.iterations += 1
        res.trace_history.append(trace(x))
        res.branches.append(branch)
        res.wall_seconds_per_iteration.append(time.perf_counter() - t0)
    res.x = x
    return res
