"""Seeded synthetic inputs for BASELINE.json's five configurations.

The paper's FreeON water clusters are not available; BASELINE.json restates
each workload as a generator, fixed here:

* cfg1: A_ij = exp(-0.1 |i-j|) u_ij, u ~ U[-1, 1) symmetrised as
  triu(u) + triu(u, 1).T (the reference's own recipe, matgen.py:481-482),
  A from seed 0, B from seed 1, N = 1024, Nb = 32, tau = 1e-8.
* cfg2-5 ("water-cluster-like"): n_mol molecule centres uniform in a cube
  of edge (n_mol / 0.0334)^(1/3) Angstrom; 25 sites per molecule = centre +
  N(0, 0.5^2) per axis; H_ij = 0.3 exp(-r_ij / 1.5) s_ij with s symmetric
  U[-1, 1); diagonal N(-1, 0.2^2) for the first 5 sites of each molecule,
  N(+1, 0.2^2) for the other 20; n_occ = 5 n_mol.  Molecules are ordered
  along a 3-D Hilbert curve (order 10, Skilling's transpose construction --
  the published algorithm the reference's ordering.py:66-105 also uses)
  and rows move as 25-row runs.  One numpy PCG64 stream per seed, draws in
  the order centres, jitter, s, diagonal.

Host-side numpy; this is input preparation, not the hot path.  The inputs
are bit-identical on every host: only correctly rounded IEEE operations are
used (no BLAS, whose kernels are chosen per CPU, and no ``np.exp``, whose
SIMD implementation is chosen per CPU) -- a last-ulp difference in H is
enough to move an SP2 run off the reference's trajectory after ~20
iterations.  ``input_digest`` pins that in the tests.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

__all__ = ["decay_pair", "water_cluster", "hilbert_keys_3d", "det_exp", "input_digest",
           "ConfigSpec", "CONFIGS"]

_LN2_HI = 6.93147180369123816490e-01   # 32 trailing zero bits: k * LN2_HI exact
_LN2_LO = 1.90821492927058770002e-10
_INV_LN2 = 1.44269504088896338700e+00


def det_exp(x) -> np.ndarray:
    """exp(x) from +, *, rint and ldexp only (host independent, < 2 ulp).

    Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2, degree-13 Taylor
    polynomial by Horner (numpy never fuses the multiply-add).
    """
    x = np.asarray(x, dtype=np.float64)
    k = np.rint(x * _INV_LN2)
    r = (x - k * _LN2_HI) - k * _LN2_LO
    p = np.full_like(r, 1.0 / 6227020800.0)          # 1/13!
    fact = 6227020800.0
    for n in range(12, -1, -1):
        fact /= (n + 1)
        p = p * r + 1.0 / fact
    return np.ldexp(p, k.astype(np.int64))


def input_digest(*arrays) -> str:
    """sha256 of the raw bytes of generated inputs (host-independence pin)."""
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def decay_pair(n: int = 1024, lam: float = 0.1, seeds=(0, 1)):
    """cfg1 operands: exp(-lam |i-j|) * symmetrised U[-1, 1)."""
    idx = np.arange(n)
    env = det_exp(-lam * np.abs(idx[:, None] - idx[None, :]))
    out = []
    for s in seeds:
        u = np.random.default_rng(s).uniform(-1.0, 1.0, size=(n, n))
        u = np.triu(u) + np.triu(u, 1).T
        out.append(env * u)
    return out


def hilbert_keys_3d(cells: np.ndarray, order: int) -> np.ndarray:
    """Hilbert keys of integer lattice cells (n, 3) in [0, 2^order).

    Skilling (2004) "Programming the Hilbert curve": axes -> transposed
    Hilbert index (inverse undo of the reflect/exchange pass from the top bit,
    then Gray encoding), then bit interleave axis 0 first.  Vectorised.
    """
    x = np.array(cells, dtype=np.int64, copy=True).reshape(-1, 3)
    m = np.int64(1) << (order - 1)
    q = m
    while q > 1:
        p = q - 1
        for a in range(3):
            hit = (x[:, a] & q) != 0
            x[hit, 0] ^= p
            miss = ~hit
            t = (x[miss, 0] ^ x[miss, a]) & p
            x[miss, 0] ^= t
            x[miss, a] ^= t
        q >>= 1
    for a in (1, 2):
        x[:, a] ^= x[:, a - 1]
    t = np.zeros(len(x), dtype=np.int64)
    q = m
    while q > 1:
        t[(x[:, 2] & q) != 0] ^= q - 1
        q >>= 1
    x ^= t[:, None]
    key = np.zeros(len(x), dtype=np.int64)
    for bit in range(order - 1, -1, -1):
        for a in range(3):
            key = (key << 1) | ((x[:, a] >> bit) & 1)
    return key


def _hilbert_molecule_order(centres: np.ndarray, order: int = 10) -> np.ndarray:
    side = 1 << order
    lo = centres.min(axis=0)
    span = centres.max(axis=0) - lo
    cells = np.zeros(centres.shape, dtype=np.int64)
    for a in range(3):
        if span[a] > 0:
            cells[:, a] = np.clip(((centres[:, a] - lo[a]) / span[a] * side).astype(np.int64),
                                  0, side - 1)
    return np.argsort(hilbert_keys_3d(cells, order), kind="stable")


def water_cluster(n_mol: int, seed: int = 0, density: float = 0.0334, sites: int = 25,
                  occupied: int = 5, jitter: float = 0.5, amp: float = 0.3,
                  decay: float = 1.5, diag_sigma: float = 0.2, hilbert: bool = True):
    """cfg2-5 Hamiltonian.  Returns (H dense (n, n) float64, n_occ)."""
    rng = np.random.default_rng(seed)
    n = n_mol * sites
    edge = (n_mol / density) ** (1.0 / 3.0)
    centres = rng.uniform(0.0, edge, size=(n_mol, 3))
    pos = np.repeat(centres, sites, axis=0) + rng.normal(0.0, jitter, size=(n, 3))
    r2 = np.zeros((n, n))
    for a in range(3):                         # fixed order, elementwise: host independent
        d = pos[:, a, None] - pos[None, :, a]
        r2 += d * d
    s = rng.uniform(-1.0, 1.0, size=(n, n))
    s = np.triu(s) + np.triu(s, 1).T
    h = amp * det_exp(-np.sqrt(r2) / decay) * s   # symmetric: r2 and s are exactly symmetric
    occ = np.tile(np.arange(sites) < occupied, n_mol)
    d = np.where(occ, -1.0, 1.0) + rng.normal(0.0, diag_sigma, size=n)
    np.fill_diagonal(h, d)
    if hilbert:
        perm = _hilbert_molecule_order(centres)
        rows = (perm[:, None] * sites + np.arange(sites)[None, :]).reshape(-1)
        h = h[np.ix_(rows, rows)]
    return np.ascontiguousarray(h), n_mol * occupied


_SM_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_SM_M1 = np.uint64(0xBF58476D1CE4E5B9)
_SM_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x) -> np.ndarray:
    """SplitMix64 finaliser (Steele et al.), uint64 wrap-around arithmetic."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + _SM_GAMMA
        z = (z ^ (z >> np.uint64(30))) * _SM_M1
        z = (z ^ (z >> np.uint64(27))) * _SM_M2
        return z ^ (z >> np.uint64(31))


def hash_sym_uniform(i, j, n: int, seed: int) -> np.ndarray:
    """Symmetric U[-1, 1) from a counter hash of (min(i,j), max(i,j)): 53-bit
    mantissa, exact arithmetic -- the CUDA twin (csrc/gen.cu) is bitwise equal."""
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    lo, hi = np.minimum(i, j), np.maximum(i, j)
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) * _SM_M1) ^ (lo * np.uint64(n) + hi)
    u = (splitmix64(key) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


@dataclass
class ClusterSites:
    """Row-ordered sites of a cluster Hamiltonian (cfg5 generator input)."""

    pos: np.ndarray      # (n, 3) site coordinates, Hilbert row order
    orig: np.ndarray     # (n,) original (pre-ordering) row index -> hash counter
    diag: np.ndarray     # (n,) diagonal values, Hilbert row order
    n_occ: int
    seed: int
    amp: float = 0.3
    decay: float = 1.5


def cluster_sites(n_mol: int, seed: int = 0, density: float = 0.0334, sites: int = 25,
                  occupied: int = 5, jitter: float = 0.5, diag_sigma: float = 0.2,
                  amp: float = 0.3, decay: float = 1.5) -> ClusterSites:
    """O(n) part of the counter-based cluster generator (config 5): geometry,
    diagonal and Hilbert row order from one PCG64 stream; the O(n^2) couplings
    are a pure function of (site positions, original indices, seed)."""
    rng = np.random.default_rng(seed)
    n = n_mol * sites
    edge = (n_mol / density) ** (1.0 / 3.0)
    centres = rng.uniform(0.0, edge, size=(n_mol, 3))
    pos = np.repeat(centres, sites, axis=0) + rng.normal(0.0, jitter, size=(n, 3))
    occ = np.tile(np.arange(sites) < occupied, n_mol)
    d = np.where(occ, -1.0, 1.0) + rng.normal(0.0, diag_sigma, size=n)
    perm = _hilbert_molecule_order(centres)
    rows = (perm[:, None] * sites + np.arange(sites)[None, :]).reshape(-1)
    return ClusterSites(np.ascontiguousarray(pos[rows]), rows.astype(np.int64),
                        np.ascontiguousarray(d[rows]), n_mol * occupied, seed, amp, decay)


def cluster_dense_cb(cs: ClusterSites) -> np.ndarray:
    """Dense H of the counter-based generator (host reference; small n only):
    H_ab = amp * exp(-r_ab / decay) * s(orig_a, orig_b), diagonal from cs.diag."""
    n = len(cs.orig)
    r2 = np.zeros((n, n))
    for a in range(3):
        dd = cs.pos[:, a, None] - cs.pos[None, :, a]
        r2 += dd * dd
    s = hash_sym_uniform(cs.orig[:, None], cs.orig[None, :], n, cs.seed)
    h = cs.amp * det_exp(-np.sqrt(r2) / cs.decay) * s
    np.fill_diagonal(h, cs.diag)
    return h


@dataclass(frozen=True)
class ConfigSpec:
    index: int
    name: str
    n_mol: int            # 0 for cfg1
    n: int
    block_size: int
    tau: float
    workload: str         # "multiply" | "sp2"


CONFIGS = {
    1: ConfigSpec(1, "cfg1-decay-N1024-Nb32", 0, 1024, 32, 1e-8, "multiply"),
    2: ConfigSpec(2, "cfg2-water30-N750-Nb32", 30, 750, 32, 1e-8, "multiply"),
    3: ConfigSpec(3, "cfg3-water90-N2250-Nb32-sp2", 90, 2250, 32, 1e-7, "sp2"),
    4: ConfigSpec(4, "cfg4-water150-N3750-Nb64-sp2", 150, 3750, 64, 1e-7, "sp2"),
    5: ConfigSpec(5, "cfg5-water4096-N102400-Nb64", 4096, 102400, 64, 1e-8, "multiply"),
}


def device_cluster(cs: ClusterSites, block_size: int, chunk_size: int | None = None,
                   shard: tuple | None = None):
    """Build the counter-based cluster H directly in HBM (spamm_mat_cluster);
    bitwise equal to build_from_dense(cluster_dense_cb(cs), block_size).
    ``shard=(lo, hi)``: only the blocks at Morton positions [lo, hi) (one
    rank's share for parallel.ShardedMultiply; spamm_mat_cluster_range)."""
    import ctypes

    import torch

    from . import _native as nat
    from .quadtree import QuadTreeMatrix, _default_chunk_size, _padded_geometry
    n = len(cs.orig)
    if chunk_size is None:
        chunk_size = _default_chunk_size(_padded_geometry(n, block_size)[0], block_size)
    pos = torch.from_numpy(np.ascontiguousarray(cs.pos, dtype=np.float64)).cuda()
    orig = torch.from_numpy(np.ascontiguousarray(cs.orig, dtype=np.int64)).cuda()
    diag = torch.from_numpy(np.ascontiguousarray(cs.diag, dtype=np.float64)).cuda()
    stream = nat.current_stream()
    out = ctypes.c_void_p()
    lib = nat.load()
    if shard is None:
        nat.check(lib.spamm_mat_cluster(pos.data_ptr(), orig.data_ptr(), diag.data_ptr(), n,
                                        int(block_size), int(chunk_size), float(cs.amp),
                                        float(cs.decay), int(cs.seed), stream,
                                        ctypes.byref(out)))
    else:
        nat.check(lib.spamm_mat_cluster_range(pos.data_ptr(), orig.data_ptr(), diag.data_ptr(),
                                              n, int(block_size), int(chunk_size),
                                              float(cs.amp), float(cs.decay), int(cs.seed),
                                              int(shard[0]), int(shard[1]), stream,
                                              ctypes.byref(out)))
    return QuadTreeMatrix(out, stream)
