"""Device-resident quadtree matrices (host mirror of ``spamm.quadtree``).

Same public surface as the reference module quadtree.py (``QuadTreeMatrix``,
``build_from_dense``, ``to_dense``, ``verify_norms``, ``add_scaled``,
``trace``, ``identity``), same validation and error messages, but the
storage lives in HBM behind a ``libspamm_b200`` handle:

* leaf blocks ``(S, Nb, Nb)`` float64 along the Morton curve of (bi, bj);
* int64 keys ``bi * G + bj`` per stored block, an int32 slot map ``G x G``;
* the bit-exact norm pyramid (reference ``_tier_norms``, quadtree.py:93).

The reference's private views ``_block_keys`` / ``_block_data`` /
``_tier_norms`` (read by its tests, quadtree.py:91-93) are materialised
lazily on the host, in the reference's key order, for parity checks only.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat

__all__ = ["QuadTreeMatrix", "Node", "build_from_dense", "to_dense", "verify_norms",
           "add_scaled", "trace", "identity", "NORM_REL_TOL"]

NORM_REL_TOL = 1e-12


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def _padded_geometry(n: int, block_size: int):
    """quadtree.py:197-201."""
    depth = 0
    while (block_size << depth) < n:
        depth += 1
    return block_size << depth, depth


def _default_chunk_size(n_padded: int, block_size: int) -> int:
    """quadtree.py:204-205."""
    return max(block_size, n_padded >> 3)


class _DevArray:
    """Minimal ``__cuda_array_interface__`` exporter over library memory."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(ptr), False), "version": 3, "strides": None,
        }


@dataclass
class Node:
    """Lazy tree view (quadtree.py:46-57): 2x2 optional children or a leaf block."""

    tier: int
    norm: float
    children: list | None = None
    block: np.ndarray | None = None

    @property
    def is_leaf(self) -> bool:
        return self.block is not None


class QuadTreeMatrix:
    """Square FP64 matrix padded to ``Nb * 2^depth``, resident in HBM.

    Immutable after construction (quadtree.py:77-83); all arithmetic returns
    new matrices.  Build with :func:`build_from_dense`, :func:`identity` or
    :meth:`from_blocks`.
    """

    def __init__(self, handle: ctypes.c_void_p, stream: int):
        self._h = handle
        self._stream = stream
        # geometry only: the storage view (count, pointers) is read on first
        # use, which settles a lazily pruned product (one host sync) -- a
        # matrix passed straight on to the next multiply never pays for it
        info = nat.MatInfo()
        nat.check(nat.load().spamm_mat_info_peek(handle, ctypes.byref(info)))
        self._peek = info
        self._full = None
        self.n_native = int(info.n_native)
        self.block_size = int(info.block_size)
        self.chunk_size = int(info.chunk_size)
        self._depth = int(info.depth)
        self._host = None
        self._root = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and nat._lib is not None:
            nat._lib.spamm_mat_free(h)
            self._h = None

    # -- geometry (quadtree.py:98-125) --------------------------------------
    @property
    def depth(self) -> int:
        return self._depth

    @property
    def n_padded(self) -> int:
        return self.block_size << self._depth

    @property
    def n_blocks(self) -> int:
        return 1 << self._depth

    @property
    def _info(self):
        if self._full is None:
            info = nat.MatInfo()
            nat.check(nat.load().spamm_mat_info_get(self._h, ctypes.byref(info)))
            self._full = info
        return self._full

    @property
    def stored_leaf_count(self) -> int:
        return int(self._info.stored)

    @property
    def symmetric(self) -> bool:
        """Exactly symmetric (X == X^T bitwise); X*X then runs the symmetric path."""
        return bool((self._full or self._peek).symmetric)

    def _refresh(self) -> None:
        """Re-read the handle after the library finalised it in place."""
        info = nat.MatInfo()
        nat.check(nat.load().spamm_mat_info_get(self._h, ctypes.byref(info)))
        self._full = info
        self._peek = info
        self._host = None
        self._root = None

    # -- Morton shards (multi-GPU, parallel.ShardedMultiply) ----------------
    def leaf_norms2_device(self):
        """(G*G,) float64 leaf tier of norm^2 (row-major bi*G+bj, 0 where no block)."""
        import torch
        g = self.n_blocks
        out = torch.empty(g * g, dtype=torch.float64, device="cuda")
        nat.check(nat.load().spamm_mat_leaf_norms2(self._h, out.data_ptr(), nat.current_stream()))
        return out

    def set_global_pyramid(self, leaf_norms2, symmetric: bool) -> None:
        """Install the pyramid of the whole matrix (a shard then culls like it)."""
        import torch
        leaf = torch.as_tensor(leaf_norms2, dtype=torch.float64).to("cuda").contiguous()
        stream = nat.current_stream()
        nat.check(nat.load().spamm_mat_set_pyramid(self._h, leaf.data_ptr(), int(bool(symmetric)),
                                                   stream))
        self._refresh()

    def norm(self) -> float:
        """Frobenius norm (root of the pyramid)."""
        return float(self.norms_device()[0].item())

    def chunk_tier(self, chunk_size: int | None = None) -> int:
        nc = self.chunk_size if chunk_size is None else int(chunk_size)
        if not _is_pow2(nc) or nc < self.block_size or nc > self.n_padded:
            raise ValueError(f"invalid chunk size {nc} for n_padded {self.n_padded}, "
                             f"block size {self.block_size}")
        return self.depth - int(np.log2(nc // self.block_size))

    # -- zero-copy device views (torch) -----------------------------------
    def _view(self, ptr, shape, typestr):
        import torch
        dt = {"<f8": torch.float64, "<i8": torch.int64, "<i4": torch.int32}[typestr]
        if int(np.prod(shape)) == 0 or not ptr:
            return torch.empty(shape, dtype=dt, device="cuda")
        return torch.as_tensor(_DevArray(ptr, shape, typestr, self), device="cuda")

    def blocks_device(self):
        """(S, Nb, Nb) float64 leaf blocks in storage (Morton) order."""
        return self._view(self._info.data, (self.stored_leaf_count, self.block_size,
                                            self.block_size), "<f8")

    def keys_device(self):
        """(S,) int64 keys bi*G+bj in storage order."""
        return self._view(self._info.keys, (self.stored_leaf_count,), "<i8")

    def norms_device(self):
        """Flat norm pyramid; tier t at offset (4^t-1)/3, row-major."""
        return self._view(self._info.norms, (((1 << (2 * (self.depth + 1))) - 1) // 3,), "<f8")

    # -- host views in the reference's layout (tests / parity only) --------
    def _host_views(self):
        if self._host is None:
            import torch
            torch.cuda.current_stream().synchronize()
            keys = self.keys_device().cpu().numpy()
            order = np.argsort(keys, kind="stable")
            data = self.blocks_device().cpu().numpy()[order]
            flat = self.norms_device().cpu().numpy()
            tiers = []
            for t in range(self.depth + 1):
                off = ((1 << (2 * t)) - 1) // 3
                w = 1 << t
                tiers.append(flat[off:off + w * w].reshape(w, w).copy())
            self._host = (keys[order].astype(np.int64), np.ascontiguousarray(data), tiers)
        return self._host

    @property
    def _block_keys(self) -> np.ndarray:
        return self._host_views()[0]

    @property
    def _block_data(self) -> np.ndarray:
        return self._host_views()[1]

    @property
    def _tier_norms(self) -> list:
        return self._host_views()[2]

    # -- lazy linked-node view (quadtree.py:129-166) ------------------------
    @property
    def root(self) -> Node:
        if self._root is None:
            self._root = self._materialize()
        return self._root

    def _materialize(self) -> Node:
        keys, data, tiers = self._host_views()
        g = self.n_blocks
        present = np.zeros((g, g), dtype=bool)
        present.reshape(-1)[keys] = True
        pres = [present]
        while pres[0].shape[0] > 1:
            p = pres[0]
            h = p.shape[0] // 2
            pres.insert(0, p.reshape(h, 2, h, 2).any(axis=(1, 3)))

        def build(t, i, j):
            nrm = float(tiers[t][i, j])
            if t == self.depth:
                pos = int(np.searchsorted(keys, i * g + j))
                return Node(tier=t, norm=nrm, block=data[pos])
            ch = [[None, None], [None, None]]
            for ci in (0, 1):
                for cj in (0, 1):
                    if pres[t + 1][2 * i + ci, 2 * j + cj]:
                        ch[ci][cj] = build(t + 1, 2 * i + ci, 2 * j + cj)
            return Node(tier=t, norm=nrm, children=ch)

        if self.depth == 0:
            if len(keys):
                return build(0, 0, 0)
            return Node(tier=0, norm=0.0, block=np.zeros((self.block_size, self.block_size)))
        if not present.any():
            return Node(tier=0, norm=0.0, children=[[None, None], [None, None]])
        return build(0, 0, 0)

    # -- constructors -------------------------------------------------------
    @classmethod
    def from_blocks(cls, n_native: int, block_size: int, chunk_size: int, block_keys,
                    block_data, depth: int) -> "QuadTreeMatrix":
        """QuadTreeMatrix._from_blocks (quadtree.py:170-194) on the device."""
        import torch
        stream = nat.current_stream()
        keys = torch.as_tensor(np.asarray(block_keys, dtype=np.int64)
                               if not isinstance(block_keys, torch.Tensor) else block_keys,
                               dtype=torch.int64).to("cuda").contiguous()
        data = (block_data if isinstance(block_data, torch.Tensor)
                else torch.as_tensor(np.ascontiguousarray(block_data, dtype=np.float64)))
        data = data.to(device="cuda", dtype=torch.float64).contiguous()
        out = ctypes.c_void_p()
        nat.check(nat.load().spamm_mat_from_blocks(
            int(n_native), int(block_size), int(chunk_size), int(depth), keys.data_ptr(),
            data.data_ptr(), int(keys.numel()), stream, ctypes.byref(out)))
        return cls(out, stream)


def _as_device_f64(dense):
    import torch
    if isinstance(dense, torch.Tensor):
        t = dense.to(device="cuda", dtype=torch.float64)
    else:
        arr = np.asarray(dense, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(arr)).to("cuda", non_blocking=False)
    return t.contiguous()


def build_from_dense(dense, block_size: int = 16, chunk_size: int | None = None) -> QuadTreeMatrix:
    """build_from_dense (quadtree.py:208-242): pad, block, keep non-zero blocks.

    ``dense`` may be a numpy array or a torch tensor (host or CUDA).
    """
    shape = tuple(dense.shape)
    if len(shape) != 2 or shape[0] != shape[1]:
        raise ValueError(f"input must be a square matrix, got shape {shape}")
    n = shape[0]
    if n < 1:
        raise ValueError("matrix must have at least one row")
    if not _is_pow2(block_size):
        raise ValueError(f"block size must be a power of two, got {block_size}")
    n_padded, _ = _padded_geometry(n, block_size)
    if chunk_size is None:
        chunk_size = _default_chunk_size(n_padded, block_size)
    if not _is_pow2(chunk_size):
        raise ValueError(f"chunk size must be a power of two, got {chunk_size}")
    if chunk_size < block_size:
        raise ValueError(f"chunk size {chunk_size} smaller than block size {block_size}")
    if chunk_size > n_padded:
        raise ValueError(f"chunk size {chunk_size} exceeds padded size {n_padded}")
    stream = nat.current_stream()
    t = _as_device_f64(dense)
    out = ctypes.c_void_p()
    nat.check(nat.load().spamm_mat_from_dense(t.data_ptr(), n, n, int(block_size),
                                              int(chunk_size), stream, ctypes.byref(out)))
    return QuadTreeMatrix(out, stream)


def to_dense_device(a: QuadTreeMatrix):
    """Dense native-size CUDA tensor (padding stripped)."""
    import torch
    out = torch.empty((a.n_native, a.n_native), dtype=torch.float64, device="cuda")
    nat.check(nat.load().spamm_mat_to_dense(a._h, out.data_ptr(), a.n_native,
                                            nat.current_stream()))
    return out


def to_dense(a: QuadTreeMatrix) -> np.ndarray:
    """to_dense (quadtree.py:245-252): host numpy array, padding stripped."""
    return to_dense_device(a).cpu().numpy()


def identity(n: int, block_size: int = 16, chunk_size: int | None = None) -> QuadTreeMatrix:
    """identity (quadtree.py:308-323)."""
    if n < 1:
        raise ValueError("identity needs n >= 1")
    if not _is_pow2(block_size):
        raise ValueError(f"block size must be a power of two, got {block_size}")
    n_padded, _ = _padded_geometry(n, block_size)
    if chunk_size is None:
        chunk_size = _default_chunk_size(n_padded, block_size)
    stream = nat.current_stream()
    out = ctypes.c_void_p()
    nat.check(nat.load().spamm_mat_identity(int(n), int(block_size), int(chunk_size), stream,
                                            ctypes.byref(out)))
    return QuadTreeMatrix(out, stream)


def _check_conformable(a: QuadTreeMatrix, b: QuadTreeMatrix) -> None:
    if (a.n_native, a.n_padded, a.block_size) != (b.n_native, b.n_padded, b.block_size):
        raise ValueError(
            f"shape/blocking mismatch: ({a.n_native}, {a.n_padded}, {a.block_size}) "
            f"vs ({b.n_native}, {b.n_padded}, {b.block_size})")


def add_scaled(alpha: float, a: QuadTreeMatrix, beta: float, b: QuadTreeMatrix) -> QuadTreeMatrix:
    """add_scaled (quadtree.py:281-293): fl(fl(alpha*a) + fl(beta*b)), norms rebuilt."""
    _check_conformable(a, b)
    stream = nat.current_stream()
    out = ctypes.c_void_p()
    nat.check(nat.load().spamm_add_scaled(float(alpha), a._h, float(beta), b._h, stream,
                                          ctypes.byref(out)))
    return QuadTreeMatrix(out, stream)


def trace(a: QuadTreeMatrix) -> float:
    """trace (quadtree.py:296-305), same summation order."""
    v = ctypes.c_double()
    nat.check(nat.load().spamm_trace(a._h, nat.current_stream(), ctypes.byref(v)))
    return float(v.value)


def verify_norms(a: QuadTreeMatrix, rel_tol: float = NORM_REL_TOL):
    """verify_norms (quadtree.py:255-278): every node norm vs a bottom-up recount.

    Diagnostic (not on the hot path): walks the lazy host Node view, so a
    caller that edits ``root`` norms sees the corruption reported.
    """
    worst = 0.0

    def walk(node: Node) -> float:
        nonlocal worst
        if node.is_leaf:
            rec2 = float(np.einsum("ij,ij->", node.block, node.block))
        else:
            rec2 = 0.0
            for row in node.children:
                for child in row:
                    if child is not None:
                        rec2 += walk(child) ** 2
        dev = abs(node.norm ** 2 - rec2) / max(1.0, node.norm ** 2)
        worst = max(worst, dev)
        return node.norm

    walk(a.root)
    return worst <= rel_tol, worst
