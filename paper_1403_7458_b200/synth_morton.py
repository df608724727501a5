"""Host-side Morton (Z-order) codes matching the device layout (csrc/common.cuh):
bit b of the row index goes to bit 2b+1, bit b of the column index to bit 2b."""

from __future__ import annotations

import numpy as np

__all__ = ["morton_keys", "morton_decode"]


def morton_keys(i, j) -> np.ndarray:
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    m = np.zeros(np.broadcast(i, j).shape, dtype=np.uint64)
    for b in range(32):
        m |= ((i >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b + 1)
        m |= ((j >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
    return m.astype(np.int64)


def morton_decode(m):
    m = np.asarray(m, dtype=np.uint64)
    i = np.zeros(m.shape, dtype=np.uint64)
    j = np.zeros(m.shape, dtype=np.uint64)
    for b in range(32):
        i |= ((m >> np.uint64(2 * b + 1)) & np.uint64(1)) << np.uint64(b)
        j |= ((m >> np.uint64(2 * b)) & np.uint64(1)) << np.uint64(b)
    return i.astype(np.int64), j.astype(np.int64)
