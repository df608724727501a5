"""ctypes binding of ``libspamm_b200.so`` (declared in ``include/spamm_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: importing the compute API without the library, or
calling it without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPAMM_LIB_PATH") or os.path.join(_HERE, "libspamm_b200.so")  # (override: A/B builds)

SPAMM_OK = 0
SPAMM_EINVAL = 1
SPAMM_ECUDA = 2
MAX_TIERS = 64
ABI_VERSION = 2

LEAF_KERNELS = {"auto": 0, "dmma": 1, "exact": 2, "dmma_cpasync": 3, "ozaki": 4}

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p


class MatInfo(ctypes.Structure):
    _fields_ = [
        ("n_native", c_i64), ("block_size", c_i32), ("depth", c_i32),
        ("chunk_size", c_i64), ("n_blocks", c_i64), ("stored", c_i64),
        ("data", c_vp), ("keys", c_vp), ("slot", c_vp), ("norms", c_vp), ("norms2", c_vp),
        ("symmetric", c_i32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("tau", c_f64), ("n_tiers", c_i32),
        ("visited", c_i64 * MAX_TIERS), ("culled", c_i64 * MAX_TIERS),
        ("leaf_products", c_i64), ("flop_estimate", c_i64), ("c_blocks", c_i64),
        ("ms_cull", ctypes.c_float), ("ms_leaf", ctypes.c_float), ("ms_finalize", ctypes.c_float),
        ("executed_products", c_i64), ("symmetric", c_i32),
        ("near_tau", c_i64 * MAX_TIERS), ("tau_margin", c_f64), ("near_tau_ulps", c_i32),
    ]


class SP2Report(ctypes.Structure):
    _fields_ = [
        ("iterations", c_i32), ("converged", c_i32), ("n_multiplies", c_i32),
        ("eps_min", c_f64), ("eps_max", c_f64),
        ("trace_history", c_vp), ("branch_history", c_vp), ("idem_history", c_vp),
        ("leaf_products", c_vp), ("executed_products", c_vp), ("ms_leaf", c_vp),
        ("branch_margin", c_vp), ("near_tau", c_vp), ("tau_margin", c_vp),
        ("wall_seconds", c_vp),
    ]


class Transfer(ctypes.Structure):
    _fields_ = [("dst", c_vp), ("src", c_vp), ("bytes", c_i64)]


class SideCopies(ctypes.Structure):
    _fields_ = [("stream", c_vp), ("items", ctypes.POINTER(Transfer)), ("n_items", c_i32),
                ("chunk_bytes", c_i64)]


# multi-GPU all-reduce callback of spamm_shard_sp2_step (dist.py)
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_vp, c_i64, c_vp)

_SIGS = {
    "spamm_abi_version": (c_i32, []),
    "spamm_last_error": (ctypes.c_char_p, []),
    "spamm_launch_count": (c_i64, []),
    "spamm_mat_from_dense": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_i64, c_vp, ctypes.POINTER(c_vp)]),
    "spamm_mat_from_blocks": (c_i32, [c_i64, c_i32, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp,
                                      ctypes.POINTER(c_vp)]),
    "spamm_mat_cluster": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_i64, c_f64, c_f64,
                                  ctypes.c_uint64, c_vp, ctypes.POINTER(c_vp)]),
    "spamm_mat_cluster_range": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_i64, c_f64, c_f64,
                                        ctypes.c_uint64, c_i64, c_i64, c_vp,
                                        ctypes.POINTER(c_vp)]),
    "spamm_mat_leaf_norms2": (c_i32, [c_vp, c_vp, c_vp]),
    "spamm_cluster_gershgorin": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_f64, c_f64, ctypes.c_uint64,
                                         c_i64, c_i64, c_vp, ctypes.POINTER(c_f64),
                                         ctypes.POINTER(c_f64)]),
    "spamm_mat_set_pyramid": (c_i32, [c_vp, c_vp, c_i32, c_vp]),
    "spamm_mat_oz_exponents": (c_i32, [c_vp, c_i32, c_vp, c_vp]),
    "spamm_mat_set_oz_exponents": (c_i32, [c_vp, c_vp, c_vp, c_vp]),
    "spamm_mat_identity": (c_i32, [c_i64, c_i32, c_i64, c_vp, ctypes.POINTER(c_vp)]),
    "spamm_mat_info_get": (c_i32, [c_vp, ctypes.POINTER(MatInfo)]),
    "spamm_mat_info_peek": (c_i32, [c_vp, ctypes.POINTER(MatInfo)]),
    "spamm_mat_free": (c_i32, [c_vp]),
    "spamm_mat_to_dense": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "spamm_multiply": (c_i32, [c_vp, c_vp, c_f64, c_i32, c_i32, c_vp, ctypes.POINTER(c_vp),
                               ctypes.POINTER(Stats)]),
    "spamm_census": (c_i32, [c_vp, c_vp, c_f64, c_vp, ctypes.POINTER(Stats)]),
    "spamm_set_symmetric_products": (c_i32, [c_i32]),
    "spamm_set_dense_cull": (c_i32, [c_i32]),
    "spamm_set_near_tau_ulps": (c_i32, [c_i32]),
    "spamm_multiply_range": (c_i32, [c_vp, c_vp, c_f64, c_i32, c_i64, c_i64, c_vp, c_vp,
                                     ctypes.POINTER(c_vp), ctypes.POINTER(Stats)]),
    "spamm_reserve_pool": (c_i32, [c_i64, c_vp]),
    "spamm_shard_plan": (c_i32, [c_vp, c_f64, c_i64, c_i64, c_i32, c_i32, c_i32, c_vp, c_i32,
                                 c_vp, c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_i64), c_vp]),
    "spamm_mat_gather_blocks": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "spamm_shard_extend": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, ctypes.POINTER(c_vp)]),
    "spamm_shard_sp2_step": (c_i32, [c_vp, c_vp, c_f64, c_f64, c_i32, c_i64, c_i64, c_vp, c_i32,
                                     ALLREDUCE_FN, c_vp, c_vp, ctypes.POINTER(c_vp),
                                     ctypes.POINTER(c_i32), ctypes.POINTER(c_f64),
                                     ctypes.POINTER(c_f64), ctypes.POINTER(c_f64),
                                     ctypes.POINTER(Stats)]),
    "spamm_tasks": (c_i32, [c_vp, c_vp, c_f64, c_vp, c_vp, c_vp, c_i64, ctypes.POINTER(c_i64), c_vp]),
    "spamm_census_range": (c_i32, [c_vp, c_vp, c_f64, c_i64, c_i64, c_vp, c_vp,
                                   ctypes.POINTER(Stats)]),
    "spamm_tasks_range": (c_i32, [c_vp, c_vp, c_f64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64,
                                  ctypes.POINTER(c_i64), c_vp]),
    "spamm_gemm_batch": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_i32, c_i32,
                                 c_vp]),
    "spamm_add_scaled": (c_i32, [c_f64, c_vp, c_f64, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    "spamm_trace": (c_i32, [c_vp, c_vp, ctypes.POINTER(c_f64)]),
    "spamm_mat_diag_traces": (c_i32, [c_vp, c_vp, c_vp]),
    "spamm_sp2_update": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_vp, ctypes.POINTER(c_f64),
                                 ctypes.POINTER(c_vp)]),
    "spamm_sp2_step": (c_i32, [c_vp, c_f64, c_f64, c_i32, c_i32, c_i32, c_vp, ctypes.POINTER(c_vp),
                               ctypes.POINTER(c_i32), ctypes.POINTER(c_f64),
                               ctypes.POINTER(c_f64), ctypes.POINTER(c_f64),
                               ctypes.POINTER(Stats)]),
    "spamm_sp2_finish": (c_i32, [c_vp, c_vp, c_f64, c_i32, c_vp, ctypes.POINTER(c_i32),
                                 ctypes.POINTER(c_f64), ctypes.POINTER(c_f64),
                                 ctypes.POINTER(c_f64), ctypes.POINTER(c_vp)]),
    "spamm_sp2_solve": (c_i32, [c_vp, c_f64, c_f64, c_i32, c_f64, c_i32, c_f64, c_f64, c_i32,
                                c_i32, c_vp, ctypes.POINTER(c_vp), ctypes.POINTER(SP2Report)]),
    "spamm_sp2_solve_ex": (c_i32, [c_vp, c_f64, c_f64, c_i32, c_f64, c_i32, c_f64, c_f64,
                                   c_i32, c_i32, c_vp, ctypes.POINTER(c_vp),
                                   ctypes.POINTER(SP2Report), ctypes.POINTER(SideCopies)]),
    "spamm_gershgorin": (c_i32, [c_vp, c_vp, ctypes.POINTER(c_f64), ctypes.POINTER(c_f64),
                                 ctypes.POINTER(c_f64)]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load the library (raises OSError with a clear message if absent)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} not found: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.spamm_abi_version() != ABI_VERSION:
            raise OSError("libspamm_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == SPAMM_OK:
        return
    msg = load().spamm_last_error().decode(errors="replace")
    if rc == SPAMM_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"libspamm_b200: {msg}")


def current_stream() -> int:
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1403_7458_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch.cuda.current_stream().cuda_stream
