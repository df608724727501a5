"""B200-native SpAMM / SP2 hot path (drop-in for the reference ``spamm`` package).

Same names and signatures as the reference's hot-path API
(``/root/reference/pkg/src/spamm/__init__.py:9-23``): quadtree storage,
``multiply`` / ``convolution_census`` / ``leaf_gemm``, and the SP2 driver.
All compute runs in ``libspamm_b200.so`` (sm_100a CUDA, C ABI in
``include/spamm_b200.h``); there is no CPU fallback.
"""

from .quadtree import (QuadTreeMatrix, Node, build_from_dense, to_dense, to_dense_device,
                       verify_norms, add_scaled, trace, identity)
from .kernel import (ProductStats, multiply, convolution_census, leaf_gemm, gemm_batch,
                     leaf_tasks, set_symmetric_products, set_dense_cull, set_near_tau_ulps,
                     WORKERS_ENV_VAR)
from .sp2 import (SpectralBounds, SP2State, gershgorin_bounds, sp2_init, sp2_step, sp2_solve,
                  energy_error, idempotency_error, SQUARE, EXPAND)
from ._native import LIB_PATH, load as load_library

__version__ = "0.1.0"

__all__ = [
    "QuadTreeMatrix", "Node", "build_from_dense", "to_dense", "to_dense_device",
    "verify_norms", "add_scaled", "trace", "identity",
    "ProductStats", "multiply", "convolution_census", "leaf_gemm", "gemm_batch", "leaf_tasks",
    "set_symmetric_products",
    "set_dense_cull",
    "set_near_tau_ulps",
    "WORKERS_ENV_VAR",
    "SpectralBounds", "SP2State", "gershgorin_bounds", "sp2_init", "sp2_step", "sp2_solve",
    "energy_error", "idempotency_error", "SQUARE", "EXPAND",
    "LIB_PATH", "load_library", "__version__",
]
