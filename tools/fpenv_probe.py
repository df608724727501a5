"""Probe host floating-point environment (subnormal handling) for oracle parity."""
import ctypes, subprocess, sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import spamm_oracle as O
a = np.array([1e-310, 3e-300]); print("numpy", a * 0.5, np.float64(1e-160) * np.float64(1e-160))
rng = np.random.default_rng(0)
A = rng.standard_normal((3, 64, 64)) * 1e-160
B = rng.standard_normal((3, 64, 64)) * 1e-155
C = np.zeros((1, 64, 64))
O.gemm_batch(np.array([0, 1, 2]), np.array([0, 1, 2]), np.array([0, 0, 0]), A, B, C, threads=1)
print("gemm checksum", repr(float(np.abs(C).sum())), np.count_nonzero(C), repr(C[0, 0, 0]))
C2 = np.zeros((1, 64, 64))
for t in range(3):
    O.leaf_gemm(A[t], B[t], C2[0])
print("pyloop equal", np.array_equal(C, C2))
