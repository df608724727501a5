// Shared helpers for the SpAMM/SP2 sm_100a library.
//
// Layout conventions:
//  * A quadtree matrix with leaf grid side G = 2^depth stores its non-null leaf
//    blocks contiguously, (S, Nb, Nb) float64, row-major inside a block (the
//    reference's _block_data layout, quadtree.py:92), ordered along the Morton
//    (Z) curve of the block coordinates (bi, bj) with the row bit above the
//    column bit at every level -- the order a depth-first quadtree walk visits
//    leaves, so every quadtree node owns a contiguous run of blocks.
//  * keys[s] = bi * G + bj (the reference's int64 key, quadtree.py:91) for the
//    block in storage slot s; slot[bi * G + bj] = s or -1 (null block).
//  * Norm pyramid: one flat float64 buffer, tier t (2^t x 2^t, row-major) at
//    offset (4^t - 1) / 3; both the norms (reference _tier_norms, quadtree.py:93)
//    and their squares (needed to rebuild parents bit-exactly) are kept.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace spamm {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& s) : std::runtime_error(s) {}
};

#define SPAMM_CK(x)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      throw ::spamm::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) +     \
                               " at " + __FILE__ + ":" + std::to_string(__LINE__));      \
  } while (0)

// Every kernel launch of the library goes through this check, which also
// counts launches (spamm_launch_count(): evidence for bench.py's gpu_launches).
extern std::atomic<long long> g_launch_count;
#define SPAMM_LAUNCH_CK()                                          \
  do {                                                             \
    SPAMM_CK(cudaGetLastError());                                  \
    ::spamm::g_launch_count.fetch_add(1, std::memory_order_relaxed); \
  } while (0)

__host__ __device__ inline int64_t tier_offset(int t) { return ((int64_t(1) << (2 * t)) - 1) / 3; }
__host__ __device__ inline int64_t pyramid_size(int depth) { return tier_offset(depth + 1); }

// Morton code with the row bit above the column bit at each level.
__host__ __device__ inline uint64_t morton_encode(uint32_t i, uint32_t j) {
  uint64_t m = 0;
  for (int b = 0; b < 32; ++b) {
    m |= (uint64_t)((i >> b) & 1u) << (2 * b + 1);
    m |= (uint64_t)((j >> b) & 1u) << (2 * b);
  }
  return m;
}

__host__ __device__ inline void morton_decode(uint64_t m, uint32_t& i, uint32_t& j) {
  i = 0;
  j = 0;
  for (int b = 0; b < 32; ++b) {
    i |= (uint32_t)((m >> (2 * b + 1)) & 1u) << b;
    j |= (uint32_t)((m >> (2 * b)) & 1u) << b;
  }
}

inline int grid_for(int64_t n, int threads, int64_t cap = 148LL * 64) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

}  // namespace spamm
