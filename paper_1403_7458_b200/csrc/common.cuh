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
#include <utility>

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

// Programmatic dependent launch (PDL) on the SP2 chain: a kernel launched
// with launch_pdl may be scheduled before its stream predecessor finishes and
// must call pdl_wait() before touching anything the predecessor writes (all
// such kernels call it first thing).  ~2.4 us less per kernel boundary
// (tools/pdl/pdl_bench.cu: 4.1 -> 1.7 us per dependent small kernel).
// SPAMM_PDL=0 launches them plainly.
bool pdl_enabled();
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// launch_plain: a kernel whose stream predecessor is a cudaStreamWaitEvent
// (work of another stream) must not be launched programmatically -- the early
// start would only wait for the last kernel of its own stream.
template <class... KArgs, class... Args>
inline void launch_plain(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                         Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.numAttrs = 0;
  SPAMM_CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}
template <class... KArgs, class... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  SPAMM_CK(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

__host__ __device__ inline int64_t tier_offset(int t) { return ((int64_t(1) << (2 * t)) - 1) / 3; }
__host__ __device__ inline int64_t pyramid_size(int depth) { return tier_offset(depth + 1); }

// Morton code with the row bit above the column bit at each level (bit b of
// i -> bit 2b + 1, bit b of j -> bit 2b), by mask-and-shift bit spreading
// (5 steps instead of a 32-iteration bit loop: these run per C position in
// the cull, the union and the trace kernels).
__host__ __device__ inline uint64_t morton_spread(uint32_t v) {
  uint64_t x = v;
  x = (x | (x << 16)) & 0x0000ffff0000ffffull;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}
__host__ __device__ inline uint32_t morton_compact(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x >> 4)) & 0x00ff00ff00ff00ffull;
  x = (x | (x >> 8)) & 0x0000ffff0000ffffull;
  x = (x | (x >> 16)) & 0x00000000ffffffffull;
  return (uint32_t)x;
}
__host__ __device__ inline uint64_t morton_encode(uint32_t i, uint32_t j) {
  return (morton_spread(i) << 1) | morton_spread(j);
}

__host__ __device__ inline void morton_decode(uint64_t m, uint32_t& i, uint32_t& j) {
  i = morton_compact(m >> 1);
  j = morton_compact(m);
}

inline int grid_for(int64_t n, int threads, int64_t cap = 148LL * 64) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Multi-block chain layout: a 256-element chunk of squares is stored as two
// parity rows (even / odd elements) permuted so each einsum lane's chain
// reads its row sequentially: element e -> row (e & 1), position
// 4 (e >> 3) + 3 - ((e & 7) >> 1).  Rows are CHAIN_ROW doubles apart (16 B
// bank skew), so 8 chains of different blocks load with one conflict-free
// LDS.128 wavefront.  chain_pos(k, lane) is the position of the pair lane
// holds at k (elements k*64 + 2 lane + {0, 1}).
constexpr int CHAIN_ROW = 130;
__device__ __forceinline__ int chain_pos(int k, int lane) {
  return 4 * (k * 8 + (lane >> 2)) + 3 - (lane & 3);
}
__device__ __forceinline__ double chain_row128(const double* row, double l) {
  const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = r2[b * 16 + i];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      l = __dadd_rn(l, v[i].x);
      l = __dadd_rn(l, v[i].y);
    }
  }
  return l;
}

// Exclusive scan of one int64 per thread across the CTA (blockDim.x a
// multiple of 32, <= 1024); *total receives the sum.  Every thread of the
// CTA must call it (it synchronises).
__device__ __forceinline__ int64_t cta_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();  // a previous call may still be reading warp_sums
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int64_t w = lane < nwarps ? warp_sums[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    warp_sums[lane] = wi - w;
    if (lane == 31) warp_sums[32] = wi;
  }
  __syncthreads();
  *total = warp_sums[32];
  return warp_sums[warp] + inc - v;
}

}  // namespace spamm
