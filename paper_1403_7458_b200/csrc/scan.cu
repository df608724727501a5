// Device-wide exclusive prefix sum (reduce-then-scan, deterministic).
// Used for stream compaction of surviving (C node, k) candidates in the cull
// (the ballot/prefix-scan compaction of DESIGN.md K2) and for block pruning.
#include "internal.h"

namespace spamm {

namespace {

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <class T>
__device__ inline int64_t as_i64(T v) { return (int64_t)v; }

// Block-wide exclusive scan of one int64 per thread; returns the block total.
__device__ inline int64_t block_exclusive_scan(int64_t v, int64_t& excl) {
  constexpr int NW = SCAN_THREADS / 32;
  __shared__ int64_t wsum[NW];
  __shared__ int64_t btot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < NW ? wsum[lane] : 0;
    int64_t z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < NW) wsum[lane] = z - w;
    if (lane == NW - 1) btot = z;
  }
  __syncthreads();
  excl = wsum[warp] + x - v;
  const int64_t total = btot;
  __syncthreads();
  return total;
}

template <class T>
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_sums(const T* in, int64_t n, int64_t* sums) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t acc = 0;
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    int64_t i = base + (int64_t)r * SCAN_THREADS + threadIdx.x;
    if (i < n) acc += as_i64(in[i]);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  __shared__ int64_t ws[SCAN_THREADS / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < SCAN_THREADS / 32; ++w) t += ws[w];
    sums[blockIdx.x] = t;
  }
}

// Each thread owns SCAN_ITEMS consecutive elements of the tile.
template <class T>
__global__ void __launch_bounds__(SCAN_THREADS)
    k_tile_scan(const T* in, int64_t n, const int64_t* tile_off, int64_t* out) {
  pdl_wait();
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS];
  int64_t sum = 0;
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    int64_t i = base + r;
    v[r] = i < n ? as_i64(in[i]) : 0;
    sum += v[r];
  }
  int64_t excl;
  int64_t total = block_exclusive_scan(sum, excl);
  const int64_t off = (tile_off ? tile_off[blockIdx.x] : 0) + excl;
  int64_t run = off;
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    int64_t i = base + r;
    if (i < n) out[i] = run;
    run += v[r];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
    out[n] = (tile_off ? tile_off[blockIdx.x] : 0) + total;
}

template <class T>
void scan_impl(const T* in, int64_t n, int64_t* out, cudaStream_t s) {
  if (n <= 0) {
    SPAMM_CK(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
    return;
  }
  const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    launch_pdl(k_tile_scan<T>, 1, SCAN_THREADS, 0, s, in, n, nullptr, out);
    SPAMM_LAUNCH_CK();
    return;
  }
  int64_t* sums = dmalloc<int64_t>(tiles, s);
  int64_t* offs = dmalloc<int64_t>(tiles + 1, s);
  k_tile_sums<T><<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, n, sums);
  SPAMM_LAUNCH_CK();
  scan_impl<int64_t>(sums, tiles, offs, s);
  launch_pdl(k_tile_scan<T>, (unsigned)tiles, SCAN_THREADS, 0, s, in, n, offs, out);
  SPAMM_LAUNCH_CK();
  dfree(sums, s);
  dfree(offs, s);
}

}  // namespace

void scan_exclusive_u8(const uint8_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  scan_impl<uint8_t>(in, n, out, s);
}
void scan_exclusive_i64(const int64_t* in, int64_t n, int64_t* out, cudaStream_t s) {
  scan_impl<int64_t>(in, n, out, s);
}

}  // namespace spamm
