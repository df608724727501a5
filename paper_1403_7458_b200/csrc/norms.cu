#include <chrono>
#include <map>
#include <string>
// K1: bit-exact Frobenius-norm pyramid + storage finalisation.
//
// Reference: QuadTreeMatrix._from_blocks, quadtree.py:170-194.
//  * leaf norm^2 = np.einsum("tij,tij->t") (quadtree.py:186-187).  numpy (SSE2
//    build baseline) evaluates it as two lanes (even / odd element), each an
//    unfused acc += x*x walking 8-element chunks in pair order
//    (6,7),(4,5),(2,3),(0,1), then lane0 + lane1.  Restated here with explicit
//    __dmul_rn/__dadd_rn so nvcc cannot contract to FMA.
//  * parents: reshape(h,2,h,2).sum(axis=(1,3)) == (c00 + c01) + (c10 + c11)
//    in the squared domain (quadtree.py:191) for h >= 2; for the root (h = 1)
//    numpy coalesces the 2x2 into one contiguous run and sums sequentially,
//    ((c00 + c01) + c10) + c11; sqrt per tier (quadtree.py:188,192).
//  * blocks whose entries are all exactly zero are pruned (quadtree.py:177-180).
// HBM roofline: S*Nb^2*8 bytes read per pass; K1.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"
#include "ozaki_common.cuh"

namespace spamm {

// ------------------------------------------------------------------ memory
namespace {
std::once_flag g_pool_once;
void init_pool() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}
}  // namespace

void* dmalloc_bytes(size_t bytes, cudaStream_t s) {
  std::call_once(g_pool_once, init_pool);
  if (bytes == 0) return nullptr;
  void* p = nullptr;
  SPAMM_CK(cudaMallocAsync(&p, bytes, s));
  return p;
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

void reserve_pool(size_t bytes, cudaStream_t s) {
  // Grow the stream-ordered pool once (release threshold is unlimited, so the
  // pages stay mapped): later cudaMallocAsync calls never block on a mapping.
  void* p = dmalloc_bytes(bytes, s);
  dfree(p, s);
  SPAMM_CK(cudaStreamSynchronize(s));
}

// Host wait for the stream: polls cudaStreamQuery (about 10 us less wake-up
// latency per wait than a blocking synchronize, ~0.5 ms per cfg4 SP2 solve);
// SPAMM_WAIT=block selects cudaStreamSynchronize.
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("SPAMM_PDL");
    return !(v && strcmp(v, "0") == 0);
  }();
  return on;
}

bool wait_blocking() {
  static const bool block = [] {
    const char* v = getenv("SPAMM_WAIT");
    return v && strcmp(v, "block") == 0;
  }();
  return block;
}

void stream_wait(cudaStream_t s) {
  if (wait_blocking()) {
    SPAMM_CK(cudaStreamSynchronize(s));
    return;
  }
  for (;;) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) SPAMM_CK(e);
  }
}

void event_wait(cudaEvent_t e) {
  for (;;) {
    const cudaError_t r = cudaEventQuery(e);
    if (r == cudaSuccess) return;
    if (r != cudaErrorNotReady) SPAMM_CK(r);
  }
}

namespace {
struct HMark {
  const char* label;
  std::chrono::steady_clock::time_point t;
};
thread_local std::vector<HMark> g_hmarks;
bool htrace_on() {
  static const bool on = [] {
    const char* v = getenv("SPAMM_HTRACE");
    return v && *v && strcmp(v, "0") != 0;
  }();
  return on;
}
}  // namespace

void htrace(const char* label) {
  if (htrace_on()) g_hmarks.push_back({label, std::chrono::steady_clock::now()});
}

void htrace_dump() {
  if (!htrace_on() || g_hmarks.size() < 2) return;
  std::map<std::pair<std::string, std::string>, std::pair<long, double>> agg;
  for (size_t i = 1; i < g_hmarks.size(); ++i) {
    auto& a = agg[{g_hmarks[i - 1].label, g_hmarks[i].label}];
    a.first += 1;
    a.second += std::chrono::duration<double, std::micro>(g_hmarks[i].t - g_hmarks[i - 1].t).count();
  }
  fprintf(stderr, "[htrace] %zu marks\n", g_hmarks.size());
  for (auto& [k, v] : agg)
    fprintf(stderr, "[htrace] %-14s -> %-14s n=%5ld mean %8.2f us total %9.1f us\n",
            k.first.c_str(), k.second.c_str(), v.first, v.second / v.first, v.second);
  g_hmarks.clear();
}

// Writes the scalars, then (after a system-scope fence) the sequence number
// the host spins on: the host sees completion as soon as the PCIe writes land,
// without a driver round trip per poll.
__global__ void k_gather_scalars(ScalarSrc src, int n, int64_t* dst, int64_t* flag, int64_t seq) {
  pdl_wait();
  const int i = threadIdx.x;
  if (i < n) dst[i] = src.p[i] ? *src.p[i] : 0;
  __threadfence_system();
  __syncthreads();
  if (i == 0) *reinterpret_cast<volatile int64_t*>(flag) = seq;
}

int64_t* pinned_scalars() {
  static thread_local int64_t* pinned = nullptr;
  if (!pinned) SPAMM_CK(cudaMallocHost(&pinned, (32 + GATHER_MAX + 8) * sizeof(int64_t)));
  return pinned;
}

PinnedGather pinned_gather_begin() {
  static thread_local int64_t seq = 0;
  PinnedGather g;
  g.vals = pinned_scalars() + 32;  // values [32, 96), sequence flag [96]
  g.flag = pinned_scalars() + 32 + GATHER_MAX;
  g.seq = ++seq;
  return g;
}

void pinned_gather_wait(int64_t* host, int n, const PinnedGather& g, cudaStream_t s) {
  htrace("gs_wait");
  const volatile int64_t* flag = g.flag;
  if (wait_blocking()) {
    stream_wait(s);
  } else {
    // spin on the flag; every 4096 polls ask the driver (surfaces a failed
    // kernel, and ends the wait if the stream completed)
    for (unsigned spins = 1; *flag != g.seq; ++spins) {
      if ((spins & 4095u) == 0) {
        const cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) SPAMM_CK(e);
      }
    }
  }
  htrace("gs_done");
  for (int i = 0; i < n; ++i) host[i] = g.vals[i];
}

void gather_sync(int64_t* host, const int64_t* const* src, int n, cudaStream_t s) {
  if (n > GATHER_MAX) throw CudaError("gather_sync: too many scalars");
  ScalarSrc ss{};
  for (int i = 0; i < n; ++i) ss.p[i] = src[i];
  const PinnedGather g = pinned_gather_begin();
  launch_pdl(k_gather_scalars, 1, 64, 0, s, ss, n, g.vals, g.flag, g.seq);
  SPAMM_LAUNCH_CK();
  pinned_gather_wait(host, n, g, s);
}

__global__ void k_copy_f64(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Small device -> pinned host copies by kernel stores (see d2h_sync).
void copy_to_pinned(double* host, const double* dev, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  k_copy_f64<<<grid_for(n, 256, 148), 256, 0, s>>>(host, dev, n);
  SPAMM_LAUNCH_CK();
}

// (a kernel store to pinned memory, not cudaMemcpyAsync: a small D2H memcpy
// queues behind any bulk D2H on the copy engines -- ~0.8 ms instead of ~20 us
// while pipeline.py downloads a density matrix)
void d2h_sync(int64_t* host, const int64_t* dev, int n, cudaStream_t s) {
  if (n > 32) throw CudaError("d2h_sync: too many scalars");
  const int64_t* src[32];
  for (int i = 0; i < n; ++i) src[i] = dev + i;
  gather_sync(host, src, n, s);
}

namespace {
// Fixed-size pinned buffers + events for the host norm mirrors (allocation
// of pinned memory and events is slow; matrices come and go every SP2 step).
std::mutex g_top_mu;
std::vector<double*> g_top_bufs;
std::vector<cudaEvent_t> g_top_evs;

void top_acquire(double** buf, cudaEvent_t* ev) {
  std::lock_guard<std::mutex> lk(g_top_mu);
  if (g_top_bufs.empty()) {
    double* b = nullptr;
    SPAMM_CK(cudaMallocHost(&b, tier_offset(HOST_TOP_TIERS + 1) * sizeof(double)));
    g_top_bufs.push_back(b);
  }
  if (g_top_evs.empty()) {
    cudaEvent_t e;
    SPAMM_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    g_top_evs.push_back(e);
  }
  *buf = g_top_bufs.back();
  g_top_bufs.pop_back();
  *ev = g_top_evs.back();
  g_top_evs.pop_back();
}

void top_release(double* buf, cudaEvent_t ev) {
  // the async copy must not land in a reused buffer (long done in practice:
  // a query is enough then)
  if (ev && cudaEventQuery(ev) != cudaSuccess) cudaEventSynchronize(ev);
  std::lock_guard<std::mutex> lk(g_top_mu);
  if (buf) g_top_bufs.push_back(buf);
  if (ev) g_top_evs.push_back(ev);
}
}  // namespace

void Mat::release() {
  dfree(tr_dev, stream);
  tr_dev = nullptr;
  dfree(oz_ex_row, stream);
  dfree(oz_ex_col, stream);
  oz_ex_row = oz_ex_col = nullptr;
  dfree(pend_nz, stream);
  dfree(pend_off, stream);
  dfree(pend_kept, stream);
  pend_nz = nullptr;
  pend_off = nullptr;
  pend_kept = nullptr;
  top_release(host_top, top_ev);
  host_top = nullptr;
  top_ev = nullptr;
  top_t = -1;
  cudaStream_t s = stream;
  dfree(data, s);
  dfree(keys, s);
  dfree(slot, s);
  dfree(norms, s);
  dfree(norms2, s);
  data = nullptr;
  keys = nullptr;
  slot = nullptr;
  norms = nullptr;
  norms2 = nullptr;
  nblocks = 0;
}

// ------------------------------------------------------------------ kernels
namespace {

__device__ __forceinline__ void sq_acc(double& l, double x) { l = __dadd_rn(l, __dmul_rn(x, x)); }

// One thread per block; the two einsum lanes are independent chains (ILP 2).
template <int NB2>
__global__ void __launch_bounds__(128)
    k_leaf_norms2(const double* __restrict__ data, int64_t m, int nb2_rt, double* __restrict__ out,
                  uint8_t* __restrict__ nz) {
  const int nb2 = NB2 ? NB2 : nb2_rt;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < m;
       b += (int64_t)gridDim.x * blockDim.x) {
    const double* x = data + b * nb2;
    double l0 = 0.0, l1 = 0.0;
    bool any = false;
    int i = 0;
    if (nb2 >= 8) {
      const double2* x2 = reinterpret_cast<const double2*>(x);
#pragma unroll 4
      for (; nb2 - i >= 8; i += 8) {
        const double2 v0 = __ldg(x2 + i / 2), v1 = __ldg(x2 + i / 2 + 1);
        const double2 v2 = __ldg(x2 + i / 2 + 2), v3 = __ldg(x2 + i / 2 + 3);
        sq_acc(l0, v3.x);
        sq_acc(l1, v3.y);
        sq_acc(l0, v2.x);
        sq_acc(l1, v2.y);
        sq_acc(l0, v1.x);
        sq_acc(l1, v1.y);
        sq_acc(l0, v0.x);
        sq_acc(l1, v0.y);
        any |= (v0.x != 0.0) | (v0.y != 0.0) | (v1.x != 0.0) | (v1.y != 0.0) | (v2.x != 0.0) |
               (v2.y != 0.0) | (v3.x != 0.0) | (v3.y != 0.0);
      }
    }
    for (; i < nb2; i += 2) {
      const double a = x[i];
      sq_acc(l0, a);
      any |= a != 0.0;
      if (i + 1 < nb2) {
        const double c = x[i + 1];
        sq_acc(l1, c);
        any |= c != 0.0;
      }
    }
    out[b] = __dadd_rn(l0, l1);
    if (nz) nz[b] = any ? 1 : 0;
  }
}

__global__ void k_scatter_leaf(const int64_t* __restrict__ keys, const double* __restrict__ n2,
                               int64_t m, double* __restrict__ leaf2, double* __restrict__ leafn) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = keys[i];
    const double v = n2[i];
    leaf2[k] = v;
    leafn[k] = __dsqrt_rn(v);
  }
}

// Tier t from tier t+1 (both row-major), squared domain, then sqrt.
__global__ void k_tier_up(const double* __restrict__ c2, double* __restrict__ p2,
                          double* __restrict__ pn, int t) {
  const int64_t w = int64_t(1) << t, W = 2 * w, n = w * w;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / w, j = idx % w;
    const double* r0 = c2 + (2 * i) * W + 2 * j;
    const double* r1 = r0 + W;
    const double s = __dadd_rn(__dadd_rn(r0[0], r0[1]), __dadd_rn(r1[0], r1[1]));
    p2[idx] = s;
    pn[idx] = __dsqrt_rn(s);
  }
}

// Tiers t_top..0 in one CTA (small tiers: <= 1024 parents).
__global__ void k_tiers_small(double* __restrict__ norms2, double* __restrict__ norms, int t_top) {
  for (int t = t_top; t >= 0; --t) {
    const int64_t w = int64_t(1) << t, W = 2 * w, n = w * w;
    const double* c2 = norms2 + tier_offset(t + 1);
    double* p2 = norms2 + tier_offset(t);
    double* pn = norms + tier_offset(t);
    for (int64_t idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int64_t i = idx / w, j = idx % w;
      const double* r0 = c2 + (2 * i) * W + 2 * j;
      const double* r1 = r0 + W;
      // root (t = 0): numpy coalesces the 2x2 into one run of 4 -> sequential
      const double s = t == 0 ? __dadd_rn(__dadd_rn(__dadd_rn(r0[0], r0[1]), r1[0]), r1[1])
                              : __dadd_rn(__dadd_rn(r0[0], r0[1]), __dadd_rn(r1[0], r1[1]));
      p2[idx] = s;
      pn[idx] = __dsqrt_rn(s);
    }
    __syncthreads();
  }
}

// Finalisation for small trees (G*G <= 16384): the kept-block count, slot
// map, leaf tier, upper tiers (same sums as k_tier_up / k_tiers_small), the
// trace (same order as k_trace_blocks + k_trace, Nb >= 2), the pinned host
// mirror of the top tiers and, for X^2 in SP2, the idempotency residual root
// and the key union with X -- one launch of four independent CTAs instead of
// ~12 small launches (the kernel is a chain of dependent memory round trips,
// so the jobs run side by side and each CTA issues a phase's loads together):
//   CTA 0: slot map, leaf tier and pyramid (squared pyramid in shared
//          memory), kept count, host mirror;
//   CTA 1: the D = X^2 - X pyramid (X's leaf norm^2 everywhere, overwritten
//          by the fused D chains at X^2's blocks) -> root norm;
//   CTA 2: trace (diagonal blocks found from the keys);
//   CTA 3: the key union (X^2's blocks flagged from its keys, X's from its
//          slot map).
// Each thread owns FS_PER positions / blocks.  Any output may be null.
constexpr int FS_THREADS = 1024;
constexpr int FS_BATCH = 4;  // global loads issued together per thread

__device__ __forceinline__ void fs_tiers(double* p2, double* norms, double* norms2, int depth) {
  const int tid = threadIdx.x;
  for (int t = depth - 1; t >= 0; --t) {
    const int w = 1 << t, W = 2 * w, n = w * w;
    const int64_t co = tier_offset(t + 1), po = tier_offset(t);
    for (int idx = tid; idx < n; idx += FS_THREADS) {
      const int i = idx >> t, j = idx & (w - 1);
      const double* r0 = p2 + co + (2 * i) * W + 2 * j;
      const double* r1 = r0 + W;
      // root (t = 0): numpy coalesces the 2x2 into one run of 4 -> sequential
      const double sm = t == 0 ? __dadd_rn(__dadd_rn(__dadd_rn(r0[0], r0[1]), r1[0]), r1[1])
                               : __dadd_rn(__dadd_rn(r0[0], r0[1]), __dadd_rn(r1[0], r1[1]));
      p2[po + idx] = sm;
      if (norms2) norms2[po + idx] = sm;
      if (norms) norms[po + idx] = __dsqrt_rn(sm);
    }
    __syncthreads();
  }
}

template <int FS_PER>
__global__ void __launch_bounds__(FS_THREADS)
    k_finalize_small(const int64_t* __restrict__ keys, const double* __restrict__ n2,
                     const double* __restrict__ n1, const uint8_t* __restrict__ nz,
                     int64_t nblocks, int depth, int64_t* __restrict__ kept,
                     int32_t* __restrict__ slot, double* __restrict__ norms,
                     double* __restrict__ norms2, const double* __restrict__ data, int nb,
                     double* __restrict__ tr_out, double* host_top, int top_t,
                     const double* __restrict__ dn2, const double* __restrict__ xleaf2,
                     double* __restrict__ idem_out, const int32_t* __restrict__ xslot = nullptr,
                     int64_t* __restrict__ ukeys = nullptr, int64_t* __restrict__ ucount = nullptr,
                     double* __restrict__ dleaf = nullptr) {
  pdl_wait();
  extern __shared__ __align__(16) double p2[];  // squared pyramid, tiers 0..depth
  __shared__ int32_t dslot[128];
  __shared__ double part[128];
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int tid = threadIdx.x;
  const int64_t leaf_off = tier_offset(depth);

  // (each CTA issues all its global loads of a phase before using any of
  // them: the kernel is latency-bound, one CTA per job)
  if (blockIdx.x == 0) {
    // ---- slot map, leaf tier, pyramid, kept count, host mirror ----
    __shared__ int kept_sh;
    if (tid == 0) kept_sh = 0;
    int cnt = 0;
#pragma unroll
    for (int j = 0; j < FS_PER; ++j) {
      const int64_t b = (int64_t)j * FS_THREADS + tid;
      cnt += b < nblocks && kept && nz ? (int)nz[b] : 0;
    }
#pragma unroll
    for (int j = 0; j < FS_PER; ++j) {
      const int64_t p = (int64_t)j * FS_THREADS + tid;
      if (p < npos) {
        p2[leaf_off + p] = 0.0;
        norms2[leaf_off + p] = 0.0;
        norms[leaf_off + p] = 0.0;
        if (slot) slot[p] = -1;
      }
    }
    __syncthreads();  // zero fill before the scatter; kept_sh initialised
    if (kept) {
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if ((tid & 31) == 0 && cnt) atomicAdd(&kept_sh, cnt);
    }
#pragma unroll
    for (int j0 = 0; j0 < FS_PER; j0 += FS_BATCH) {
      int64_t kk[FS_BATCH];
      double vv[FS_BATCH], ww[FS_BATCH];
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t b = (int64_t)(j0 + u) * FS_THREADS + tid;
        const bool in = b < nblocks;
        kk[u] = in ? keys[b] : -1;
        vv[u] = in ? n2[b] : 0.0;
        ww[u] = in && n1 ? n1[b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t k = kk[u];
        if (k < 0) continue;
        p2[leaf_off + k] = vv[u];
        norms2[leaf_off + k] = vv[u];
        norms[leaf_off + k] = n1 ? ww[u] : __dsqrt_rn(vv[u]);
        if (slot) slot[k] = (int32_t)((int64_t)(j0 + u) * FS_THREADS + tid);
      }
    }
    __syncthreads();
    if (kept && tid == 0) *kept = kept_sh;
    fs_tiers(p2, norms, norms2, depth);
    if (host_top) {
      for (int64_t i = tid; i < tier_offset(top_t + 1); i += FS_THREADS)
        host_top[i] = __dsqrt_rn(p2[i]);
    }
  } else if (blockIdx.x == 1) {
    // ---- D = add_scaled(1, X^2, -1, X): root norm ----
    if (!idem_out) return;
#pragma unroll
    for (int j0 = 0; j0 < FS_PER; j0 += FS_BATCH) {
      double xv[FS_BATCH];
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t p = (int64_t)(j0 + u) * FS_THREADS + tid;
        // X-only blocks: (-x)^2 == x^2 -- only blocks this matrix stores (a
        // multi-GPU shard carries the whole matrix's pyramid)
        xv[u] = xleaf2 && p < npos && (!xslot || xslot[p] >= 0) ? xleaf2[p] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t p = (int64_t)(j0 + u) * FS_THREADS + tid;
        if (p < npos) p2[leaf_off + p] = xv[u];
      }
    }
    __syncthreads();
#pragma unroll
    for (int j0 = 0; j0 < FS_PER; j0 += FS_BATCH) {
      int64_t kk[FS_BATCH];
      double dv[FS_BATCH];
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t b = (int64_t)(j0 + u) * FS_THREADS + tid;
        kk[u] = b < nblocks ? keys[b] : -1;
        dv[u] = b < nblocks ? dn2[b] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u)
        if (kk[u] >= 0) p2[leaf_off + kk[u]] = dv[u];
    }
    __syncthreads();
    if (dleaf) {  // the leaf tier of ||X^2 - X||^2 (multi-GPU: all-reduced by the caller)
#pragma unroll 4
      for (int j = 0; j < FS_PER; ++j) {
        const int64_t p = (int64_t)j * FS_THREADS + tid;
        if (p < npos) dleaf[p] = p2[leaf_off + p];
      }
    }
    fs_tiers(p2, nullptr, nullptr, depth);
    if (tid == 0) *idem_out = __dsqrt_rn(p2[0]);
  } else if (blockIdx.x == 2) {
    // ---- trace: diagonal blocks found from the keys ----
    if (!tr_out) return;
    if (tid < 128) dslot[tid] = -1;
    __syncthreads();
#pragma unroll
    for (int j0 = 0; j0 < FS_PER; j0 += FS_BATCH) {
      int64_t kk[FS_BATCH];
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t b = (int64_t)(j0 + u) * FS_THREADS + tid;
        kk[u] = b < nblocks ? keys[b] : -1;
      }
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t k = kk[u];
        if (k >= 0 && (k >> depth) == (k & (G - 1)))
          dslot[k & (G - 1)] = (int32_t)((int64_t)(j0 + u) * FS_THREADS + tid);
      }
    }
    __syncthreads();
    // stage the diagonals of the G diagonal blocks, then one thread per
    // block sums its diagonal in order, thread 0 the blocks in order
    double* dg = p2;
    const int64_t nb2 = (int64_t)nb * nb, nd = G * nb;
    constexpr int DQ = 4;  // loads in flight per thread
    for (int64_t q0 = tid; q0 < nd; q0 += (int64_t)DQ * FS_THREADS) {
      double v[DQ];
#pragma unroll
      for (int u = 0; u < DQ; ++u) {
        const int64_t q = q0 + (int64_t)u * FS_THREADS;
        const int64_t b = q / nb, d = q % nb;
        const int32_t sl = q < nd ? dslot[b] : -1;
        v[u] = sl >= 0 ? data[(int64_t)sl * nb2 + d * nb + d] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < DQ; ++u) {
        const int64_t q = q0 + (int64_t)u * FS_THREADS;
        if (q < nd) dg[q] = v[u];
      }
    }
    __syncthreads();
    // (sequential sums; the operands are read 16 at a time ahead of the adds)
    if (tid < G && dslot[tid] >= 0) {
      const double* x = dg + (int64_t)tid * nb;
      double acc = 0.0;
      for (int d0 = 0; d0 < nb; d0 += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = d0 + u < nb ? x[d0 + u] : 0.0;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (d0 + u < nb) acc = __dadd_rn(acc, v[u]);
      }
      part[tid] = acc;
    }
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int64_t b0 = 0; b0 < G; b0 += 16) {
        double v[16];
        bool in[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          in[u] = b0 + u < G && dslot[b0 + u] >= 0;
          v[u] = in[u] ? part[b0 + u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (in[u]) tot = __dadd_rn(tot, v[u]);
      }
      *tr_out = tot;
    }
  } else {
    // ---- key union of X and X^2 in Morton order ----
    if (!ukeys) return;
    uint8_t* cflag = reinterpret_cast<uint8_t*>(p2);
#pragma unroll 4
    for (int j = 0; j < FS_PER; ++j) {
      const int64_t p = (int64_t)j * FS_THREADS + tid;
      if (p < npos) cflag[p] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int j0 = 0; j0 < FS_PER; j0 += FS_BATCH) {
      int64_t kk[FS_BATCH];
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t b = (int64_t)(j0 + u) * FS_THREADS + tid;
        kk[u] = b < nblocks ? keys[b] : -1;
      }
#pragma unroll
      for (int u = 0; u < FS_BATCH; ++u) {
        const int64_t k = kk[u];
        if (k >= 0) cflag[morton_encode((uint32_t)(k >> depth), (uint32_t)(k & (G - 1)))] = 1;
      }
    }
    __syncthreads();
    // FS_PER consecutive positions per thread: count, scan, write
    int fs = 0;
    bool in_u[FS_PER];
#pragma unroll
    for (int j = 0; j < FS_PER; ++j) {
      const int64_t p = (int64_t)tid * FS_PER + j;
      uint32_t bi, bj;
      morton_decode((uint64_t)p, bi, bj);
      in_u[j] = p < npos && (xslot[(int64_t)bi * G + bj] >= 0 || cflag[p]);
      fs += in_u[j] ? 1 : 0;
    }
    int64_t tot = 0;
    int64_t o = cta_exclusive_scan(fs, &tot);
#pragma unroll
    for (int j = 0; j < FS_PER; ++j) {
      const int64_t p = (int64_t)tid * FS_PER + j;
      uint32_t bi, bj;
      morton_decode((uint64_t)p, bi, bj);
      if (in_u[j]) ukeys[o++] = (int64_t)bi * G + bj;
    }
    if (tid == 0) *ucount = tot;
  }
}

template <class... Args>
void launch_finalize_small(int depth, int nb, cudaStream_t s, Args... args) {
  // the larger of the squared pyramid and (diagonal staging + union flags)
  const int64_t G = int64_t(1) << depth;
  const size_t smem = std::max((size_t)pyramid_size(depth) * sizeof(double),
                               (size_t)(G * nb) * sizeof(double) + (size_t)(G * G) + 64);
  if (smem > 220 * 1024) throw CudaError("finalize: shared memory budget exceeded");
  if (depth <= 6 && smem <= 48 * 1024) {
    launch_pdl(k_finalize_small<4>, 4, FS_THREADS, smem, s, args...);
  } else {
    static std::once_flag once;
    std::call_once(once, [] {
      SPAMM_CK(cudaFuncSetAttribute(k_finalize_small<16>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    });
    launch_pdl(k_finalize_small<16>, 4, FS_THREADS, smem, s, args...);
  }
  SPAMM_LAUNCH_CK();
}

// Gather the kept blocks (nz[b] = 1) to their compacted positions.
__global__ void k_compact_blocks(const double* __restrict__ din, const int64_t* __restrict__ kin,
                                 const double* __restrict__ nin, const uint8_t* __restrict__ nz,
                                 const int64_t* __restrict__ off, int64_t m, int nb2,
                                 double* __restrict__ dout, int64_t* __restrict__ kout,
                                 double* __restrict__ nout) {
  for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
    if (!nz[b]) continue;
    const int64_t d = off[b];
    for (int e = threadIdx.x; e < nb2; e += blockDim.x) dout[d * nb2 + e] = din[b * nb2 + e];
    if (threadIdx.x == 0) {
      kout[d] = kin[b];
      if (nout) nout[d] = nin[b];
    }
  }
}

__global__ void k_scatter_slots(const int64_t* __restrict__ keys, int64_t m, int32_t* __restrict__ slot) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    slot[keys[i]] = (int32_t)i;
}

}  // namespace

// Multi-block variant (the production path for Nb = 32 / 64): each warp
// reduces BPW blocks at once, chains of all of them on lanes 0 .. 2 BPW - 1
// reading the permuted parity rows (common.cuh) with LDS.128.  Same recipe and
// bits as k_leaf_norms2 (an earlier one-block-per-warp form, lanes 0/1
// chaining from LDS.64, was bound by shared-load wavefronts: L1 83 %).
template <int NB2, int BPW, int WARPS>
__global__ void __launch_bounds__(32 * WARPS)
    k_leaf_norms2_multi(const double* __restrict__ data, int64_t m, double* __restrict__ out,
                        uint8_t* __restrict__ nz, double* __restrict__ out1 = nullptr) {
  constexpr int NCH = NB2 / 256;
  __shared__ __align__(16) double rows_all[WARPS][BPW * 2 * CHAIN_ROW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* rows = rows_all[warp];
  const int64_t stride = (int64_t)gridDim.x * WARPS * BPW;
  for (int64_t b0 = ((int64_t)blockIdx.x * WARPS + warp) * BPW; b0 < m; b0 += stride) {
    const double2* x[BPW];
    double2 r[BPW][4];
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      x[q] = b0 + q < m ? reinterpret_cast<const double2*>(data + (b0 + q) * NB2) : nullptr;
#pragma unroll
      for (int k = 0; k < 4; ++k) r[q][k] = x[q] ? __ldg(x[q] + k * 32 + lane) : make_double2(0.0, 0.0);
    }
    double acc = 0.0;
    unsigned anyq = 0;
    for (int c = 0; c < NCH; ++c) {
      __syncwarp();
#pragma unroll
      for (int q = 0; q < BPW; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double* rq = rows + q * 2 * CHAIN_ROW + chain_pos(k, lane);
          rq[0] = __dmul_rn(r[q][k].x, r[q][k].x);
          rq[CHAIN_ROW] = __dmul_rn(r[q][k].y, r[q][k].y);
          if ((r[q][k].x != 0.0) | (r[q][k].y != 0.0)) anyq |= 1u << q;
        }
      __syncwarp();
      if (c + 1 < NCH) {
#pragma unroll
        for (int q = 0; q < BPW; ++q)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (x[q]) r[q][k] = __ldg(x[q] + (c + 1) * 128 + k * 32 + lane);
      }
      if (lane < 2 * BPW) acc = chain_row128(rows + lane * CHAIN_ROW, acc);
    }
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      const double l0 = __shfl_sync(0xffffffffu, acc, 2 * q);
      const double l1 = __shfl_sync(0xffffffffu, acc, 2 * q + 1);
      const bool any = __any_sync(0xffffffffu, (anyq >> q) & 1u);
      if (lane == 0 && b0 + q < m) {
        const double v = __dadd_rn(l0, l1);
        out[b0 + q] = v;
        if (out1) out1[b0 + q] = __dsqrt_rn(v);
        if (nz) nz[b0 + q] = any ? 1 : 0;
      }
    }
  }
}

// K1 for C = X*X with the idempotency residual fused in: besides C's leaf
// norm^2 it chains D = fl(c - x) (= add_scaled(1, C, -1, X) blockwise; x = 0
// where X has no block, which leaves c unchanged) for every C block.  Lanes
// 4q + 2 set + parity: set 0 = C chain, set 1 = D chain (BPW = 2 -> 8 rows,
// one LDS.128 wavefront).
template <int NB2, int WARPS>
__global__ void __launch_bounds__(32 * WARPS)
    k_leaf_norms2_cd(const double* __restrict__ data, const int64_t* __restrict__ keys,
                     int64_t m, const double* __restrict__ xdata,
                     const int32_t* __restrict__ xslot, double* __restrict__ out,
                     uint8_t* __restrict__ nz, double* __restrict__ dout,
                     double* __restrict__ out1, int* __restrict__ ex_col, int64_t G) {
  pdl_wait();
  constexpr int NCH = NB2 / 256, BPW = 2;
  constexpr int NB = NB2 == 4096 ? 64 : 32;
  __shared__ __align__(16) double rows_all[WARPS][BPW * 4 * CHAIN_ROW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* rows = rows_all[warp];
  const int64_t stride = (int64_t)gridDim.x * WARPS * BPW;
  for (int64_t b0 = ((int64_t)blockIdx.x * WARPS + warp) * BPW; b0 < m; b0 += stride) {
    const double2* c[BPW];
    const double2* x[BPW];
    double2 r[BPW][4], y[BPW][4];
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      c[q] = x[q] = nullptr;
      if (b0 + q < m) {
        c[q] = reinterpret_cast<const double2*>(data + (b0 + q) * NB2);
        const int32_t xs = xslot[keys[b0 + q]];
        if (xs >= 0) x[q] = reinterpret_cast<const double2*>(xdata + (int64_t)xs * NB2);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        r[q][k] = c[q] ? __ldg(c[q] + k * 32 + lane) : make_double2(0.0, 0.0);
        y[q][k] = x[q] ? __ldg(x[q] + k * 32 + lane) : make_double2(0.0, 0.0);
      }
    }
    double acc = 0.0;
    unsigned anyq = 0;
    double cm[BPW][2];  // K4z column maxima (ex_col)
#pragma unroll
    for (int q = 0; q < BPW; ++q) cm[q][0] = cm[q][1] = 0.0;
    for (int ch = 0; ch < NCH; ++ch) {
      __syncwarp();
#pragma unroll
      for (int q = 0; q < BPW; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double* rq = rows + q * 4 * CHAIN_ROW + chain_pos(k, lane);
          if (ex_col) {
            cm[q][0] = fmax(cm[q][0], ozk::oz_absf(r[q][k].x));
            cm[q][1] = fmax(cm[q][1], ozk::oz_absf(r[q][k].y));
          }
          const double d0 = __dsub_rn(r[q][k].x, y[q][k].x);
          const double d1 = __dsub_rn(r[q][k].y, y[q][k].y);
          rq[0] = __dmul_rn(r[q][k].x, r[q][k].x);
          rq[CHAIN_ROW] = __dmul_rn(r[q][k].y, r[q][k].y);
          rq[2 * CHAIN_ROW] = __dmul_rn(d0, d0);
          rq[3 * CHAIN_ROW] = __dmul_rn(d1, d1);
          if ((r[q][k].x != 0.0) | (r[q][k].y != 0.0)) anyq |= 1u << q;
        }
      __syncwarp();
      if (ch + 1 < NCH) {
#pragma unroll
        for (int q = 0; q < BPW; ++q)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (c[q]) r[q][k] = __ldg(c[q] + (ch + 1) * 128 + k * 32 + lane);
            if (x[q]) y[q][k] = __ldg(x[q] + (ch + 1) * 128 + k * 32 + lane);
          }
      }
      if (lane < 4 * BPW) acc = chain_row128(rows + lane * CHAIN_ROW, acc);
    }
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      const double c0 = __shfl_sync(0xffffffffu, acc, 4 * q);
      const double c1 = __shfl_sync(0xffffffffu, acc, 4 * q + 1);
      const double e0 = __shfl_sync(0xffffffffu, acc, 4 * q + 2);
      const double e1 = __shfl_sync(0xffffffffu, acc, 4 * q + 3);
      const bool any = __any_sync(0xffffffffu, (anyq >> q) & 1u);
      if (lane == 0 && b0 + q < m) {
        const double v = __dadd_rn(c0, c1);
        out[b0 + q] = v;
        out1[b0 + q] = __dsqrt_rn(v);
        nz[b0 + q] = any ? 1 : 0;
        dout[b0 + q] = __dadd_rn(e0, e1);
      }
      if (ex_col && b0 + q < m)
        ozk::oz_col_exponents<NB>(cm[q][0], cm[q][1], keys[b0 + q] % G, ex_col, lane);
    }
  }
}

void leaf_norms2(const double* data, int64_t m, int nb, double* norms2, uint8_t* nonzero,
                 cudaStream_t s, double* norms1) {
  if (m <= 0) return;
  const int nb2 = nb * nb;
  if (nb2 == 1024 || nb2 == 4096) {
    constexpr int BPW = 2, WARPS = 4;
    const int grid = grid_for((m + BPW - 1) / BPW * 32, 32 * WARPS, 1LL << 20);
    if (nb2 == 1024)
      k_leaf_norms2_multi<1024, BPW, WARPS><<<grid, 32 * WARPS, 0, s>>>(data, m, norms2, nonzero,
                                                                        norms1);
    else
      k_leaf_norms2_multi<4096, BPW, WARPS><<<grid, 32 * WARPS, 0, s>>>(data, m, norms2, nonzero,
                                                                        norms1);
  } else {
    const int threads = 128;
    k_leaf_norms2<0><<<grid_for(m, threads, 1LL << 20), threads, 0, s>>>(data, m, nb2, norms2,
                                                                        nonzero);
  }
  SPAMM_LAUNCH_CK();
}

void build_pyramid(const int64_t* keys, const double* blk_norms2, int64_t m, int depth,
                   double* norms, double* norms2, cudaStream_t s) {
  if (depth <= SMALL_TREE_DEPTH) {
    launch_finalize_small(depth, 0, s, keys, blk_norms2, (const double*)nullptr,
                          (const uint8_t*)nullptr, m, depth, (int64_t*)nullptr,
                          (int32_t*)nullptr, norms, norms2, (const double*)nullptr, 0,
                          (double*)nullptr, (double*)nullptr, 0, (const double*)nullptr,
                          (const double*)nullptr, (double*)nullptr, (const int32_t*)nullptr,
                          (int64_t*)nullptr, (int64_t*)nullptr, (double*)nullptr);
    return;
  }
  const int64_t G = int64_t(1) << depth;
  double* leaf2 = norms2 + tier_offset(depth);
  double* leafn = norms + tier_offset(depth);
  SPAMM_CK(cudaMemsetAsync(leaf2, 0, G * G * sizeof(double), s));
  SPAMM_CK(cudaMemsetAsync(leafn, 0, G * G * sizeof(double), s));
  if (m > 0) {
    k_scatter_leaf<<<grid_for(m, 256), 256, 0, s>>>(keys, blk_norms2, m, leaf2, leafn);
    SPAMM_LAUNCH_CK();
  }
  int t = depth - 1;
  for (; t >= 0 && (int64_t(1) << (2 * t)) > 4096; --t) {
    const int64_t n = int64_t(1) << (2 * t);
    k_tier_up<<<grid_for(n, 256), 256, 0, s>>>(norms2 + tier_offset(t + 1), norms2 + tier_offset(t),
                                                norms + tier_offset(t), t);
    SPAMM_LAUNCH_CK();
  }
  if (t >= 0) {
    k_tiers_small<<<1, 1024, 0, s>>>(norms2, norms, t);
    SPAMM_LAUNCH_CK();
  }
}

namespace {
__global__ void k_leaf_from_norms2(const double* __restrict__ in, int64_t n,
                                   double* __restrict__ n2, double* __restrict__ n1) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = in[i];
    n2[i] = v;
    n1[i] = __dsqrt_rn(v);
  }
}
}  // namespace

void set_leaf_pyramid(Mat& m, const double* leaf_norms2, cudaStream_t s) {
  const int64_t G = int64_t(1) << m.depth;
  const int64_t off = tier_offset(m.depth);
  k_leaf_from_norms2<<<grid_for(G * G, 256), 256, 0, s>>>(leaf_norms2, G * G, m.norms2 + off,
                                                          m.norms + off);
  SPAMM_LAUNCH_CK();
  int t = m.depth - 1;
  for (; t >= 0 && (int64_t(1) << (2 * t)) > 4096; --t) {
    const int64_t n = int64_t(1) << (2 * t);
    k_tier_up<<<grid_for(n, 256), 256, 0, s>>>(m.norms2 + tier_offset(t + 1),
                                                m.norms2 + tier_offset(t), m.norms + tier_offset(t),
                                                t);
    SPAMM_LAUNCH_CK();
  }
  if (t >= 0) {
    k_tiers_small<<<1, 1024, 0, s>>>(m.norms2, m.norms, t);
    SPAMM_LAUNCH_CK();
  }
  if (m.host_top) {  // refresh the host mirror of the top tiers
    event_wait(m.top_ev);
    copy_to_pinned(m.host_top, m.norms, tier_offset(m.top_t + 1), s);
    SPAMM_CK(cudaEventRecord(m.top_ev, s));
  }
}

void scatter_slots(const int64_t* keys, int64_t m, int32_t* slot, cudaStream_t s) {
  if (m <= 0) return;
  k_scatter_slots<<<grid_for(m, 256), 256, 0, s>>>(keys, m, slot);
  SPAMM_LAUNCH_CK();
}

void finalize_impl(Mat& m, cudaStream_t s, double* pre_n2, uint8_t* pre_nz, bool defer,
                   IdemFuse idem, double* pre_n1 = nullptr);

bool idem_fusable(const Mat& x) {
  return x.depth <= SMALL_TREE_DEPTH && (x.nb == 32 || x.nb == 64);
}

void finalize(Mat& m, cudaStream_t s, IdemFuse idem, bool defer) {
  if (!idem.x || !defer || !idem_fusable(m)) throw CudaError("finalize: idempotency fusion unsupported");
  finalize_impl(m, s, nullptr, nullptr, defer, idem);
}

void finalize(Mat& m, cudaStream_t s, double* pre_n2, uint8_t* pre_nz, bool defer,
              double* pre_n1) {
  finalize_impl(m, s, pre_n2, pre_nz, defer, IdemFuse{}, pre_n1);
}

void finalize_with_residual(Mat& m, cudaStream_t s, double* pre_n2, uint8_t* pre_nz,
                            double* pre_n1, const double* pre_dn2, double* out) {
  if (!idem_fusable(m)) throw CudaError("finalize_with_residual: small trees, Nb 32 / 64");
  IdemFuse f;
  f.out = out;
  f.pre_dn2 = pre_dn2;
  finalize_impl(m, s, pre_n2, pre_nz, /*defer=*/true, f, pre_n1);
}

void finalize_impl(Mat& m, cudaStream_t s, double* pre_n2, uint8_t* pre_nz, bool defer,
                   IdemFuse idem, double* pre_n1) {
  m.stream = s;
  const int nb2 = m.nb * m.nb;
  double* n2 = pre_n2;
  if (defer && m.depth <= SMALL_TREE_DEPTH) {
    // one launch (after K1 unless the producer already computed the norms)
    uint8_t* nz = pre_nz;
    double* n1 = pre_n1;
    double* dn2 = nullptr;
    const double* dn2_in = idem.pre_dn2;  // (caller-owned)
    const bool multi = nb2 == 1024 || nb2 == 4096;
    if (m.nblocks > 0 && !n2) {
      n2 = dmalloc<double>(2 * m.nblocks, s);
      n1 = multi ? n2 + m.nblocks : nullptr;
      nz = dmalloc<uint8_t>(m.nblocks, s);
      if (idem.x) {
        dn2 = dmalloc<double>(m.nblocks, s);
        constexpr int WARPS = 4;
        const int grid = grid_for((m.nblocks + 1) / 2 * 32, 32 * WARPS, 1LL << 20);
        if (nb2 == 4096)
          launch_pdl(k_leaf_norms2_cd<4096, WARPS>, grid, 32 * WARPS, 0, s,
              m.data, m.keys, m.nblocks, idem.x->data, idem.x->slot, n2, nz, dn2, n1,
              idem.ex_col, int64_t(1) << m.depth);
        else
          launch_pdl(k_leaf_norms2_cd<1024, WARPS>, grid, 32 * WARPS, 0, s,
              m.data, m.keys, m.nblocks, idem.x->data, idem.x->slot, n2, nz, dn2, n1,
              idem.ex_col, int64_t(1) << m.depth);
        SPAMM_LAUNCH_CK();
      } else {
        leaf_norms2(m.data, m.nblocks, m.nb, n2, nz, s, n1);
      }
    }
    m.G = int64_t(1) << m.depth;
    dfree(m.slot, s);  // (a provisional slot map from the cull, trace-first SP2)
    m.slot = dmalloc<int32_t>(m.G * m.G, s);
    const int64_t ps = pyramid_size(m.depth);
    m.norms = dmalloc<double>(ps, s);
    m.norms2 = dmalloc<double>(ps, s);
    int64_t* kept = m.nblocks > 0 ? dmalloc<int64_t>(1, s) : nullptr;
    const bool want_tr = m.nb >= 2 && m.nb <= m.G;
    if (want_tr) m.tr_dev = dmalloc<double>(1, s);
    if (m.depth >= 2 && !m.host_top) {
      m.top_t = std::min(m.depth - 1, HOST_TOP_TIERS);
      top_acquire(&m.host_top, &m.top_ev);
    }
    launch_finalize_small(
        m.depth, m.nb, s, (const int64_t*)m.keys, (const double*)n2, (const double*)n1,
        (const uint8_t*)nz, m.nblocks, m.depth, kept, m.slot, m.norms, m.norms2,
        (const double*)m.data, m.nb, m.tr_dev, m.host_top, m.host_top ? m.top_t : -1,
        dn2_in ? dn2_in : (const double*)dn2,
        idem.x ? (const double*)(idem.x->norms2 + tier_offset(m.depth)) : (const double*)nullptr,
        idem.out, idem.x ? (const int32_t*)idem.x->slot : (const int32_t*)nullptr, idem.ukeys,
        idem.ucount, idem.dleaf);
    if (m.host_top) SPAMM_CK(cudaEventRecord(m.top_ev, s));
    dfree(dn2, s);
    dfree(n2, s);  // (a locally computed n1 shares n2's allocation)
    dfree(pre_n1, s);
    if (m.nblocks > 0) {
      m.pend_nz = nz;
      m.pend_kept = kept;
    } else {
      dfree(nz, s);
    }
    return;
  }
  dfree(pre_n1, s);  // (the tiered path takes sqrt per tier itself)
  if (m.nblocks > 0) {
    uint8_t* nz = pre_nz;
    if (!n2) {
      n2 = dmalloc<double>(m.nblocks, s);
      nz = dmalloc<uint8_t>(m.nblocks, s);
      leaf_norms2(m.data, m.nblocks, m.nb, n2, nz, s);
    }
    int64_t* off = dmalloc<int64_t>(m.nblocks + 1, s);
    scan_exclusive_u8(nz, m.nblocks, off, s);
    if (defer) {
      // Lazy prune: exact-zero blocks stay in storage and in the slot map for
      // now (their norm is exactly 0, so they never survive a cull, add zero
      // to traces and norms, and produce zero / pruned blocks in updates);
      // settle() drops them once the kept count rides on a later host sync.
      m.pend_nz = nz;
      m.pend_off = off;
    } else {
      int64_t kept = 0;
      d2h_sync(&kept, off + m.nblocks, 1, s);
      if (kept < m.nblocks) {
        double* d2 = dmalloc<double>((size_t)kept * nb2, s);
        int64_t* k2 = dmalloc<int64_t>(kept, s);
        double* nn = dmalloc<double>(kept, s);
        if (kept > 0) {
          k_compact_blocks<<<grid_for(m.nblocks, 1, 148LL * 32), 128, 0, s>>>(
              m.data, m.keys, n2, nz, off, m.nblocks, nb2, d2, k2, nn);
          SPAMM_LAUNCH_CK();
        }
        dfree(m.data, s);
        dfree(m.keys, s);
        dfree(n2, s);
        m.data = d2;
        m.keys = k2;
        n2 = nn;
        m.nblocks = kept;
      }
      dfree(nz, s);
      dfree(off, s);
    }
  }
  m.G = int64_t(1) << m.depth;
  m.slot = dmalloc<int32_t>(m.G * m.G, s);
  SPAMM_CK(cudaMemsetAsync(m.slot, 0xFF, m.G * m.G * sizeof(int32_t), s));
  if (m.nblocks > 0) {
    k_scatter_slots<<<grid_for(m.nblocks, 256), 256, 0, s>>>(m.keys, m.nblocks, m.slot);
    SPAMM_LAUNCH_CK();
  }
  const int64_t ps = pyramid_size(m.depth);
  m.norms = dmalloc<double>(ps, s);
  m.norms2 = dmalloc<double>(ps, s);
  build_pyramid(m.keys, n2, m.nblocks, m.depth, m.norms, m.norms2, s);
  dfree(n2, s);
  // Host mirror of the small top of the pyramid for the cull (no sync here).
  if (m.depth >= 2 && !m.host_top) {
    m.top_t = std::min(m.depth - 1, HOST_TOP_TIERS);
    top_acquire(&m.host_top, &m.top_ev);
    copy_to_pinned(m.host_top, m.norms, tier_offset(m.top_t + 1), s);
    SPAMM_CK(cudaEventRecord(m.top_ev, s));
  }
}

void attach_host_top(Mat& m, cudaStream_t s) {
  if (m.depth < 2) return;
  if (!m.host_top) {
    m.top_t = std::min(m.depth - 1, HOST_TOP_TIERS);
    top_acquire(&m.host_top, &m.top_ev);
  } else {
    event_wait(m.top_ev);
  }
  copy_to_pinned(m.host_top, m.norms, tier_offset(m.top_t + 1), s);
  SPAMM_CK(cudaEventRecord(m.top_ev, s));
}

void* pinned_scratch(size_t bytes) {
  thread_local void* buf = nullptr;
  thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    cap = std::max(bytes, (size_t)4096);
    SPAMM_CK(cudaMallocHost(&buf, cap));
  }
  return buf;
}

const int64_t* pending_kept(const Mat& m) {
  if (m.pend_kept) return m.pend_kept;
  return m.pend_off ? m.pend_off + m.nblocks : nullptr;
}

void settle(Mat& m, int64_t kept, cudaStream_t s) {
  if (!m.pend_nz) return;
  if (kept < m.nblocks) {
    const int nb2 = m.nb * m.nb;
    if (!m.pend_off) {  // only the count was produced: offsets now
      m.pend_off = dmalloc<int64_t>(m.nblocks + 1, s);
      scan_exclusive_u8(m.pend_nz, m.nblocks, m.pend_off, s);
    }
    double* d2 = dmalloc<double>((size_t)kept * nb2, s);
    int64_t* k2 = dmalloc<int64_t>(kept, s);
    if (kept > 0) {
      k_compact_blocks<<<grid_for(m.nblocks, 1, 148LL * 32), 128, 0, s>>>(
          m.data, m.keys, nullptr, m.pend_nz, m.pend_off, m.nblocks, nb2, d2, k2, nullptr);
      SPAMM_LAUNCH_CK();
    }
    dfree(m.data, s);
    dfree(m.keys, s);
    m.data = d2;
    m.keys = k2;
    m.nblocks = kept;
    // the pyramid is unchanged (the dropped blocks had norm 0); the slot map is rebuilt
    SPAMM_CK(cudaMemsetAsync(m.slot, 0xFF, m.G * m.G * sizeof(int32_t), s));
    if (kept > 0) {
      k_scatter_slots<<<grid_for(kept, 256), 256, 0, s>>>(m.keys, kept, m.slot);
      SPAMM_LAUNCH_CK();
    }
  }
  dfree(m.pend_nz, s);
  dfree(m.pend_off, s);
  dfree(m.pend_kept, s);
  m.pend_nz = nullptr;
  m.pend_off = nullptr;
  m.pend_kept = nullptr;
}

void settle_sync(Mat& m, cudaStream_t s) {
  if (!m.pend_nz) return;
  int64_t kept = 0;
  d2h_sync(&kept, pending_kept(m), 1, s);
  settle(m, kept, s);
}

}  // namespace spamm

