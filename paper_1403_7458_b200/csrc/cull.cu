// K2 + K3: tiered culling with in-order compaction.
//
// Reference: kernel._sweep (kernel.py:96-122) + the task sort / searchsorted
// block of multiply (kernel.py:189-204).
//
// The reference expands every surviving triple (i,k,j) of tier t into its 8
// children, keeps those with nA[t+1][i,k] * nB[t+1][k,j] > tau (strict), and
// finally sorts the leaf triples by C block then k.  Here the survivors are
// kept grouped by their C node (I,J) with K ascending, so no sort is needed:
// a C node with K-list L has 4 children (di,dj) whose candidate lists are
// [2K+dk for K in L for dk in (0,1)] -- already ascending.  Per tier:
//   pass 1 (count): one warp per parent node counts survivors per child
//                   with __ballot_sync/__popc, packing (node>0, count) into
//                   one int64 so a single scan yields both offsets;
//   pass 2 (scan):  device-wide exclusive scan (scan.cu);
//   pass 3 (write): same predicate, ballot + popc(lanemask_lt) compaction
//                   into the child node's segment (deterministic order).
// Candidates per tier are 8 x survivors of the previous tier, exactly the
// reference's expansion, so visited/culled per tier are identical.  The
// surviving C nodes come out in Morton (Z) order of (i, j).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace spamm {

namespace {

constexpr int NODE_SHIFT = 40;
constexpr int64_t TASK_MASK = (int64_t(1) << NODE_SHIFT) - 1;
constexpr int CULL_THREADS = 256;

__device__ __forceinline__ bool keep_pair(double na, double nb, double tau) {
  return __dmul_rn(na, nb) > tau;
}

// Near-tau probe (the north star's "documented norm ties within one ulp of
// tau"): a tested product p = fl(nA nB) with |p - tau| <= band (k ulp(tau),
// spamm_set_near_tau_ulps) is counted per tier, and the smallest relative
// distance |p - tau| / tau among tested products within `wide` (tau 2^-20) is
// kept as the bit pattern of a non-negative double in inverted form (atomicMax
// of ~bits: zero-initialised memory reads as "none").  Products this close
// are the only ones whose decision can differ from the reference's when the
// operand norms differ from the reference operand's by a few ulps.  Both
// bands are < 0 (off) for tau = 0.
struct TieBand {
  double tau = 0.0, band = -1.0, wide = -1.0;
};
int g_near_ulps = 64;
TieBand tie_band(double tau) {
  TieBand tb;
  tb.tau = tau;
  if (tau > 0.0 && std::isfinite(tau)) {
    tb.band = g_near_ulps * (std::nextafter(tau, INFINITY) - tau);
    tb.wide = std::ldexp(tau, -20);
  }
  return tb;
}
double margin_from_bits(int64_t inv) {  // see tie_probe; +inf: nothing within tau 2^-20
  if (inv == 0) return INFINITY;
  const uint64_t bits = ~(uint64_t)inv;
  double d;
  std::memcpy(&d, &bits, sizeof d);
  return d;
}

__device__ __forceinline__ void tie_probe(double p, const TieBand& tb,
                                          unsigned long long* __restrict__ near,
                                          unsigned long long* __restrict__ margin) {
  const double d = fabs(p - tb.tau);
  if (!(d <= tb.wide)) return;
  if (d <= tb.band) atomicAdd(near, 1ull);
  atomicMax(margin, ~(unsigned long long)__double_as_longlong(d / tb.tau));
}

__global__ void k_cull_root(const double* __restrict__ nA, const double* __restrict__ nB,
                            double tau, int32_t* ci, int32_t* cj, int64_t* seg, int32_t* K,
                            int64_t* count, const int32_t* slotA, const int32_t* slotB,
                            int32_t* aidx, int32_t* bidx, TieBand tb,
                            unsigned long long* near, unsigned long long* margin) {
  const bool keep = keep_pair(nA[0], nB[0], tau);
  tie_probe(__dmul_rn(nA[0], nB[0]), tb, near, margin);
  ci[0] = 0;
  cj[0] = 0;
  seg[0] = 0;
  seg[1] = keep ? 1 : 0;
  K[0] = 0;
  count[0] = keep ? 1 : 0;
  if (aidx && keep) {
    aidx[0] = slotA[0];
    bidx[0] = slotB[0];
  }
}

// WRITE=false: count pass.  WRITE=true: compaction pass (LEAF: also A/B slots).
template <bool WRITE, bool LEAF>
__global__ void __launch_bounds__(CULL_THREADS)
    k_cull_expand(int t1, const double* __restrict__ nA, const double* __restrict__ nB, double tau,
                  int64_t M, const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                  const int64_t* __restrict__ seg, const int32_t* __restrict__ K,
                  int64_t* __restrict__ cnt4, const int64_t* __restrict__ off4,
                  int32_t* __restrict__ ci_o, int32_t* __restrict__ cj_o,
                  int64_t* __restrict__ seg_o, int32_t* __restrict__ K_o,
                  const int32_t* __restrict__ slotA, const int32_t* __restrict__ slotB,
                  int32_t* __restrict__ aidx, int32_t* __restrict__ bidx, int64_t Mn, int64_t Vn,
                  int sym, unsigned long long* __restrict__ aux, int64_t lo, int64_t hi,
                  int shift, int32_t* __restrict__ work, TieBand tb) {
  const int64_t W = int64_t(1) << t1;
  const double* A = nA + tier_offset(t1);
  const double* B = nB + tier_offset(t1);
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (WRITE && gw == 0 && lane == 0) seg_o[Mn] = Vn;
  for (int64_t p = gw; p < M; p += nw) {
    const int64_t I = ci[p], J = cj[p];
    const int64_t s = seg[p], e = seg[p + 1];
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      const int64_t row = 2 * I + (c >> 1), col = 2 * J + (c & 1);
      // Symmetric mode (A == B == X, X = X^T bitwise): only C nodes with
      // i <= j are carried; the lower child of a diagonal parent is the
      // mirror of its (0,1) child and is skipped.
      if (sym && row > col) {
        if (!WRITE && lane == 0) cnt4[4 * p + c] = 0;
        continue;
      }
      // Shard filter (multi-GPU): keep the child only if its Morton subtree
      // [m << shift, (m + 1) << shift) of leaf C positions meets [lo, hi).
      if (lo > 0 || hi >= 0) {
        const int64_t m0 = (int64_t)morton_encode((uint32_t)row, (uint32_t)col) << shift;
        if (m0 >= hi || m0 + (int64_t(1) << shift) <= lo) {
          if (!WRITE && lane == 0) cnt4[4 * p + c] = 0;
          continue;
        }
      }
      const double* Arow = A + row * W;
      int64_t toff = 0;
      if (WRITE) {
        const int64_t v = off4[4 * p + c], vn = off4[4 * p + c + 1];
        if (((vn - v) & TASK_MASK) == 0) continue;
        const int64_t node = v >> NODE_SHIFT;
        toff = v & TASK_MASK;
        if (lane == 0) {
          ci_o[node] = (int32_t)row;
          cj_o[node] = (int32_t)col;
          seg_o[node] = toff;
          if (LEAF && work)
            work[morton_encode((uint32_t)row, (uint32_t)col)] = (int32_t)((vn - v) & TASK_MASK);
        }
      }
      int64_t cnt = 0;
      for (int64_t q0 = s; q0 < e; q0 += 16) {
        const int64_t q = q0 + (lane >> 1);
        const bool valid = q < e;
        const int64_t kk = valid ? 2 * (int64_t)K[q] + (lane & 1) : 0;
        const bool keep = valid && keep_pair(Arow[kk], B[kk * W + col], tau);
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (!WRITE && valid) tie_probe(__dmul_rn(Arow[kk], B[kk * W + col]), tb, aux + 4, aux + 5);
        if (!WRITE && sym && row != col) {
          // mirror triple (col, kk, row) must agree, else the survivor set is
          // not symmetric (an ulp tie between norm(X_ik) and norm(X_ki^T)).
          const bool keep_m = valid && keep_pair(A[col * W + kk], B[kk * W + row], tau);
          if (valid) tie_probe(__dmul_rn(A[col * W + kk], B[kk * W + row]), tb, aux + 4, aux + 5);
          if (__any_sync(0xffffffffu, keep != keep_m) && lane == 0) atomicOr(aux + 1, 1ull);
        }
        if (WRITE) {
          if (keep) {
            const int64_t pos = toff + __popc(mask & lt_mask);
            K_o[pos] = (int32_t)kk;
            if (LEAF) {
              aidx[pos] = slotA[row * W + kk];
              bidx[pos] = slotB[kk * W + col];
            }
          }
          toff += __popc(mask);
        } else {
          cnt += __popc(mask);
        }
      }
      if (!WRITE && lane == 0) {
        cnt4[4 * p + c] = cnt + (cnt > 0 ? (int64_t(1) << NODE_SHIFT) : 0);
        // leaf tier: per-C-block task counts (census with work, persistence LB)
        if (work && shift == 0 && cnt)
          work[morton_encode((uint32_t)row, (uint32_t)col)] = (int32_t)cnt;
        if (sym && row == col && cnt) {
          atomicAdd(aux, (unsigned long long)cnt);
          atomicAdd(aux + 3, 1ull);
        }
      }
    }
  }
}

int cull_grid(int64_t M) { return grid_for(M * 32, CULL_THREADS, 148LL * 64); }


// Host-side cull of the top tiers (K2): the pyramid's tiers
// 0..T0 are mirrored to pinned host memory when a matrix is finalised, so the
// small top of the tree is expanded here in C++ with the same IEEE predicate
// (one double multiply, strict >) and the same order (parents in Morton
// order, children (0,0),(0,1),(1,0),(1,1), K ascending) as the device passes,
// instead of paying one kernel chain + host sync per tier.
struct HostLevel {
  std::vector<int32_t> ci, cj, K;
  std::vector<int64_t> seg;
};

void host_tie_probe(double p, const TieBand& tb, int64_t& near, double& margin) {
  const double d = std::fabs(p - tb.tau);
  if (!(d <= tb.wide)) return;
  if (d <= tb.band) ++near;
  margin = std::min(margin, d / tb.tau);
}

bool host_cull_top(const double* nA, const double* nB, int T0, int depth, double tau, bool sym,
                   int64_t lo, int64_t hi, CullResult& r, HostLevel& L, int64_t& full_prev,
                   int64_t& diag_nodes, const TieBand& tb) {
  const bool keep0 = nA[0] * nB[0] > tau;
  host_tie_probe(nA[0] * nB[0], tb, r.near[0], r.margin);
  r.visited[0] = keep0 ? 1 : 0;
  r.culled[0] = keep0 ? 0 : 1;
  L.ci.assign(1, 0);
  L.cj.assign(1, 0);
  L.seg.assign({0, keep0 ? 1 : 0});
  L.K.assign(keep0 ? 1 : 0, 0);
  full_prev = keep0 ? 1 : 0;
  diag_nodes = full_prev;
  if (!keep0) {
    L.ci.clear();
    L.cj.clear();
    L.seg.assign(1, 0);
    return true;
  }
  HostLevel N;
  for (int t1 = 1; t1 <= T0; ++t1) {
    const int64_t W = int64_t(1) << t1;
    const double* A = nA + tier_offset(t1);
    const double* B = nB + tier_offset(t1);
    const int shift = 2 * (depth - t1);
    N.ci.clear();
    N.cj.clear();
    N.K.clear();
    N.seg.clear();
    int64_t D = 0, dn = 0;
    const int64_t M = (int64_t)L.ci.size();
    for (int64_t p = 0; p < M; ++p) {
      const int64_t I = L.ci[p], J = L.cj[p];
      for (int c = 0; c < 4; ++c) {
        const int64_t row = 2 * I + (c >> 1), col = 2 * J + (c & 1);
        if (sym && row > col) continue;
        if (lo > 0 || hi >= 0) {
          const int64_t m0 = (int64_t)morton_encode((uint32_t)row, (uint32_t)col) << shift;
          if (m0 >= hi || m0 + (int64_t(1) << shift) <= lo) continue;
        }
        const size_t start = N.K.size();
        for (int64_t q = L.seg[p]; q < L.seg[p + 1]; ++q)
          for (int dk = 0; dk < 2; ++dk) {
            const int64_t kk = 2 * (int64_t)L.K[q] + dk;
            const bool keep = A[row * W + kk] * B[kk * W + col] > tau;
            host_tie_probe(A[row * W + kk] * B[kk * W + col], tb, r.near[t1], r.margin);
            if (sym && row != col) {
              host_tie_probe(A[col * W + kk] * B[kk * W + row], tb, r.near[t1], r.margin);
              if (keep != (A[col * W + kk] * B[kk * W + row] > tau)) return false;
            }
            if (keep) N.K.push_back((int32_t)kk);
          }
        const int64_t cnt = (int64_t)(N.K.size() - start);
        if (cnt) {
          N.ci.push_back((int32_t)row);
          N.cj.push_back((int32_t)col);
          N.seg.push_back((int64_t)start);
          if (sym && row == col) {
            D += cnt;
            ++dn;
          }
        }
      }
    }
    const int64_t Vn = (int64_t)N.K.size();
    N.seg.push_back(Vn);
    const int64_t full = sym ? 2 * Vn - D : Vn;
    r.visited[t1] = full;
    r.culled[t1] = 8 * full_prev - full;
    full_prev = full;
    diag_nodes = dn;
    std::swap(L, N);
    if (Vn == 0) break;
  }
  return true;
}

// ---------------------------------------------------------------- dense cull
// For a small tree (depth <= DENSE_MAX_DEPTH, G <= 256) the whole cull is two
// data-parallel passes and ONE host sync instead of a tier-by-tier walk.  A
// leaf triple (i,k,j) is a survivor of _sweep iff its own product and every
// ancestor's product pass (kernel.py:108-113: a triple is only ever tested
// when its parent survived), so each triple is evaluated directly with its
// ancestor chain -- the same IEEE predicates, hence the same set and the same
// per-tier counts as the recursive walk, in the same output order (C blocks
// in Morton order, k ascending).
constexpr int DENSE_MAX_DEPTH = 8;
bool g_dense_enabled = true;

// The ancestor chain of a triple is evaluated without early exit: the 2 (t+1)
// norm loads are independent (one L1 round trip instead of t + 1 dependent
// ones), and the AND of the same IEEE predicates is the same decision.
__device__ __forceinline__ bool keep_chain(const double* __restrict__ nA,
                                           const double* __restrict__ nB, double tau, int t,
                                           int64_t i, int64_t k, int64_t j) {
  bool ok = true;
  for (int u = t; u >= 0; --u) {
    const int sh = t - u;
    const int64_t W = int64_t(1) << u;
    const int64_t off = tier_offset(u);
    ok &= keep_pair(nA[off + (i >> sh) * W + (k >> sh)], nB[off + (k >> sh) * W + (j >> sh)], tau);
  }
  return ok;
}

// every tier u < t of the triple's ancestor chain passes (the triple is tested)
__device__ __forceinline__ bool ancestors_pass(const double* __restrict__ nA,
                                               const double* __restrict__ nB, double tau, int t,
                                               int64_t i, int64_t k, int64_t j) {
  bool ok = true;
  for (int u = t - 1; u >= 0; --u) {
    const int sh = t - u;
    const int64_t W = int64_t(1) << u;
    const int64_t off = tier_offset(u);
    ok &= keep_pair(nA[off + (i >> sh) * W + (k >> sh)], nB[off + (k >> sh) * W + (j >> sh)], tau);
  }
  return ok;
}
// tie probe of the tier-t triple (i, k, j) if it is tested (see tie_probe)
__device__ __forceinline__ void chain_tie_probe(const double* __restrict__ nA,
                                                const double* __restrict__ nB, const TieBand& tb,
                                                int t, int64_t i, int64_t k, int64_t j,
                                                unsigned long long* near,
                                                unsigned long long* margin) {
  const int64_t W = int64_t(1) << t, off = tier_offset(t);
  const double p = __dmul_rn(nA[off + i * W + k], nB[off + k * W + j]);
  if (!(fabs(p - tb.tau) <= tb.wide)) return;
  if (ancestors_pass(nA, nB, tb.tau, t, i, k, j)) tie_probe(p, tb, near, margin);
}

// Leaf tier, one warp per C position m (Morton order).  Each m gets one
// packed int64 so a single scan yields every offset the layout needs:
//   bits  0..26  tasks of the node if it is emitted (symmetric: i <= j only)
//   bits 27..44  1 if the node is emitted with >= 1 task  -> node index
//   bits 45..62  1 if C block (i,j) exists at all         -> storage slot
// (G <= 256: tasks <= 2^24, nodes <= 2^16.)
constexpr int DT_NODE = 27, DT_FULL = 45;
constexpr int64_t DT_TASK_MASK = (int64_t(1) << DT_NODE) - 1;
constexpr int64_t DT_IDX_MASK = (int64_t(1) << (DT_FULL - DT_NODE)) - 1;

// Block-wide (CULL_THREADS) exclusive scan of one int64 per thread; returns
// the block total.
__device__ __forceinline__ int64_t cull_block_scan(int64_t v, int64_t& excl, int64_t* wsum) {
  constexpr int NW = CULL_THREADS / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int64_t w = lane < NW ? wsum[lane] : 0;
    int64_t z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < NW) wsum[lane] = z - w;
    if (lane == NW - 1) wsum[NW] = z;
  }
  __syncthreads();
  excl = wsum[warp] + x - v;
  const int64_t total = wsum[NW];
  __syncthreads();
  return total;
}

// Count pass of the dense cull, one launch:
//  * CTAs [0, n_tier): survivor counts and near-tau probes of every upper
//    tier t < depth - 1 (full enumeration, 8^t triples; warp-reduced counts)
//    -- first in the grid, so they are in the first wave;
//  * CTAs [n_tier, grid): the leaf tier, DC_PPC = 32 consecutive Morton
//    positions per CTA, one warp per tier-(depth-1) parent node and its four
//    children.  The ancestor chains of the children's leaf triples are the
//    parent's chains over K = k/2: the warp evaluates them once (and, on the
//    symmetric path, its mirror's) into bit masks, so every leaf test is one
//    product plus a mask bit -- the same predicates as keep_chain.  The
//    parents' tested triples are exactly tier depth-1, so its survivor count
//    and near-tau probes are taken there too.  Per position: the packed count
//    (cnt), the keep masks of its k-range (kmask, 32 k per word: the write
//    pass compacts from them without re-testing), the LPT length histogram,
//    the symmetric mirror check and the near-tau probes; per CTA the
//    exclusive prefix of its positions (lofs) and their total (ctasum);
//  * the last CTA to finish scans the CTA totals (ctapre: off[q] =
//    ctapre[q / DC_PPC] + lofs[q]), scans the histogram in place, and
//    publishes the scalars the host needs to pinned memory (gather_sync's
//    protocol) -- one launch before the cull's host sync.
constexpr int DC_PPC = 32;  // positions per leaf CTA (8 warps x 4 children)
__device__ __forceinline__ int64_t dc_off(const int64_t* __restrict__ ctapre,
                                          const int64_t* __restrict__ lofs, int64_t q) {
  return ctapre[q / DC_PPC] + lofs[q];
}

__global__ void __launch_bounds__(CULL_THREADS, 2)
    k_dense_count(int depth, const double* __restrict__ nA, const double* __restrict__ nB,
                  double tau, int sym, int64_t* __restrict__ cnt, uint32_t* __restrict__ kmask,
                  int* __restrict__ hist, int want_tasks, unsigned long long* __restrict__ aux,
                  TieBand tb, unsigned long long* __restrict__ near_tiers,
                  unsigned long long* __restrict__ margin, int64_t lo, int64_t hi,
                  int32_t* __restrict__ work, int n_tier, int tiers, unsigned* __restrict__ done,
                  int64_t* __restrict__ lofs, int64_t* __restrict__ ctasum,
                  int64_t* __restrict__ ctapre, ScalarSrc src, int n_src, int64_t* gvals,
                  int64_t* gflag, int64_t seq, unsigned long long* __restrict__ prof) {
  // prof (SPAMM_CULL_PROF): %globaltimer per CTA [start, end] + last CTA phases
  auto gtime = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (prof && threadIdx.x == 0) prof[2 * blockIdx.x] = gtime();
  pdl_wait();
  __shared__ int64_t wsum[CULL_THREADS / 32 + 1];
  __shared__ int64_t pcnt[DC_PPC];
  __shared__ unsigned long long cta_full;
  __shared__ unsigned int sc[DENSE_MAX_DEPTH];
  __shared__ bool last;
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int KW = (int)((G + 31) >> 5);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_leaf = (int)gridDim.x - n_tier;
  if ((int)blockIdx.x >= n_tier) {
    const int64_t cta = blockIdx.x - n_tier;
    auto in_range = [&](int64_t q) { return hi < 0 || (q >= lo && q < hi); };
    unsigned long long* near = near_tiers + depth;
    if (threadIdx.x == 0) {
      cta_full = 0;
      sc[0] = 0;
    }
    if (threadIdx.x < DC_PPC) pcnt[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long full = 0;
    // one C position m: counts, histogram, work; keep(k) / keep_m(k) are the
    // leaf triple (i,k,j) / its mirror (j,k,i)
    auto finish_pos = [&](int64_t m, bool emitted, int64_t c) {
      if (lane == 0) {
        const int64_t v = (emitted ? c + (c > 0 ? int64_t(1) << DT_NODE : 0) : 0) +
                          (c > 0 ? int64_t(1) << DT_FULL : 0);
        cnt[m] = v;
        pcnt[m - cta * DC_PPC] = v;
        if (work && emitted && c) work[m] = (int32_t)c;  // persistence load balancing input
        full += c;
        if (want_tasks && c && emitted) atomicAdd(hist + (G - c), 1);
      }
    };
    if (depth >= 2) {
      const int64_t P = cta * (DC_PPC / 4) + warp;  // this warp's tier-(depth-1) parent
      if (P < npos / 4) {
        const int64_t GH = G >> 1;
        const int PW = (int)((GH + 31) >> 5);  // <= 4 (G <= 256)
        const int64_t leaf_off = tier_offset(depth);
        uint32_t I, J;
        morton_decode((uint64_t)P, I, J);
        uint32_t pk[4] = {0u, 0u, 0u, 0u}, px[4] = {0u, 0u, 0u, 0u};
        unsigned pc = 0;
#pragma unroll
        for (int kw = 0; kw < 4; ++kw) {
          if (kw >= PW) break;
          const int64_t K = (int64_t)kw * 32 + lane;
          const bool valid = K < GH;
          const bool keep = valid && keep_chain(nA, nB, tau, depth - 1, I, K, J);
          const bool keepx = sym && valid && keep_chain(nA, nB, tau, depth - 1, J, K, I);
          pk[kw] = __ballot_sync(0xffffffffu, keep);
          px[kw] = __ballot_sync(0xffffffffu, keepx);
          if (tiers) {
            if (valid)
              chain_tie_probe(nA, nB, tb, depth - 1, I, K, J, near_tiers + depth - 1, margin);
            pc += __popc(pk[kw]);
          }
        }
        if (tiers && lane == 0 && pc) atomicAdd(sc, pc);
        // the four children (Morton order: ch = 2 (i & 1) + (j & 1)); leaf
        // norms are loaded one 32-k chunk ahead (rows 2I, 2I+1 of nA, columns
        // 2J, 2J+1 of nB, and the mirror's), all in flight together
        bool owned[4], emitted[4];
        int64_t c[4];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int64_t m = 4 * P + ch;
          const int64_t i = 2 * (int64_t)I + (ch >> 1), j = 2 * (int64_t)J + (ch & 1);
          owned[ch] = sym && i > j ? in_range((int64_t)morton_encode((uint32_t)j, (uint32_t)i))
                                   : in_range(m);
          emitted[ch] = owned[ch] && (!sym || i <= j);
          c[ch] = 0;
          if (!owned[ch] && lane == 0) cnt[m] = 0;
        }
        const int64_t i0 = 2 * (int64_t)I, j0 = 2 * (int64_t)J;
        auto load = [&](int it, double (&v)[8]) {
          const int64_t k = (int64_t)it * 32 + lane;
          const bool valid = k < G;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            v[u] = valid ? nA[leaf_off + (i0 + u) * G + k] : 0.0;      // A row 2I + u
            v[2 + u] = valid ? nB[leaf_off + k * G + j0 + u] : 0.0;    // B column 2J + u
            v[4 + u] = valid && sym ? nA[leaf_off + (j0 + u) * G + k] : 0.0;  // mirror A row
            v[6 + u] = valid && sym ? nB[leaf_off + k * G + i0 + u] : 0.0;    // mirror B col
          }
        };
        double cur[8], nxt[8];
        load(0, cur);
#pragma unroll
        for (int it = 0; it < 8; ++it) {  // G <= 256: <= 8 chunks of 32 k
          const int64_t k0 = (int64_t)it * 32;
          if (k0 >= G) break;
          if (k0 + 32 < G) load(it + 1, nxt);
          const int64_t k = k0 + lane;
          const bool valid = k < G;
          const int w = it >> 1, sh = (int)(((k0 >> 1) + (lane >> 1)) & 31);
          const bool par = valid && ((pk[w] >> sh) & 1u);
          const bool parm = valid && ((px[w] >> sh) & 1u);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (!owned[ch]) continue;
            const int ri = ch >> 1, cj = ch & 1;
            const int64_t m = 4 * P + ch;
            const bool mirror = sym && i0 + ri < j0 + cj;
            const double pr = __dmul_rn(cur[ri], cur[2 + cj]);
            const bool keep = par && pr > tau;
            const unsigned mask = __ballot_sync(0xffffffffu, keep);
            if (valid && emitted[ch] && par && fabs(pr - tb.tau) <= tb.wide)
              tie_probe(pr, tb, near, margin);
            if (mirror) {
              const double pm = __dmul_rn(cur[4 + cj], cur[6 + ri]);
              const bool keep_m = parm && pm > tau;
              if (valid && emitted[ch] && parm && fabs(pm - tb.tau) <= tb.wide)
                tie_probe(pm, tb, near, margin);
              if (__any_sync(0xffffffffu, keep != keep_m) && lane == 0) atomicOr(aux + 1, 1ull);
            }
            if (want_tasks && emitted[ch] && lane == 0) kmask[m * KW + it] = mask;
            c[ch] += __popc(mask);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
        }
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
          if (owned[ch]) finish_pos(4 * P + ch, emitted[ch], c[ch]);
      }
    } else {
      // G <= 2: one CTA, one warp per position, full chains
      const int64_t m = warp;
      if (cta == 0 && m < npos) {
        uint32_t ui, uj;
        morton_decode((uint64_t)m, ui, uj);
        const int64_t i = ui, j = uj;
        const bool owned = sym && i > j ? in_range((int64_t)morton_encode(uj, ui)) : in_range(m);
        const bool emitted = owned && (!sym || i <= j);
        if (!owned) {
          if (lane == 0) cnt[m] = 0;
        } else {
          const int64_t k = lane;
          const bool valid = k < G;
          const bool keep = valid && keep_chain(nA, nB, tau, depth, i, k, j);
          const unsigned mask = __ballot_sync(0xffffffffu, keep);
          if (valid && emitted) {
            chain_tie_probe(nA, nB, tb, depth, i, k, j, near, margin);
            if (sym && i < j) chain_tie_probe(nA, nB, tb, depth, j, k, i, near, margin);
          }
          if (sym && i < j) {
            const bool keep_m = valid && keep_chain(nA, nB, tau, depth, j, k, i);
            if (__any_sync(0xffffffffu, keep != keep_m) && lane == 0) atomicOr(aux + 1, 1ull);
          }
          if (want_tasks && emitted && lane == 0) kmask[m * KW] = mask;
          finish_pos(m, emitted, __popc(mask));
        }
      }
    }
    // full (reference) leaf count: one global atomic per CTA
    if (lane == 0 && full) atomicAdd(&cta_full, full);
    __syncthreads();
    if (threadIdx.x == 0 && cta_full) atomicAdd(aux, cta_full);
    if (threadIdx.x == 0 && depth >= 2 && sc[0])
      atomicAdd(aux + 4 + depth - 1, (unsigned long long)sc[0]);
    if (warp == 0) {  // the CTA's positions: exclusive prefix and total
      const int64_t v = pcnt[lane];
      int64_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const int64_t q = cta * DC_PPC + lane;
      if (q < npos) lofs[q] = x - v;
      if (lane == 31) ctasum[cta] = x;
    }
  } else {
    if (threadIdx.x < DENSE_MAX_DEPTH) sc[threadIdx.x] = 0;
    __syncthreads();
    // tiers 0 .. depth-2 here (tier depth-1 is counted by the leaf CTAs)
    const int64_t total = depth >= 2 ? ((int64_t(1) << (3 * (depth - 1))) - 1) / 7
                                     : ((int64_t(1) << (3 * depth)) - 1) / 7;
    const int64_t tb0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t tstride = (int64_t)n_tier * blockDim.x;
    // warp-uniform trip count so the per-tier reductions see full warps
    for (int64_t q0 = (tb0 + threadIdx.x) & ~int64_t(31); q0 < total; q0 += tstride) {
      const int64_t q = q0 + lane;
      int t = -1;
      if (q < total) {
        t = 0;
        while ((((int64_t(1) << (3 * (t + 1))) - 1) / 7) <= q) ++t;
        const int64_t r = q - ((int64_t(1) << (3 * t)) - 1) / 7;
        const int64_t i = r >> (2 * t), k = (r >> t) & ((int64_t(1) << t) - 1),
                      j = r & ((int64_t(1) << t) - 1);
        chain_tie_probe(nA, nB, tb, t, i, k, j, near_tiers + t, margin);
        if (!keep_chain(nA, nB, tau, t, i, k, j)) t = -1;
      }
      for (int u = 0; u < depth; ++u) {
        const unsigned v = __reduce_add_sync(0xffffffffu, t == u ? 1u : 0u);
        if (lane == 0 && v) atomicAdd(sc + u, v);
      }
    }
    __syncthreads();
    if (threadIdx.x < depth && sc[threadIdx.x])
      atomicAdd(aux + 4 + threadIdx.x, (unsigned long long)sc[threadIdx.x]);
  }
  // ---- last CTA: the CTA-total scan and the host-visible scalars
  __threadfence();
  __syncthreads();
  if (prof && threadIdx.x == 0) prof[2 * blockIdx.x + 1] = gtime();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (prof && threadIdx.x == 0) prof[2 * gridDim.x] = gtime();
  // three independent jobs, one warp each, one barrier: warp 0 scans the CTA
  // totals, warp 1 the LPT length histogram (in place), warp 2 gathers the
  // other scalars; then one thread publishes
  __shared__ int64_t total_sh;
  if (warp == 0) {
    int64_t carry = 0;
    for (int64_t b0 = 0; b0 < n_leaf; b0 += 32 * 8) {
      int64_t v[8];
      int64_t sum = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int64_t b = b0 + lane * 8 + r;
        v[r] = b < n_leaf ? __ldcg(ctasum + b) : 0;
        sum += v[r];
      }
      int64_t x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int64_t run = carry + x - sum;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int64_t b = b0 + lane * 8 + r;
        if (b < n_leaf) ctapre[b] = run;
        run += v[r];
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) total_sh = carry;
  } else if (warp == 1 && want_tasks) {  // G + 1 <= 257 bins
    const int nbins = (int)G + 1;
    int64_t carry = 0;
    for (int b0 = 0; b0 < nbins; b0 += 32 * 9) {
      int v[9];
      int sum = 0;
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const int b = b0 + lane * 9 + r;
        v[r] = b < nbins ? __ldcg(hist + b) : 0;
        sum += v[r];
      }
      int x = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int64_t run = carry + x - sum;
#pragma unroll
      for (int r = 0; r < 9; ++r) {
        const int b = b0 + lane * 9 + r;
        if (b < nbins) hist[b] = (int)run;
        run += v[r];
      }
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  } else if (warp == 2) {
    for (int i = lane; i < n_src; i += 32)
      if (i != 2) gvals[i] = src.p[i] ? __ldcg(src.p[i]) : 0;
    __threadfence_system();  // (pinned host memory: before the flag below)
  }
  __threadfence();
  __syncthreads();
  if (prof && threadIdx.x == 0) prof[2 * gridDim.x + 1] = gtime();
  if (prof && threadIdx.x == 0) prof[2 * gridDim.x + 2] = gtime();
  if (threadIdx.x == 0) {
    aux[2] = total_sh;   // packed totals
    gvals[2] = total_sh;
    __threadfence_system();
    *reinterpret_cast<volatile int64_t*>(gflag) = seq;
  }
  if (prof && threadIdx.x == 0) prof[2 * gridDim.x + 3] = gtime();
}

// Write pass: the task lists, C keys, storage / mirror slots and the LPT
// order of the nodes, compacted from the count pass's keep masks (no norm is
// read again).  One warp per C position.
__global__ void __launch_bounds__(CULL_THREADS)
    k_dense_write(int depth, int sym, const int64_t* __restrict__ cnt,
                  const int64_t* __restrict__ lofs, const int64_t* __restrict__ ctapre,
                  const uint32_t* __restrict__ kmask, int* __restrict__ hist,
                  int32_t* __restrict__ ci_o, int32_t* __restrict__ cj_o,
                  int64_t* __restrict__ seg_o, int32_t* __restrict__ K_o,
                  const int32_t* __restrict__ slotA, const int32_t* __restrict__ slotB,
                  int32_t* __restrict__ aidx, int32_t* __restrict__ bidx,
                  int64_t* __restrict__ keys, int64_t* __restrict__ c_out,
                  int64_t* __restrict__ c_mirror, int32_t* __restrict__ order, int64_t Mn,
                  int64_t Vn, int32_t* __restrict__ c_slot) {
  pdl_wait();
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int KW = (int)((G + 31) >> 5);
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (gw == 0 && lane == 0) seg_o[Mn] = Vn;
  for (int64_t m = gw; m < npos; m += nw) {
    const int64_t d = cnt[m];
    uint32_t ui, uj;
    morton_decode((uint64_t)m, ui, uj);
    const int64_t i = ui, j = uj;
    if ((d >> DT_FULL) == 0) {  // no C block here (or not owned)
      if (c_slot && lane == 0) c_slot[i * G + j] = -1;
      continue;
    }
    const int64_t v = dc_off(ctapre, lofs, m);
    const int64_t pfull = v >> DT_FULL;
    if (lane == 0) {
      keys[pfull] = i * G + j;
      if (c_slot) c_slot[i * G + j] = (int32_t)pfull;
    }
    if ((d & DT_TASK_MASK) == 0) continue;  // mirror of an emitted node
    const int64_t ntask = d & DT_TASK_MASK;
    const int64_t node = (v >> DT_NODE) & DT_IDX_MASK;
    int64_t toff = v & DT_TASK_MASK;
    if (lane == 0) {
      ci_o[node] = (int32_t)i;
      cj_o[node] = (int32_t)j;
      seg_o[node] = toff;
      if (c_out) {
        c_out[node] = pfull;
        c_mirror[node] =
            i < j ? dc_off(ctapre, lofs, (int64_t)morton_encode((uint32_t)j, (uint32_t)i)) >>
                        DT_FULL
                  : -1;
      }
      order[atomicAdd(hist + (G - ntask), 1)] = (int32_t)node;
    }
    const uint32_t* mk = kmask + m * KW;
    for (int w = 0; w < KW; ++w) {
      const unsigned mask = mk[w];
      if (mask >> lane & 1u) {
        const int64_t k = (int64_t)w * 32 + lane;
        const int64_t pos = toff + __popc(mask & lt_mask);
        K_o[pos] = (int32_t)k;
        aidx[pos] = slotA[i * G + k];
        bidx[pos] = slotB[k * G + j];
      }
      toff += __popc(mask);
    }
  }
}

bool dense_cull(const Mat& a, const Mat& b, double tau, bool want_tasks, CullResult& r,
                cudaStream_t s, bool sym, int64_t lo = 0, int64_t hi = -1,
                int32_t* work = nullptr, void (*after_launch)(void*) = nullptr,
                void* after_ctx = nullptr, bool want_slot = false,
                const int64_t* extra_src = nullptr) {
  const bool ranged = hi >= 0;
  const int depth = a.depth;
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int64_t KW = (G + 31) >> 5;
  // aux[0]: full leaf survivors, [1]: mirror mismatch, [2]: packed totals,
  // [3]: count-pass CTAs done, [4 + t]: tier-t survivors (t < depth),
  // [NEAR + t]: near-tau products of tier t (t <= depth), [MARGIN]: inverted
  // min relative margin.  [aux | LPT schedule: G + 1 length bins (bin 0 = G
  // tasks) + the K4 counter] zeroed by one memset; the schedule part is
  // handed to K4 (r.sched).
  htrace("dc_start");
  constexpr int NEAR = 4 + DENSE_MAX_DEPTH, MARGIN = NEAR + DENSE_MAX_DEPTH + 1,
                CUTS = MARGIN + 1;
  const size_t aux_bytes = (size_t)CUTS * sizeof(int64_t);
  const TieBand tb = tie_band(tau);
  char* zbuf = dmalloc<char>(aux_bytes + (G + 2) * sizeof(int), s);
  int64_t* aux = reinterpret_cast<int64_t*>(zbuf);
  int* sched = reinterpret_cast<int*>(zbuf + aux_bytes);
  const int n_leaf = (int)((npos + DC_PPC - 1) / DC_PPC);
  // cnt | lofs (npos each) | ctasum | ctapre (n_leaf each) | keep masks (npos x KW words)
  char* cbuf = dmalloc<char>((2 * npos + 2 * n_leaf) * sizeof(int64_t) +
                                 (want_tasks ? (size_t)npos * KW * sizeof(uint32_t) : 0), s);
  int64_t* cnt = reinterpret_cast<int64_t*>(cbuf);
  int64_t* lofs = cnt + npos;
  int64_t* ctasum = lofs + npos;
  int64_t* ctapre = ctasum + n_leaf;
  uint32_t* kmask = want_tasks ? reinterpret_cast<uint32_t*>(ctapre + n_leaf) : nullptr;
  SPAMM_CK(cudaMemsetAsync(zbuf, 0, aux_bytes + (G + 2) * sizeof(int), s));
  auto* u64 = reinterpret_cast<unsigned long long*>(aux);
  // gathered: aux[0..4+depth), near[0..depth], margin
  const int n_base = 4 + depth, n_near = depth + 1;
  const int nsc = n_base + n_near + 1;
  ScalarSrc src{};
  for (int i = 0; i < n_base; ++i) src.p[i] = aux + i;
  src.p[3] = nullptr;
  for (int t = 0; t < n_near; ++t) src.p[n_base + t] = aux + NEAR + t;
  src.p[n_base + n_near] = aux + MARGIN;
  const int nsc_all = nsc + (extra_src ? 1 : 0);
  if (extra_src) src.p[nsc] = extra_src;
  const int64_t tri = depth >= 2 && !ranged ? ((int64_t(1) << (3 * (depth - 1))) - 1) / 7
                      : depth == 1 && !ranged ? 1
                                              : 0;
  const int n_tier = tri > 0 ? grid_for(tri, CULL_THREADS, 148LL) : 0;
  const PinnedGather pg = pinned_gather_begin();
  static const bool cprof = getenv("SPAMM_CULL_PROF") != nullptr;
  unsigned long long* prof = nullptr;
  const int grid_c = n_leaf + n_tier;
  if (cprof) prof = dmalloc<unsigned long long>(2 * grid_c + 4, s);
  launch_pdl(k_dense_count, grid_c, CULL_THREADS, 0, s, depth, a.norms, b.norms, tau,
             sym ? 1 : 0, cnt, kmask, sched, want_tasks ? 1 : 0, u64, tb, u64 + NEAR,
             u64 + MARGIN, lo, hi, work, n_tier, ranged ? 0 : 1,
             reinterpret_cast<unsigned*>(aux + 3), lofs, ctasum, ctapre, src, nsc_all, pg.vals,
             pg.flag, pg.seq, prof);
  SPAMM_LAUNCH_CK();
  if (after_launch) after_launch(after_ctx);
  int64_t h[64];
  pinned_gather_wait(h, nsc_all, pg, s);
  if (extra_src) r.extra = h[nsc];
  if (prof) {  // diagnostics (syncs): CTA start spread, end spread, last-CTA phases
    std::vector<unsigned long long> hp(2 * grid_c + 4);
    SPAMM_CK(cudaMemcpyAsync(hp.data(), prof, hp.size() * 8, cudaMemcpyDeviceToHost, s));
    SPAMM_CK(cudaStreamSynchronize(s));
    unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
    double tier_end = 0, leaf_end = 0;
    for (int b = 0; b < grid_c; ++b) {
      s0 = std::min(s0, hp[2 * b]);
      s1 = std::max(s1, hp[2 * b]);
      e0 = std::min(e0, hp[2 * b + 1]);
      e1 = std::max(e1, hp[2 * b + 1]);
    }
    for (int b = 0; b < grid_c; ++b) {
      const double d = (double)(hp[2 * b + 1] - s0) / 1e3;
      if (b < n_tier) tier_end = std::max(tier_end, d); else leaf_end = std::max(leaf_end, d);
    }
    const unsigned long long* L = hp.data() + 2 * grid_c;
    fprintf(stderr, "[cull] us from first CTA start: starts %.2f..%.2f ends %.2f..%.2f "
            "(tiers %.2f leaf %.2f) last: begin %.2f scan %.2f hist %.2f published %.2f\n",
            0.0, (s1 - s0) / 1e3, (e0 - s0) / 1e3, (e1 - s0) / 1e3, tier_end, leaf_end,
            (L[0] - s0) / 1e3, (L[1] - s0) / 1e3, (L[2] - s0) / 1e3, (L[3] - s0) / 1e3);
    dfree(prof, s);
  }
  for (int t = 0; t < n_near; ++t) r.near[t] = h[n_base + t];
  r.margin = margin_from_bits(h[n_base + n_near]);
  if (h[1]) {  // leaf survivor set not mirror-symmetric (ulp tie): full cull
    dfree(cbuf, s);
    dfree(zbuf, s);
    return false;
  }
  const int64_t V = h[2] & DT_TASK_MASK, M = (h[2] >> DT_NODE) & DT_IDX_MASK,
                F = h[2] >> DT_FULL;
  for (int t = 0; t < depth; ++t) r.visited[t] = h[4 + t];
  r.visited[depth] = h[0];
  for (int t = 0; t <= depth; ++t)
    r.culled[t] = ranged ? 0 : (t == 0 ? 1 : 8 * r.visited[t - 1]) - r.visited[t];
  if (want_slot) r.c_slot = dmalloc<int32_t>(npos, s);
  if (!want_tasks || V == 0) {
    if (r.c_slot) SPAMM_CK(cudaMemsetAsync(r.c_slot, 0xff, npos * sizeof(int32_t), s));
    dfree(cbuf, s);
    dfree(zbuf, s);
    if (!want_tasks) r.n_tasks = r.visited[depth];
    return true;
  }
  // all outputs carved from one allocation (owned through r.block)
  // (C's keys are allocated on their own: multiply hands them to the product)
  const size_t n64 = (M + 1) + (sym ? 2 * M : 0), n32 = 2 * M + 3 * V + M;
  char* blk = dmalloc<char>(n64 * 8 + n32 * 4, s);
  int64_t* p64 = reinterpret_cast<int64_t*>(blk);
  int32_t* p32 = reinterpret_cast<int32_t*>(blk + n64 * 8);
  r.block = blk;
  r.seg = p64;
  p64 += M + 1;
  r.keys = dmalloc<int64_t>(F, s);
  if (sym) {
    r.c_out = p64;
    r.c_mirror = p64 + M;
  }
  r.ci = p32;
  r.cj = p32 + M;
  r.k = p32 + 2 * M;
  r.a_idx = r.k + V;
  r.b_idx = r.a_idx + V;
  r.order = r.b_idx + V;
  r.sched = reinterpret_cast<int*>(zbuf);  // frees the aux + schedule buffer
  r.counter = sched + G + 1;
  launch_pdl(k_dense_write, grid_for(npos * 32, CULL_THREADS, 148LL * 8), CULL_THREADS, 0, s,
             depth, sym ? 1 : 0, cnt, lofs, ctapre, kmask, sched, r.ci, r.cj, r.seg, r.k,
             a.slot, b.slot, r.a_idx, r.b_idx, r.keys, r.c_out, r.c_mirror, r.order, M, V,
             r.c_slot);
  SPAMM_LAUNCH_CK();
  dfree(cbuf, s);
  r.n_c = M;
  r.n_c_full = F;
  r.n_tasks = V;
  return true;
}

void* pinned_staging(size_t bytes) {
  static thread_local void* buf = nullptr;
  static thread_local size_t cap = 0;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    cap = std::max(bytes, cap * 2);
    SPAMM_CK(cudaMallocHost(&buf, cap));
  }
  return buf;
}

}  // namespace

void set_dense_cull(bool enabled) { g_dense_enabled = enabled; }
void set_near_tau_ulps(int k) { g_near_ulps = k; }

void CullResult::release(cudaStream_t s) {
  dfree(c_slot, s);
  c_slot = nullptr;
  if (block) {  // dense cull: every array but keys lives in one allocation
    dfree(block, s);
    dfree(sched, s);
    dfree(keys, s);
    block = nullptr;
    ci = cj = nullptr;
    seg = nullptr;
    k = a_idx = b_idx = nullptr;
    keys = c_out = c_mirror = nullptr;
    order = nullptr;
    sched = counter = nullptr;
    n_c = n_tasks = 0;
    return;
  }
  dfree(ci, s);
  dfree(cj, s);
  dfree(seg, s);
  dfree(k, s);
  dfree(a_idx, s);
  dfree(b_idx, s);
  dfree(keys, s);
  dfree(c_out, s);
  dfree(c_mirror, s);
  dfree(order, s);
  dfree(sched, s);
  ci = cj = nullptr;
  seg = nullptr;
  k = a_idx = b_idx = nullptr;
  keys = c_out = c_mirror = nullptr;
  order = nullptr;
  sched = counter = nullptr;
  n_c = n_tasks = 0;
}

bool dense_cull_applies(int depth) { return g_dense_enabled && depth <= DENSE_MAX_DEPTH; }

bool cull(const Mat& a, const Mat& b, double tau, bool want_tasks, CullResult& r, cudaStream_t s,
          bool sym, int64_t lo, int64_t hi, int32_t* work, void (*after_launch)(void*),
          void* after_ctx, bool want_slot, const int64_t* extra_src) {
  // hi < 0: no shard filter (the whole C grid)
  const int depth = a.depth;
  r.visited.assign(depth + 1, 0);
  r.culled.assign(depth + 1, 0);
  r.n_c = r.n_tasks = 0;
  r.sym = sym;
  r.near.assign(depth + 1, 0);
  r.margin = INFINITY;
  if (g_dense_enabled && depth <= DENSE_MAX_DEPTH)
    return dense_cull(a, b, tau, want_tasks, r, s, sym, lo, hi, work, after_launch, after_ctx,
                      want_slot, extra_src);

  int32_t* ci = dmalloc<int32_t>(1, s);
  int32_t* cj = dmalloc<int32_t>(1, s);
  int64_t* seg = dmalloc<int64_t>(2, s);
  int32_t* K = dmalloc<int32_t>(1, s);
  // aux[0]: survivors in diagonal C nodes (symmetric mode), aux[1]: mirror
  // mismatch flag, aux[2]: packed scan total (root count first), aux[3]:
  // diagonal C nodes with survivors, aux[4]: near-tau products of the tier,
  // aux[5]: inverted min relative margin (tie_probe; kept across tiers).
  int64_t* aux = dmalloc<int64_t>(6, s);
  SPAMM_CK(cudaMemsetAsync(aux, 0, 6 * sizeof(int64_t), s));
  const TieBand tb = tie_band(tau);
  auto* u64 = reinterpret_cast<unsigned long long*>(aux);
  int32_t* aidx = nullptr;
  int32_t* bidx = nullptr;
  int64_t V = 0, M = 0, full_prev = 0, diag_nodes = 0;
  int t0 = 0;
  const int T0 = std::min(a.top_t, b.top_t);
  if (T0 >= 1 && T0 < depth) {
    event_wait(a.top_ev);
    event_wait(b.top_ev);
    HostLevel L;
    if (!host_cull_top(a.host_top, b.host_top, T0, depth, tau, sym, lo, hi, r, L, full_prev,
                       diag_nodes, tb)) {
      dfree(ci, s);
      dfree(cj, s);
      dfree(seg, s);
      dfree(K, s);
      dfree(aux, s);
      return false;
    }
    M = (int64_t)L.ci.size();
    V = (int64_t)L.K.size();
    t0 = T0;
    for (int t = T0 + 1; t <= depth; ++t) r.visited[t] = r.culled[t] = 0;
    dfree(ci, s);
    dfree(cj, s);
    dfree(seg, s);
    dfree(K, s);
    ci = cj = K = nullptr;
    seg = nullptr;
    if (V > 0) {
      ci = dmalloc<int32_t>(M, s);
      cj = dmalloc<int32_t>(M, s);
      seg = dmalloc<int64_t>(M + 1, s);
      K = dmalloc<int32_t>(V, s);
      const size_t b1 = M * 4, b2 = (M + 1) * 8, b3 = V * 4;
      char* st = static_cast<char*>(pinned_staging(2 * b1 + b2 + b3));
      memcpy(st, L.ci.data(), b1);
      memcpy(st + b1, L.cj.data(), b1);
      memcpy(st + 2 * b1, L.seg.data(), b2);
      memcpy(st + 2 * b1 + b2, L.K.data(), b3);
      SPAMM_CK(cudaMemcpyAsync(ci, st, b1, cudaMemcpyHostToDevice, s));
      SPAMM_CK(cudaMemcpyAsync(cj, st + b1, b1, cudaMemcpyHostToDevice, s));
      SPAMM_CK(cudaMemcpyAsync(seg, st + 2 * b1, b2, cudaMemcpyHostToDevice, s));
      SPAMM_CK(cudaMemcpyAsync(K, st + 2 * b1 + b2, b3, cudaMemcpyHostToDevice, s));
    }
  } else {
    if (depth == 0 && want_tasks) {
      aidx = dmalloc<int32_t>(1, s);
      bidx = dmalloc<int32_t>(1, s);
    }
    k_cull_root<<<1, 1, 0, s>>>(a.norms, b.norms, tau, ci, cj, seg, K, aux + 2, a.slot, b.slot,
                                aidx, bidx, tb, u64 + 4, u64 + 5);
    SPAMM_LAUNCH_CK();
    int64_t h0[6];
    d2h_sync(h0, aux, 6, s);
    V = h0[2];
    r.near[0] = h0[4];
    r.margin = margin_from_bits(h0[5]);
    r.visited[0] = V;
    r.culled[0] = 1 - V;
    M = V;
    full_prev = V;  // the root node is diagonal: full count == emitted count
    diag_nodes = V;
  }

  auto free_level = [&]() {
    dfree(ci, s);
    dfree(cj, s);
    dfree(seg, s);
    dfree(K, s);
    dfree(aidx, s);
    dfree(bidx, s);
    ci = cj = nullptr;
    seg = nullptr;
    K = aidx = bidx = nullptr;
  };

  int t = t0;
  for (; V > 0 && t < depth; ++t) {
    const int t1 = t + 1;
    const bool leaf = t1 == depth;
    int64_t* cnt4 = dmalloc<int64_t>(4 * M, s);
    int64_t* off4 = dmalloc<int64_t>(4 * M + 1, s);
    SPAMM_CK(cudaMemsetAsync(aux, 0, 5 * sizeof(int64_t), s));
    k_cull_expand<false, false><<<cull_grid(M), CULL_THREADS, 0, s>>>(
        t1, a.norms, b.norms, tau, M, ci, cj, seg, K, cnt4, nullptr, nullptr, nullptr, nullptr,
        nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, sym ? 1 : 0, u64, lo, hi,
        2 * (depth - t1), leaf ? work : nullptr, tb);
    SPAMM_LAUNCH_CK();
    scan_exclusive_i64(cnt4, 4 * M, off4, s);
    SPAMM_CK(cudaMemcpyAsync(aux + 2, off4 + 4 * M, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    int64_t h[6];
    d2h_sync(h, aux, 6, s);
    diag_nodes = h[3];
    r.near[t1] = h[4];
    r.margin = std::min(r.margin, margin_from_bits(h[5]));
    if (h[1]) {  // survivor set not symmetric: the caller falls back to the full cull
      dfree(cnt4, s);
      dfree(off4, s);
      free_level();
      dfree(aux, s);
      return false;
    }
    const int64_t packed = h[2];
    const int64_t Vn = packed & TASK_MASK, Mn = packed >> NODE_SHIFT;
    const int64_t full = sym ? 2 * Vn - h[0] : Vn;
    r.visited[t1] = full;
    r.culled[t1] = 8 * full_prev - full;
    full_prev = full;
    if (Vn == 0 || (leaf && !want_tasks)) {
      dfree(cnt4, s);
      dfree(off4, s);
      free_level();
      V = Vn;
      M = Mn;
      t = t1;
      break;
    }
    int32_t* ci_o = dmalloc<int32_t>(Mn, s);
    int32_t* cj_o = dmalloc<int32_t>(Mn, s);
    int64_t* seg_o = dmalloc<int64_t>(Mn + 1, s);
    int32_t* K_o = dmalloc<int32_t>(Vn, s);
    int32_t* ai = nullptr;
    int32_t* bi = nullptr;
    if (leaf) {
      ai = dmalloc<int32_t>(Vn, s);
      bi = dmalloc<int32_t>(Vn, s);
      k_cull_expand<true, true><<<cull_grid(M), CULL_THREADS, 0, s>>>(
          t1, a.norms, b.norms, tau, M, ci, cj, seg, K, nullptr, off4, ci_o, cj_o, seg_o, K_o,
          a.slot, b.slot, ai, bi, Mn, Vn, sym ? 1 : 0, nullptr, lo, hi, 2 * (depth - t1), work,
          tb);
    } else {
      k_cull_expand<true, false><<<cull_grid(M), CULL_THREADS, 0, s>>>(
          t1, a.norms, b.norms, tau, M, ci, cj, seg, K, nullptr, off4, ci_o, cj_o, seg_o, K_o,
          nullptr, nullptr, nullptr, nullptr, Mn, Vn, sym ? 1 : 0, nullptr, lo, hi,
          2 * (depth - t1), nullptr, tb);
    }
    SPAMM_LAUNCH_CK();
    dfree(cnt4, s);
    dfree(off4, s);
    free_level();
    ci = ci_o;
    cj = cj_o;
    seg = seg_o;
    K = K_o;
    aidx = ai;
    bidx = bi;
    V = Vn;
    M = Mn;
  }
  dfree(aux, s);
  // Tiers after an early exit keep zero counts (kernel.py:114-117).
  if (V > 0 && want_tasks && ci != nullptr) {
    r.n_c = M;
    r.n_c_full = sym ? 2 * M - diag_nodes : M;
    r.n_tasks = V;
    r.ci = ci;
    r.cj = cj;
    r.seg = seg;
    r.k = K;
    r.a_idx = aidx;
    r.b_idx = bidx;
  } else {
    free_level();
    if (!want_tasks) r.n_tasks = r.visited[depth];
  }
  return true;
}

}  // namespace spamm
