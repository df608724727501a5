// K6: fused SP2 update.
//
// Reference: sp2._step (sp2.py:92-101) and BASELINE cfg3's idempotency test
// ||X^2 - X||_F = add_scaled(1.0, X2, -1.0, X).norm() (quadtree.py:281-293).
// The reference materialises X^2 - X (a full matrix, norms rebuilt) just to
// read its root norm, then materialises 2X - X^2 for an EXPAND step.  Here one
// warp-per-block pass over the key union of X and X^2 reads each operand
// block once and produces
//   D = fl(fl(1*x2) + fl(-1*x))   -> leaf norm^2 only (never written),
//   E = fl(fl(2*x)  + fl(-1*x2))  -> written, with leaf norm^2 + nonzero flag,
// with exactly the reference's rounding (absent operand = no term) and the
// einsum norm recipe (lanes 0/1 chain D, lanes 2/3 chain E).  The D pyramid
// is reduced to its root with the same tier order as any other matrix.
// HBM roofline: reads 2 S Nb^2 8 B, writes S Nb^2 8 B (EXPAND).
#include "internal.h"
#include "ozaki_common.cuh"

namespace spamm {

namespace {

__global__ void k_union_keys(const int32_t* __restrict__ sa, const int32_t* __restrict__ sb,
                             int depth, uint8_t* __restrict__ flags) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npos;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    const int64_t key = (int64_t)bi * G + bj;
    flags[p] = (sa[key] >= 0 || sb[key] >= 0) ? 1 : 0;
  }
}

__global__ void k_union_compact(const uint8_t* __restrict__ flags, const int64_t* __restrict__ off,
                                int depth, int64_t* __restrict__ keys) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npos;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[p]) continue;
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    keys[off[p]] = (int64_t)bi * G + bj;
  }
}

// Small trees (G*G <= 16384): union flags, scan and compaction in one CTA
// (1024 threads x PER consecutive Morton positions, all slot loads in flight).
template <int PER>
__global__ void __launch_bounds__(1024)
    k_union_small(const int32_t* __restrict__ sa, const int32_t* __restrict__ sb, int depth,
                  int64_t* __restrict__ keys, int64_t* __restrict__ count) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  int64_t key[PER];
  int f[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int64_t p = (int64_t)threadIdx.x * PER + j;
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    key[j] = (int64_t)bi * G + bj;
  }
  int fs = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const bool ok = (int64_t)threadIdx.x * PER + j < npos;
    const int32_t va = ok ? sa[key[j]] : -1, vb = ok ? sb[key[j]] : -1;
    f[j] = (va >= 0) | (vb >= 0);
    fs += f[j];
  }
  int64_t tot = 0;
  int64_t o = cta_exclusive_scan(fs, &tot);
#pragma unroll
  for (int j = 0; j < PER; ++j)
    if (f[j]) keys[o++] = key[j];
  if (threadIdx.x == 0) *count = tot;
}

// Trace-first SP2 pre-branch pass (one CTA, one launch): tr X^2 from the
// diagonal blocks of the unfinalised product (the cull's slot map) in the
// trace()'s order (each block's diagonal summed in order, then the blocks in
// order: k_trace_blocks + k_trace), the key union of X and X^2 with its size
// (k_union_small), and tr X copied from its finalisation if not cached --
// all published to pinned memory for the branch rule (gather_sync protocol).
template <int NB, int NPER>
__global__ void __launch_bounds__(1024)
    k_tf_prebranch(const int32_t* __restrict__ xslot, const int32_t* __restrict__ cslot,
                   const double* __restrict__ cdata, int depth,
                   int64_t* __restrict__ ukeys, const double* __restrict__ xtr_dev,
                   double* __restrict__ ctr_out, int64_t* __restrict__ ucount_out,
                   int64_t* gvals, int64_t* gflag, int64_t seq,
                   unsigned long long* __restrict__ prof) {
  auto gtime = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (prof && threadIdx.x == 0) prof[0] = gtime();
  pdl_wait();
  if (prof && threadIdx.x == 0) prof[1] = gtime();
  __shared__ double partial[16 * NPER];  // G <= 16 NPER (small trees: G <= 128)
  __shared__ unsigned char present[16 * NPER];
  __shared__ int64_t wtot[17];
  constexpr int NV = NB / 32;  // diagonal values per lane and block
  const int64_t G = int64_t(1) << depth, npos = G * G;
  constexpr int64_t nb2 = (int64_t)NB * NB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < 16) {
    // warps 0-15: tr X^2.  Warp w takes blocks w, w + 16, ... (NPER); all slot
    // and diagonal loads are issued before the (sequential, per block) sums,
    // whose chains are interleaved across the warp's blocks.
    const int64_t bl = warp + 16 * (int64_t)lane;
    const int32_t sl_l = lane < NPER && bl < G ? cslot[bl * G + bl] : -1;
    double v[NPER][NV];
    int32_t sl[NPER];
#pragma unroll
    for (int q = 0; q < NPER; ++q) {
      sl[q] = __shfl_sync(0xffffffffu, sl_l, q);
      const bool ok = sl[q] >= 0;
      const double* x = cdata + (int64_t)(ok ? sl[q] : 0) * nb2;
#pragma unroll
      for (int u = 0; u < NV; ++u) v[q][u] = ok ? x[(int64_t)(lane + 32 * u) * (NB + 1)] : 0.0;
    }
    if (prof && threadIdx.x == 0) prof[2] = gtime();
    double acc[NPER];
#pragma unroll
    for (int q = 0; q < NPER; ++q) acc[q] = 0.0;
    // (fully unrolled: the shuffles run ahead of the dependent add chains)
#pragma unroll
    for (int u = 0; u < NV; ++u)
#pragma unroll
      for (int i = 0; i < 32; ++i) {
#pragma unroll
        for (int q = 0; q < NPER; ++q)
          acc[q] = __dadd_rn(acc[q], __shfl_sync(0xffffffffu, v[q][u], i));
      }
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < NPER; ++q) {
        const int64_t b = warp + 16 * q;
        if (b < G) {
          present[b] = sl[q] >= 0;
          partial[b] = acc[q];
        }
      }
    }
    if (prof && threadIdx.x == 0) prof[3] = gtime();
  } else {
    // warps 16-31: the key union of X and X^2 (Morton order) and its size;
    // thread t owns positions t NP .. t NP + NP - 1 (NP <= 32: a bit mask)
    const int t = threadIdx.x - 512;
    constexpr int NP = NPER * NPER / 2 > 0 ? NPER * NPER / 2 : 1;  // npos / 512, <= 32
    constexpr int NB8 = NP < 8 ? NP : 8;  // slot loads in flight per batch
    uint32_t fm = 0;
#pragma unroll
    for (int j0 = 0; j0 < NP; j0 += NB8) {
      int32_t va[NB8], vb[NB8];
#pragma unroll
      for (int u = 0; u < NB8; ++u) {
        const int64_t p = (int64_t)t * NP + j0 + u;
        uint32_t bi, bj;
        morton_decode((uint64_t)p, bi, bj);
        const int64_t key = (int64_t)bi * G + bj;
        const bool ok = p < npos;
        va[u] = ok ? xslot[key] : -1;
        vb[u] = ok ? cslot[key] : -1;
      }
#pragma unroll
      for (int u = 0; u < NB8; ++u)
        if ((va[u] >= 0) | (vb[u] >= 0)) fm |= 1u << (j0 + u);
    }
    const int fs = __popc(fm);
    int64_t x = fs;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wtot[warp - 16] = x;
    asm volatile("bar.sync 1, 512;\n" ::: "memory");
    if (warp == 16) {
      const int64_t w = lane < 16 ? wtot[lane] : 0;
      int64_t z = w;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      if (lane < 16) wtot[lane] = z - w;
      if (lane == 15) wtot[16] = z;
    }
    asm volatile("bar.sync 1, 512;\n" ::: "memory");
    if (prof && threadIdx.x == 512) prof[4] = gtime();
    int64_t o = wtot[warp - 16] + x - fs;
    while (fm) {
      const int j = __ffs(fm) - 1;
      fm &= fm - 1;
      uint32_t bi, bj;
      morton_decode((uint64_t)((int64_t)t * NP + j), bi, bj);  // (NP as above)
      ukeys[o++] = (int64_t)bi * G + bj;
    }
  }
  __syncthreads();
  if (prof && threadIdx.x == 0) prof[5] = gtime();
  if (threadIdx.x == 0) {
    const int64_t tot = wtot[16];
    double tr = 0.0;
    for (int64_t b0 = 0; b0 < G; b0 += 16) {  // (shared loads batched ahead of the chain)
      double pv[16];
      bool pp[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        pp[u] = b0 + u < G && present[b0 + u];
        pv[u] = pp[u] ? partial[b0 + u] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (pp[u]) tr = __dadd_rn(tr, pv[u]);
    }
    *ctr_out = tr;
    *ucount_out = tot;
    gvals[0] = __double_as_longlong(tr);
    gvals[1] = xtr_dev ? __double_as_longlong(*xtr_dev) : 0;
    gvals[2] = tot;
    if (prof) prof[6] = gtime();
    __threadfence_system();
    *reinterpret_cast<volatile int64_t*>(gflag) = seq;
    if (prof) prof[7] = gtime();
  }
}

// K6: BPW union blocks per warp; D = fl(fl(1*x2) + fl(-1*x)) (norm^2 only) and
// E = fl(fl(2*x) + fl(-1*x2)) (written) with exactly the reference's rounding
// (absent operand = no term); the D and E chains of all of them run on lanes
// 0 .. 4 BPW - 1 (lane = 4 q + 2 set + parity) over the permuted parity rows
// (common.cuh).
template <int NB2, bool IDEM, bool EXPAND, int BPW, int WARPS>
__global__ void __launch_bounds__(32 * WARPS)
    k_sp2_update_multi(const int64_t* __restrict__ ukeys, int64_t U, const double* __restrict__ X,
                       const int32_t* __restrict__ sx, const double* __restrict__ X2,
                       const int32_t* __restrict__ sx2, double* __restrict__ E,
                       double* __restrict__ nD2, double* __restrict__ nE2,
                       uint8_t* __restrict__ nzE, double* __restrict__ nE1,
                       int* __restrict__ ex_col, int64_t G) {
  pdl_wait();
  constexpr int NCH = NB2 / 256;
  constexpr int NB = NB2 == 4096 ? 64 : 32;
  __shared__ __align__(16) double rows_all[WARPS][BPW * 4 * CHAIN_ROW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* rows = rows_all[warp];
  const int64_t stride = (int64_t)gridDim.x * WARPS * BPW;
  for (int64_t u0 = ((int64_t)blockIdx.x * WARPS + warp) * BPW; u0 < U; u0 += stride) {
    const double2* px[BPW];
    const double2* px2[BPW];
    double2* pe[BPW];
    double2 a[BPW][4], b[BPW][4];
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      px[q] = px2[q] = nullptr;
      pe[q] = nullptr;
      if (u0 + q < U) {
        const int64_t key = ukeys[u0 + q];
        const int32_t ix = sx[key], ix2 = sx2[key];
        if (ix >= 0) px[q] = reinterpret_cast<const double2*>(X + (int64_t)ix * NB2);
        if (ix2 >= 0) px2[q] = reinterpret_cast<const double2*>(X2 + (int64_t)ix2 * NB2);
        if (EXPAND) pe[q] = reinterpret_cast<double2*>(E + (u0 + q) * NB2);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        a[q][k] = px[q] ? __ldg(px[q] + k * 32 + lane) : make_double2(0.0, 0.0);
        b[q][k] = px2[q] ? __ldg(px2[q] + k * 32 + lane) : make_double2(0.0, 0.0);
      }
    }
    double acc = 0.0;
    unsigned anyq = 0;
    double cm[BPW][2];  // E's K4z column maxima (ex_col)
#pragma unroll
    for (int q = 0; q < BPW; ++q) cm[q][0] = cm[q][1] = 0.0;
    for (int c = 0; c < NCH; ++c) {
      __syncwarp();
#pragma unroll
      for (int q = 0; q < BPW; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double d0, d1, e0, e1;
          // D = add_scaled(1.0, X2, -1.0, X): first operand X2, second X
          d0 = px2[q] ? __dmul_rn(1.0, b[q][k].x) : 0.0;
          d1 = px2[q] ? __dmul_rn(1.0, b[q][k].y) : 0.0;
          if (px[q]) {
            d0 = __dadd_rn(d0, __dmul_rn(-1.0, a[q][k].x));
            d1 = __dadd_rn(d1, __dmul_rn(-1.0, a[q][k].y));
          }
          // E = add_scaled(2.0, X, -1.0, X2): first operand X, second X2
          e0 = px[q] ? __dmul_rn(2.0, a[q][k].x) : 0.0;
          e1 = px[q] ? __dmul_rn(2.0, a[q][k].y) : 0.0;
          if (px2[q]) {
            e0 = __dadd_rn(e0, __dmul_rn(-1.0, b[q][k].x));
            e1 = __dadd_rn(e1, __dmul_rn(-1.0, b[q][k].y));
          }
          double* rq = rows + q * 4 * CHAIN_ROW + chain_pos(k, lane);
          if (IDEM) {
            rq[0] = __dmul_rn(d0, d0);
            rq[CHAIN_ROW] = __dmul_rn(d1, d1);
          }
          if (EXPAND) {
            rq[2 * CHAIN_ROW] = __dmul_rn(e0, e0);
            rq[3 * CHAIN_ROW] = __dmul_rn(e1, e1);
            if (pe[q]) pe[q][c * 128 + k * 32 + lane] = make_double2(e0, e1);
            if ((e0 != 0.0) | (e1 != 0.0)) anyq |= 1u << q;
            if (ex_col) {
              cm[q][0] = fmax(cm[q][0], ozk::oz_absf(e0));
              cm[q][1] = fmax(cm[q][1], ozk::oz_absf(e1));
            }
          }
        }
      __syncwarp();
      if (c + 1 < NCH) {
#pragma unroll
        for (int q = 0; q < BPW; ++q)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (px[q]) a[q][k] = __ldg(px[q] + (c + 1) * 128 + k * 32 + lane);
            if (px2[q]) b[q][k] = __ldg(px2[q] + (c + 1) * 128 + k * 32 + lane);
          }
      }
      const int set = (lane >> 1) & 1;
      if (lane < 4 * BPW && (set ? EXPAND : IDEM))
        acc = chain_row128(rows + lane * CHAIN_ROW, acc);
    }
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      const double d0 = __shfl_sync(0xffffffffu, acc, 4 * q);
      const double d1 = __shfl_sync(0xffffffffu, acc, 4 * q + 1);
      const double e0 = __shfl_sync(0xffffffffu, acc, 4 * q + 2);
      const double e1 = __shfl_sync(0xffffffffu, acc, 4 * q + 3);
      const bool any = __any_sync(0xffffffffu, (anyq >> q) & 1u);
      if (lane == 0 && u0 + q < U) {
        if (IDEM) nD2[u0 + q] = __dadd_rn(d0, d1);
        if (EXPAND) {
          const double v = __dadd_rn(e0, e1);
          nE2[u0 + q] = v;
          if (nE1) nE1[u0 + q] = __dsqrt_rn(v);
          nzE[u0 + q] = any ? 1 : 0;
        }
      }
      if (EXPAND && ex_col && u0 + q < U)
        ozk::oz_col_exponents<NB>(cm[q][0], cm[q][1], ukeys[u0 + q] % G, ex_col, lane);
    }
  }
}

template <int NB2>
void launch_update(bool idem, bool expand, const int64_t* ukeys, int64_t U, const Mat& x,
                   const Mat& x2, double* E, double* nD2, double* nE2, uint8_t* nzE,
                   cudaStream_t s, double* nE1, int* ex_col) {
  constexpr int BPW = 2, WARPS = 4;
  const int grid = grid_for((U + BPW - 1) / BPW * 32, 32 * WARPS, 1LL << 20);
  if (idem && expand)
    launch_pdl(k_sp2_update_multi<NB2, true, true, BPW, WARPS>, grid, 32 * WARPS, 0, s,
        ukeys, U, x.data, x.slot, x2.data, x2.slot, E, nD2, nE2, nzE, nE1, ex_col, x.G);
  else if (idem)
    launch_pdl(k_sp2_update_multi<NB2, true, false, BPW, WARPS>, grid, 32 * WARPS, 0, s,
        ukeys, U, x.data, x.slot, x2.data, x2.slot, E, nD2, nE2, nzE, nE1, ex_col, x.G);
  else
    launch_pdl(k_sp2_update_multi<NB2, false, true, BPW, WARPS>, grid, 32 * WARPS, 0, s,
        ukeys, U, x.data, x.slot, x2.data, x2.slot, E, nD2, nE2, nzE, nE1, ex_col, x.G);
  SPAMM_LAUNCH_CK();
}

}  // namespace

void sp2_update(const Mat& x, const Mat& x2, bool want_idem, bool expand, double* idem_norm,
                Mat& e, cudaStream_t s) {
  const int nb2 = x.nb * x.nb;
  if (!want_idem && !expand) return;
  if (nb2 != 1024 && nb2 != 4096) {
    // Generic block sizes: the unfused reference sequence.
    if (want_idem) {
      Mat d;
      add_scaled(1.0, x2, -1.0, x, d, s);
      int64_t bits = 0;
      d2h_sync(&bits, reinterpret_cast<const int64_t*>(d.norms), 1, s);
      memcpy(idem_norm, &bits, sizeof(double));
      d.release();
    }
    if (expand) add_scaled(2.0, x, -1.0, x2, e, s);
    return;
  }
  int64_t* u_dev = dmalloc<int64_t>(1, s);
  UnionPrep prep = sp2_union_prepare(x, x2, u_dev, s);
  int64_t U = 0;
  d2h_sync(&U, u_dev, 1, s);
  dfree(u_dev, s);
  sp2_update_finish(x, x2, prep, U, want_idem, expand, idem_norm, e, s);
}

bool sp2_fused_supported(int nb) { return nb == 32 || nb == 64; }

UnionPrep tf_prebranch(const Mat& x, const Mat& c, double* ctr_dev, int64_t* u_dev,
                       int64_t* host3, cudaStream_t s) {
  UnionPrep p;
  p.npos = x.G * x.G;
  p.keys = dmalloc<int64_t>(p.npos, s);
  const double* xtr = x.tr_valid ? nullptr : x.tr_dev;
  const PinnedGather g = pinned_gather_begin();
  static const bool tprof = getenv("SPAMM_TF_PROF") != nullptr;
  unsigned long long* prof = tprof ? dmalloc<unsigned long long>(8, s) : nullptr;
  auto go = [&](auto kern) {
    launch_pdl(kern, 1, 1024, 0, s, (const int32_t*)x.slot, (const int32_t*)c.slot,
               (const double*)c.data, x.depth, p.keys, xtr, ctr_dev, u_dev, g.vals, g.flag, g.seq,
               prof);
  };
  const int nper = x.G <= 16 ? 1 : (int)(x.G / 16);  // G <= 128
  if (x.nb == 64) {
    if (nper == 1) go(k_tf_prebranch<64, 1>);
    else if (nper == 2) go(k_tf_prebranch<64, 2>);
    else if (nper == 4) go(k_tf_prebranch<64, 4>);
    else go(k_tf_prebranch<64, 8>);
  } else {
    if (nper == 1) go(k_tf_prebranch<32, 1>);
    else if (nper == 2) go(k_tf_prebranch<32, 2>);
    else if (nper == 4) go(k_tf_prebranch<32, 4>);
    else go(k_tf_prebranch<32, 8>);
  }
  SPAMM_LAUNCH_CK();
  pinned_gather_wait(host3, 3, g, s);
  if (prof) {  // diagnostics (syncs)
    unsigned long long h[8];
    SPAMM_CK(cudaMemcpyAsync(h, prof, sizeof h, cudaMemcpyDeviceToHost, s));
    SPAMM_CK(cudaStreamSynchronize(s));
    fprintf(stderr, "[tf] us: waited %.2f loads %.2f chains %.2f union %.2f joined %.2f "
            "summed %.2f published %.2f\n", (h[1] - h[0]) / 1e3, (h[2] - h[1]) / 1e3,
            (h[3] - h[1]) / 1e3, (h[4] - h[1]) / 1e3, (h[5] - h[1]) / 1e3, (h[6] - h[1]) / 1e3,
            (h[7] - h[1]) / 1e3);
    dfree(prof, s);
  }
  return p;
}

UnionPrep sp2_union_prepare(const Mat& x, const Mat& x2, int64_t* u_dev, cudaStream_t s) {
  UnionPrep p;
  p.npos = x.G * x.G;
  if (x.depth <= SMALL_TREE_DEPTH) {
    p.keys = dmalloc<int64_t>(p.npos, s);
    if (x.depth <= 6)
      k_union_small<4><<<1, 1024, 0, s>>>(x.slot, x2.slot, x.depth, p.keys, u_dev);
    else
      k_union_small<16><<<1, 1024, 0, s>>>(x.slot, x2.slot, x.depth, p.keys, u_dev);
    SPAMM_LAUNCH_CK();
    return p;
  }
  p.flags = dmalloc<uint8_t>(p.npos, s);
  p.off = dmalloc<int64_t>(p.npos + 1, s);
  k_union_keys<<<grid_for(p.npos, 256), 256, 0, s>>>(x.slot, x2.slot, x.depth, p.flags);
  SPAMM_LAUNCH_CK();
  scan_exclusive_u8(p.flags, p.npos, p.off, s);
  SPAMM_CK(cudaMemcpyAsync(u_dev, p.off + p.npos, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  return p;
}

void sp2_update_finish(const Mat& x, const Mat& x2, UnionPrep& prep, int64_t U, bool want_idem,
                       bool expand, double* idem_norm, Mat& e, cudaStream_t s, bool settle_now,
                       void (*after_update)(void*), void* after_ctx, bool want_oz_ex,
                       double* idem_dev_out) {
  const int nb2 = x.nb * x.nb;
  int64_t* ukeys = prep.keys;
  prep.keys = nullptr;
  if (!ukeys) ukeys = dmalloc<int64_t>(U, s);
  if (U > 0 && prep.flags) {
    k_union_compact<<<grid_for(prep.npos, 256), 256, 0, s>>>(prep.flags, prep.off, x.depth, ukeys);
    SPAMM_LAUNCH_CK();
  }
  dfree(prep.flags, s);
  dfree(prep.off, s);
  prep.flags = nullptr;
  prep.off = nullptr;
  if (!want_idem && !expand) {
    dfree(ukeys, s);
    return;
  }
  double* nD2 = want_idem ? dmalloc<double>(U, s) : nullptr;
  double* nE2 = expand ? dmalloc<double>(U, s) : nullptr;
  double* nE1 = expand ? dmalloc<double>(U, s) : nullptr;
  uint8_t* nzE = expand ? dmalloc<uint8_t>(U, s) : nullptr;
  double* E = expand ? dmalloc<double>((size_t)U * nb2, s) : nullptr;
  // E's K4z row exponents (= its column exponents: E is bitwise symmetric
  // when X and X^2 are), so E's first multiply skips its exponent pass
  int* ex = nullptr;
  if (expand && want_oz_ex && x.sym && x2.sym) {
    ex = dmalloc<int>(x.G * x.nb, s);
    SPAMM_CK(cudaMemsetAsync(ex, 0x80, x.G * x.nb * sizeof(int), s));
  }
  if (U > 0) {
    if (nb2 == 4096)
      launch_update<4096>(want_idem, expand, ukeys, U, x, x2, E, nD2, nE2, nzE, s, nE1, ex);
    else
      launch_update<1024>(want_idem, expand, ukeys, U, x, x2, E, nD2, nE2, nzE, s, nE1, ex);
  }
  double* pn = nullptr;
  // (trace-first SP2: E's finalisation reduces the residual's leaf tier too)
  const bool resid_in_fin = want_idem && expand && idem_dev_out && idem_fusable(x);
  if (want_idem && !resid_in_fin) {
    const int64_t ps = pyramid_size(x.depth);
    pn = dmalloc<double>(2 * ps, s);
    build_pyramid(ukeys, nD2, U, x.depth, pn, pn + ps, s);
    dfree(nD2, s);
  }
  if (expand) {
    e.n_native = x.n_native;
    e.nb = x.nb;
    e.chunk_size = x.chunk_size;
    e.depth = x.depth;
    e.G = x.G;
    e.nblocks = U;
    e.data = E;
    e.keys = ukeys;
    e.sym = x.sym && x2.sym;
    e.stream = s;
    e.oz_ex_row = ex;
    if (after_update) after_update(after_ctx);
    if (resid_in_fin) {
      finalize_with_residual(e, s, nE2, nzE, nE1, nD2, idem_dev_out);
      dfree(nD2, s);
      want_idem = false;  // (delivered on the device)
    } else {
      finalize(e, s, nE2, nzE, /*defer=*/true, nE1);
    }
  } else {
    dfree(ukeys, s);
  }
  // idem_dev_out (trace-first SP2): the residual stays on the device (read
  // at a later sync), and so does E's kept count (settle_now = false)
  if (want_idem && idem_dev_out) {
    SPAMM_CK(cudaMemcpyAsync(idem_dev_out, pn, sizeof(double), cudaMemcpyDeviceToDevice, s));
    want_idem = false;
  }
  // One host sync for the idempotency norm and E's kept-block count.
  const int64_t* kept_dev = expand && settle_now ? pending_kept(e) : nullptr;
  if (want_idem || kept_dev) {
    const int64_t* src[2] = {want_idem ? reinterpret_cast<const int64_t*>(pn) : nullptr, kept_dev};
    int64_t h[2] = {0, 0};
    gather_sync(h, src, 2, s);
    if (want_idem) memcpy(idem_norm, &h[0], sizeof(double));
    if (kept_dev) settle(e, h[1], s);
  }
  dfree(pn, s);
}

}  // namespace spamm
