// K4 (Nb = 32 / 64): persistent, warp-specialised FP64-DMMA leaf products.
//
// Reference: _gemm_acc / _gemm_batch (kernel.py:64-77).  Same contract as
// leaf.cu: segment m (tasks of one C block, k ascending) is reduced by ONE
// CTA in registers, in task order -> deterministic, no atomics.
//
// B200 mapping
//  * one producer warp: a single lane issues TMA tiled loads
//    (cp.async.bulk.tensor.2d, SWIZZLE_128B, box 16 x Nb doubles) of the
//    A_ik / B_kj leaf blocks into a STAGES-deep smem ring, completion through
//    mbarrier transaction counts (full[]), slot reuse through empty[];
//  * CONSUMERS warps: FP64 tensor cores via mma.sync.m8n8k4.f64 (DMMA; sm_100a
//    has no f64 tcgen05 kind), fragments read from the swizzled tiles,
//    accumulators in registers; the epilogue of C block m overlaps the TMA
//    loads of block m + grid;
//  * persistent grid (min(#segments, SMs x CTAs/SM)), static round-robin over
//    the Morton-ordered C blocks.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace spamm {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// L2 cache-policy variants (hint bit 0: operand tiles evict_last; bit 1:
// product stores evict_first).
__device__ __forceinline__ void tma_load_2d_pol(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                int c0, int c1, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st2_pol(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st1_pol(double* p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

// A stage holds the k-range [h KH, (h + 1) KH) of one task, KH = NB / KS:
// A as KH/16 column slabs of NB rows, B as NB/16 column slabs of KH rows (so
// KS = 2 gives twice the stages of half the size: finer-grained refills and
// a deeper look-ahead in the same shared memory).
template <int NB, int WARPS_M, int WARPS_N, int STAGES, int KS = 1>
struct TmaCfg {
  static constexpr int CONSUMERS = WARPS_M * WARPS_N;
  static constexpr int THREADS = 32 * (CONSUMERS + 1);
  static constexpr int KH = NB / KS;                 // k-extent of a stage
  static constexpr int SLAB = NB * 128;              // A: one 16-column slab, NB rows
  static constexpr int SLAB_B = KH * 128;            // B: one 16-column slab, KH rows
  static constexpr int A_BYTES = (KH / 16) * SLAB;
  static constexpr int STAGE = A_BYTES + (NB / 16) * SLAB_B;   // = 2 NB KH 8
  static constexpr size_t SMEM = (size_t)STAGES * STAGE + 1024 + 3 * STAGES * 8 + 64;
};

// Byte offset of element (r, c) inside a swizzled tile: 16-column slabs of
// NB rows x 128 B, 16-byte chunk index XOR (r mod 8) (TMA SWIZZLE_128B).
template <int NB>
__host__ __device__ constexpr int swz(int r, int c) {
  return (c >> 4) * (NB * 128) + r * 128 + ((((c & 15) >> 1) ^ (r & 7)) << 4) + ((c & 1) << 3);
}

template <int NB, int WARPS_M, int WARPS_N, int STAGES, int KS, bool PAIRK, class Idx>
__global__ void __launch_bounds__(32 * (WARPS_M * WARPS_N + 1), 1)
    k_leaf_dmma_tma(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    int64_t n_seg, const int64_t* __restrict__ seg, const Idx* __restrict__ a_idx,
                    const Idx* __restrict__ b_idx, const int64_t* __restrict__ c_out,
                    const int64_t* __restrict__ c_mirror, int accumulate, double* __restrict__ C,
                    const int32_t* __restrict__ order, int* __restrict__ next_block, int hint) {
  pdl_wait();
  using Cfg = TmaCfg<NB, WARPS_M, WARPS_N, STAGES, KS>;
  constexpr int KH = Cfg::KH;
  constexpr int WTM = NB / WARPS_M, WTN = NB / WARPS_N, MT = WTM / 8, NT = WTN / 8;
  static_assert(WTN % 8 == 0 && WTM % 8 == 0, "warp tile must be a multiple of 8");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SWIZZLE_128B needs 1024-B alignment
  const uint32_t bars = base + STAGES * Cfg::STAGE;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (STAGES + s); };
  // Per-stage work descriptor written by the producer: (C segment << 2) |
  // first-task bit | last-task bit, or -1 = no more work (sentinel stage).
  int64_t* meta = reinterpret_cast<int64_t*>(smem_raw + (bars + 16u * STAGES - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), Cfg::CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == Cfg::CONSUMERS) {
    // ---------------- producer warp ----------------
    // Dynamic scheduling: C segments are taken from a global counter in
    // longest-first order (LPT), so the tail of the launch is one short block.
    // The whole warp runs the loop (lane 0 issues barriers and TMA): task
    // indices are loaded 32 at a time, coalesced, and handed out by shuffle,
    // and the next block is claimed and its bounds loaded while the current
    // one streams -- no global-load latency between two stages (this bound
    // the Nb = 32 kernel, whose stages are only ~500 cycles of DMMA).
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    int stage = 0;
    uint32_t phase = 0;
    auto claim = [&](int64_t& m, int64_t& t0, int64_t& t1) -> bool {
      int64_t i = 0;
      if (lane == 0) i = atomicAdd(next_block, 1);
      i = __shfl_sync(0xffffffffu, i, 0);
      if (i >= n_seg) return false;
      m = order ? (int64_t)order[i] : i;
      t0 = seg[m];
      t1 = seg[m + 1];
      return true;
    };
    int64_t m = 0, t0 = 0, t1 = 0;
    bool have = claim(m, t0, t1);
    while (have) {
      int64_t mn = 0, t0n = 0, t1n = 0;
      const bool next = claim(mn, t0n, t1n);  // in flight while this block streams
      for (int64_t c0 = t0; c0 < t1; c0 += 32) {
        const int64_t t = c0 + lane;
        const int ra_l = t < t1 ? (int)a_idx[t] * NB : 0;
        const int rb_l = t < t1 ? (int)b_idx[t] * NB : 0;
        const int cnt = t1 - c0 < 32 ? (int)(t1 - c0) : 32;
        for (int q = 0; q < cnt; ++q) {
          const int ra = __shfl_sync(0xffffffffu, ra_l, q);
          const int rb = __shfl_sync(0xffffffffu, rb_l, q);
#pragma unroll 1
          for (int h = 0; h < KS; ++h) {
            mbar_wait(empty(stage), phase ^ 1u);
            if (lane == 0) {
              const int64_t tq = c0 + q;
              meta[stage] = (m << 2) | (tq == t0 && h == 0 ? 1 : 0) |
                            (tq + 1 == t1 && h == KS - 1 ? 2 : 0);
              mbar_expect_tx(full(stage), Cfg::STAGE);
              const uint32_t sa = base + stage * Cfg::STAGE, sb = sa + Cfg::A_BYTES;
#pragma unroll
              if (hint & 1) {
                const uint64_t pol = policy_evict_last();
#pragma unroll
                for (int sl = 0; sl < KH / 16; ++sl)
                  tma_load_2d_pol(sa + sl * Cfg::SLAB, &tmA, full(stage), h * KH + sl * 16, ra, pol);
#pragma unroll
                for (int sl = 0; sl < NB / 16; ++sl)
                  tma_load_2d_pol(sb + sl * Cfg::SLAB_B, &tmB, full(stage), sl * 16, rb + h * KH,
                                  pol);
              } else {
#pragma unroll
                for (int sl = 0; sl < KH / 16; ++sl)
                  tma_load_2d(sa + sl * Cfg::SLAB, &tmA, full(stage), h * KH + sl * 16, ra);
#pragma unroll
                for (int sl = 0; sl < NB / 16; ++sl)
                  tma_load_2d(sb + sl * Cfg::SLAB_B, &tmB, full(stage), sl * 16, rb + h * KH);
              }
            }
            __syncwarp();
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1u;
            }
          }
        }
      }
      have = next;
      m = mn;
      t0 = t0n;
      t1 = t1n;
    }
    mbar_wait(empty(stage), phase ^ 1u);
    if (lane == 0) {
      meta[stage] = -1;
      mbar_arrive(full(stage));
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int r8 = lane >> 2, c4 = lane & 3;
  const int row0 = wm * WTM, col0 = wn * WTN;
  // Lane-constant swizzle offsets (see swz): A by (kk & 15) >> 2, B by (half, kk & 4).
  uint32_t offA[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    offA[q] = (uint32_t)((((2 * q + (c4 >> 1)) ^ r8) << 4) + ((c4 & 1) << 3) + r8 * 128);
  uint32_t offB[2][2];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int g = 0; g < 2; ++g)
      offB[h][g] = (uint32_t)((((h * 4 + (r8 >> 1)) ^ (g * 4 + c4)) << 4) + ((r8 & 1) << 3) + c4 * 128);
  // Paired k-steps (PAIRK): steps 2t / 2t+1 take the even / odd columns of
  // the 8-column group t, so a lane's two A values are one 16-byte chunk
  // (one LDS.128 instead of two LDS.64); B rows follow the same k order.
  // PAIRN (with PAIRK, two 8-column n-tiles per warp): tile nt takes the
  // columns col0 + 2 q + nt, so a lane's two B values (tiles 0 and 1) are one
  // 16-byte chunk, and its four C values of a row are contiguous.
  // (measured: +3.8 % at Nb = 32, where K4 is shared-load bound; -4 % at
  //  Nb = 64, so only the former uses it)
  constexpr bool PAIRN = PAIRK && NT == 2 && WTN == 16 && NB == 32;
  uint32_t offBn[2];
#pragma unroll
  for (int o = 0; o < 2; ++o)
    offBn[o] = (uint32_t)(((r8 ^ (2 * c4 + o)) << 4) + (2 * c4 + o) * 128);
  auto ccol = [&](int nt, int e) {  // C column held in acc[.][nt][e]
    return PAIRN ? col0 + 4 * c4 + 2 * e + nt : col0 + nt * 8 + 2 * c4 + e;
  };
  uint32_t offA2[2], offBp[2][2];
#pragma unroll
  for (int t = 0; t < 2; ++t)
    offA2[t] = (uint32_t)((((4 * t + c4) ^ r8) << 4) + r8 * 128);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int o = 0; o < 2; ++o)
      offBp[h][o] = (uint32_t)((((h * 4 + (r8 >> 1)) ^ (2 * c4 + o)) << 4) + ((r8 & 1) << 3) +
                               (2 * c4 + o) * 128);

  int stage = 0, held = -1;
  uint32_t phase = 0;
  double acc[MT][NT][2];
  for (;;) {
    mbar_wait(full(stage), phase);
    // Stage release: the previous stage is handed back only here, after the
    // wait loop -- every DMMA that read it was issued in the preceding basic
    // block, and an issued DMMA has its fragments.  (Releasing right after
    // the k-loop let the arrive be scheduled above the final DMMAs, and a fast
    // refill could overwrite fragments still in flight.)
    if (held >= 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(empty(held));
    }
    const int64_t md = meta[stage];
    if (md < 0) break;
    const int64_t m = md >> 2;
    double* Cb = C + (c_out ? c_out[m] : m) * (int64_t)(NB * NB);
    if (md & 1) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          if (accumulate && PAIRN) {
            const double* row = Cb + (row0 + mt * 8 + r8) * NB;
            acc[mt][nt][0] = row[ccol(nt, 0)];
            acc[mt][nt][1] = row[ccol(nt, 1)];
          } else if (accumulate) {
            const double2 v = *reinterpret_cast<const double2*>(
                Cb + (row0 + mt * 8 + r8) * NB + col0 + nt * 8 + 2 * c4);
            acc[mt][nt][0] = v.x;
            acc[mt][nt][1] = v.y;
          } else {
            acc[mt][nt][0] = 0.0;
            acc[mt][nt][1] = 0.0;
          }
        }
    }
    const uint32_t sa = base + stage * Cfg::STAGE, sb = sa + Cfg::A_BYTES;
    if (PAIRK) {
#pragma unroll
      for (int k8 = 0; k8 < KH; k8 += 8) {
        double ae[MT], ao[MT], be[NT], bo[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const double2 v = lds128(sa + (k8 >> 4) * Cfg::SLAB + (row0 + mt * 8) * 128 +
                                   offA2[(k8 >> 3) & 1]);
          ae[mt] = v.x;
          ao[mt] = v.y;
        }
        if (PAIRN) {
          const uint32_t rowb = sb + (col0 >> 4) * Cfg::SLAB_B + k8 * 128;
          const double2 ve = lds128(rowb + offBn[0]), vo = lds128(rowb + offBn[1]);
          be[0] = ve.x;
          be[NT - 1] = ve.y;
          bo[0] = vo.x;
          bo[NT - 1] = vo.y;
        } else {
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int cb = col0 + nt * 8;
            const uint32_t rowb = sb + (cb >> 4) * Cfg::SLAB_B + k8 * 128;
            be[nt] = lds64(rowb + offBp[(cb >> 3) & 1][0]);
            bo[nt] = lds64(rowb + offBp[(cb >> 3) & 1][1]);
          }
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], ae[mt], be[nt]);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], ao[mt], bo[nt]);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < KH; kk += 4) {
        double af[MT], bf[NT];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
          af[mt] = lds64(sa + (kk >> 4) * Cfg::SLAB + (row0 + mt * 8) * 128 + offA[(kk >> 2) & 3]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int cb = col0 + nt * 8;
          bf[nt] = lds64(sb + (cb >> 4) * Cfg::SLAB_B + kk * 128 + offB[(cb >> 3) & 1][(kk >> 2) & 1]);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], af[mt], bf[nt]);
      }
    }
    held = stage;  // handed back after the next wait (see the release above)
    if (++stage == STAGES) {
      stage = 0;
      phase ^= 1u;
    }
    if (!(md & 2)) continue;
    // last task of this C block: epilogue
    const bool ef = hint & 2;
    const uint64_t spol = ef ? policy_evict_first() : 0;
    if (PAIRN) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        double* row = Cb + (row0 + mt * 8 + r8) * NB + col0 + 4 * c4;
        if (ef) {
          st2_pol(row, make_double2(acc[mt][0][0], acc[mt][NT - 1][0]), spol);
          st2_pol(row + 2, make_double2(acc[mt][0][1], acc[mt][NT - 1][1]), spol);
        } else {
          *reinterpret_cast<double2*>(row) = make_double2(acc[mt][0][0], acc[mt][NT - 1][0]);
          *reinterpret_cast<double2*>(row + 2) = make_double2(acc[mt][0][1], acc[mt][NT - 1][1]);
        }
      }
    } else if (ef) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          st2_pol(Cb + (row0 + mt * 8 + r8) * NB + col0 + nt * 8 + 2 * c4,
                  make_double2(acc[mt][nt][0], acc[mt][nt][1]), spol);
    } else {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          double2 v;
          v.x = acc[mt][nt][0];
          v.y = acc[mt][nt][1];
          *reinterpret_cast<double2*>(Cb + (row0 + mt * 8 + r8) * NB + col0 + nt * 8 + 2 * c4) = v;
        }
    }
    // The stores above consumed every accumulator, so every DMMA -- and every
    // fragment read of the held stage -- is complete: hand the stage back now
    // rather than after the mirror stores and the next wait.
    __syncwarp();
    if (lane == 0) mbar_arrive(empty(held));
    held = -1;
    // Symmetric product: the mirror block C_ji = C_ij^T (bitwise what the full
    // product computes).
    const int64_t mi = c_mirror ? c_mirror[m] : -1;
    if (mi >= 0) {
      double* Cm = C + mi * (int64_t)(NB * NB);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int r = row0 + mt * 8 + r8;
          if (PAIRN) {
            if (ef) {
              st1_pol(Cm + ccol(nt, 0) * NB + r, acc[mt][nt][0], spol);
              st1_pol(Cm + ccol(nt, 1) * NB + r, acc[mt][nt][1], spol);
            } else {
              Cm[ccol(nt, 0) * NB + r] = acc[mt][nt][0];
              Cm[ccol(nt, 1) * NB + r] = acc[mt][nt][1];
            }
          } else {
            const int c = col0 + nt * 8 + 2 * c4;
            if (ef) {
              st1_pol(Cm + c * NB + r, acc[mt][nt][0], spol);
              st1_pol(Cm + (c + 1) * NB + r, acc[mt][nt][1], spol);
            } else {
              Cm[c * NB + r] = acc[mt][nt][0];
              Cm[(c + 1) * NB + r] = acc[mt][nt][1];
            }
          }
        }
    }
  }
}

// LPT order of the C segments: counting sort by task count, longest first.
// (Order within equal lengths is arbitrary: it only changes which CTA runs a
// block, never its result.)
__global__ void k_len_hist(const int64_t* __restrict__ seg, int64_t n, int maxlen,
                           int* __restrict__ hist) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = seg[m + 1] - seg[m];
    atomicAdd(hist + (l < maxlen ? maxlen - l : 0), 1);  // bin 0 = longest
  }
}

// Exclusive scan of the (maxlen + 1)-bin histogram, one 1024-thread CTA.
__global__ void __launch_bounds__(1024) k_hist_scan(int* __restrict__ hist, int nbins) {
  pdl_wait();
  __shared__ int warp_tot[32];
  const int per = (nbins + 1023) / 1024, b0 = threadIdx.x * per;
  int loc = 0;
  for (int b = b0; b < b0 + per && b < nbins; ++b) loc += hist[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = warp_tot[lane], wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += v;
    }
    warp_tot[lane] = wi - w;
  }
  __syncthreads();
  int run = warp_tot[warp] + inc - loc;
  for (int b = b0; b < b0 + per && b < nbins; ++b) {
    const int c = hist[b];
    hist[b] = run;
    run += c;
  }
}

__global__ void k_len_scatter(const int64_t* __restrict__ seg, int64_t n, int maxlen,
                              int* __restrict__ start, int32_t* __restrict__ order) {
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = seg[m + 1] - seg[m];
    order[atomicAdd(start + (l < maxlen ? maxlen - l : 0), 1)] = (int32_t)m;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

CUtensorMap make_map(const double* data, int64_t nblocks, int nb, int box_rows) {
  CUtensorMap m;
  const int64_t rows = nblocks > 0 ? nblocks * nb : nb;
  cuuint64_t dims[2] = {(cuuint64_t)nb, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)nb * sizeof(double)};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(data), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    SPAMM_CK(cudaGetDevice(&dev));
    SPAMM_CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

template <int NB, int WM, int WN, int ST, int CTAS_PER_SM, int KS, bool PAIRK, class Idx>
void launch_tma(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                const int64_t* c_out, const int64_t* c_mirror, bool acc, const double* A,
                int64_t a_blocks, const double* B, int64_t b_blocks, double* C, cudaStream_t s,
                LptSchedule lpt) {
  using Cfg = TmaCfg<NB, WM, WN, ST, KS>;
  auto kern = k_leaf_dmma_tma<NB, WM, WN, ST, KS, PAIRK, Idx>;
  static std::once_flag once;
  std::call_once(once, [&] {
    SPAMM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  });
  const CUtensorMap ta = make_map(A, a_blocks, NB, NB), tb = make_map(B, b_blocks, NB, NB / KS);
  int64_t grid = (int64_t)sm_count() * CTAS_PER_SM;
  if (grid > n_seg) grid = n_seg;
  int* scratch = nullptr;
  const int32_t* order = lpt.order;
  int* counter = lpt.counter;
  static const int order_mode = [] {  // experiment switch: 1 = Morton order (no LPT)
    const char* v = getenv("SPAMM_K4_ORDER");
    return v && strcmp(v, "morton") == 0 ? 1 : 0;
  }();
  if (order_mode == 1) {
    scratch = dmalloc<int>(1, s);
    SPAMM_CK(cudaMemsetAsync(scratch, 0, sizeof(int), s));
    counter = scratch;
    order = nullptr;
  } else if (!order) {
    scratch = lpt_schedule(n_seg, seg, &order, &counter, s);
  }
  static const int hint = [] {  // L2 policy bits (see tma_load_2d_pol)
    const char* v = getenv("SPAMM_K4_HINT");
    const char* pv = getenv("SPAMM_L2_PERSIST");
    if (pv && atoi(pv) > 0) {  // evict_last lines live in the persisting set-aside
      int dev = 0, mx = 0;
      SPAMM_CK(cudaGetDevice(&dev));
      SPAMM_CK(cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev));
      const size_t want = std::min<size_t>((size_t)mx, (size_t)atoi(pv) << 20);
      SPAMM_CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
      size_t got = 0;
      SPAMM_CK(cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize));
      fprintf(stderr, "[spamm] persisting L2 set-aside %zu MiB (max %d MiB)\n", got >> 20, mx >> 20);
    }
    return v ? atoi(v) : 0;
  }();
  launch_pdl(kern, (unsigned)grid, Cfg::THREADS, Cfg::SMEM, s, ta, tb, n_seg, seg, a_idx, b_idx, c_out,
                                                       c_mirror, acc ? 1 : 0, C, order, counter,
                                                       hint);
  SPAMM_LAUNCH_CK();
  dfree(scratch, s);
}

}  // namespace

bool tma_leaf_supported(int nb) { return nb == 32 || nb == 64; }

int multiprocessors() { return sm_count(); }

int* lpt_schedule(int64_t n_seg, const int64_t* seg, const int32_t** order, int** counter,
                  cudaStream_t s) {
  // scratch: [next-block counter | length histogram (maxlen + 1 bins) | LPT order]
  const int maxlen = 4096;
  int* scratch = dmalloc<int>(1 + (maxlen + 1) + n_seg, s);
  int* hist = scratch + 1;
  int32_t* ord = scratch + 2 + maxlen;
  SPAMM_CK(cudaMemsetAsync(scratch, 0, (2 + maxlen) * sizeof(int), s));
  k_len_hist<<<grid_for(n_seg, 256), 256, 0, s>>>(seg, n_seg, maxlen, hist);
  SPAMM_LAUNCH_CK();
  launch_pdl(k_hist_scan, 1, 1024, 0, s, hist, maxlen + 1);
  SPAMM_LAUNCH_CK();
  k_len_scatter<<<grid_for(n_seg, 256), 256, 0, s>>>(seg, n_seg, maxlen, hist, ord);
  SPAMM_LAUNCH_CK();
  *order = ord;
  *counter = scratch;
  return scratch;
}

template <class Idx>
void leaf_products_tma(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                       const int64_t* c_out, const int64_t* c_mirror, bool accumulate,
                       const double* A, int64_t a_blocks, const double* B, int64_t b_blocks,
                       double* C, int nb, cudaStream_t s, LptSchedule lpt) {
  if (n_seg <= 0) return;
  // (KS = 2 -- twice the stages at half the k-extent -- measured slower for both:
  //  33.2 vs 34.9 TF/s at Nb = 64, 26.6 vs 29.4 at Nb = 32: more barrier
  //  round trips per flop outweigh the deeper look-ahead.)
  // PAIRK (paired k-steps, one LDS.128 per two A fragments): +0.4 % on cfg4,
  // A/B-measured over 3 alternating runs (35.02 vs 34.88 TF/s).
  if (nb == 64)
    launch_tma<64, 2, 4, 3, 1, 1, true, Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror,
                                             accumulate, A, a_blocks, B, b_blocks, C, s, lpt);
  else if (nb == 32)  // 4 CTAs/SM x 4 consumer warps (fastest of 9 measured configurations)
    launch_tma<32, 2, 2, 3, 4, 1, true, Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror,
                                             accumulate, A, a_blocks, B, b_blocks, C, s, lpt);
  else
    throw CudaError("TMA leaf kernel needs block size 32 or 64");
}

void hist_scan_exclusive(int* hist, int nbins, cudaStream_t s) {
  launch_pdl(k_hist_scan, 1, 1024, 0, s, hist, nbins);
  SPAMM_LAUNCH_CK();
}

template void leaf_products_tma<int32_t>(int64_t, const int64_t*, const int32_t*, const int32_t*,
                                         const int64_t*, const int64_t*, bool, const double*,
                                         int64_t, const double*, int64_t, double*, int,
                                         cudaStream_t, LptSchedule);
template void leaf_products_tma<int64_t>(int64_t, const int64_t*, const int64_t*, const int64_t*,
                                         const int64_t*, const int64_t*, bool, const double*,
                                         int64_t, const double*, int64_t, double*, int,
                                         cudaStream_t, LptSchedule);

}  // namespace spamm
