// K4z for Nb = 32: the same exact signed-8-bit digit products as leaf_ozaki.cu
// (scheme, scales and digit split described there), laid out for 32x32 blocks.
//
// A 32-row block gives 32 TMEM lanes per digit slice, so one 128-lane MMA
// operand stacks FOUR slices (p .. p+3) of A and one 128-column operand four
// slices of B: a single tcgen05.mma (M = N = 128, K = 32 = the whole block)
// forms 16 digit pairs.  Three MMAs per leaf product -- anchors (0,0), (0,4),
// (4,0) -- form every pair with p + q <= 7 exactly once (and some with
// p + q <= 10), into two 128-column tiles whose 32x32 sub-blocks (i, j) hold
// digit sum D + i + j (D = 0 for the first, 4 for the other two).  Two tiles
// are 256 TMEM columns, so two CTAs fit on an SM (the default shape: the
// epilogue of one CTA overlaps the MMAs of the other), or one CTA can
// double-buffer its accumulators.
//
// Epilogue: the 16 sub-blocks of a C element (r, c) live in four TMEM lane
// quarters (one per warp) and four column groups; each warp loads its quarter
// and folds its own 8 sub-blocks into two exact int64 (Th, Tl: the digit sums
// d <= 4 and 5..8 at their weights, as in leaf_ozaki.cu), the pairs go through
// shared memory (16 KB), and the owning thread adds the four warps' pairs
// (exact) and rounds once (oz_round2) -- so results are deterministic and a
// symmetric X gives a bitwise symmetric X*X.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "internal.h"
#include "ozaki_common.cuh"

namespace spamm {

namespace {

using namespace ozk;

constexpr int Z_NB = 32;
constexpr int Z_SLICES = 8;
constexpr int Z_SLICE_BYTES = Z_NB * Z_NB;                 // 1 KB
constexpr int Z_BLOCK_BYTES = Z_SLICES * Z_SLICE_BYTES;    // 8 KB
// A stage holds up to Z_TPS tasks of one accumulation chunk (A and B slices
// of each): one barrier round trip per Z_TPS tasks -- with only 3 MMAs per
// task (~200 tensor cycles) the per-task synchronisation would otherwise
// dominate.
constexpr int Z_TASK = 2 * Z_BLOCK_BYTES;                  // 16 KB
// Kernel shapes: NBUF accumulator sets of 256 TMEM columns (2: double
// buffered, one CTA per SM; 1: two CTAs per SM share the 512 columns),
// STAGES x TPS tasks of operand ring.
// Epilogue exchange: per warp w, column c8 and row r one exact int64 pair
// (Th, Tl) -- the warp's own 8 sub-blocks already folded -- 16 KB.
constexpr int Z_XBUF = 2 * 4 * 8 * 32 * 8;                 // [H/L][w][c8][r] int64
constexpr int Z_PAD = 128;    // base alignment (no-swizzle operands need 16 B)
template <int NBUF, int TPS, int STAGES>
struct ZCfg {
  static constexpr int STAGE = TPS * Z_TASK;
  static constexpr size_t SMEM = Z_PAD + (size_t)STAGES * STAGE + Z_XBUF + 512;
  static constexpr int CTAS = NBUF == 2 ? 1 : 2;
  // two CTAs per SM: 228 KB per SM, 1 KB reserved per CTA
  static_assert(CTAS == 1 || 2 * (SMEM + 1024) <= 233472, "two CTAs do not fit an SM");
};
constexpr int Z_CHUNK = 128;  // tasks per accumulation: |sub-block| <= 128 x 32 x 2^14 = 2^26
constexpr int Z_EPI = 128;    // 4 epilogue warps = the 4 TMEM lane quarters
constexpr int Z_THREADS = Z_EPI + 64;
constexpr uint32_t Z_SBO = 256;  // 8-row group stride: 2 k-chunks x 128 B

// element (n, k) of a 32x32 slice: 8-row x 16-byte core matrices, the two
// k-chunks of a row group adjacent (LBO 128 B), row groups 256 B apart -- four
// consecutive slices form one 128-row operand.
__host__ __device__ constexpr int z_off(int n, int k) {
  return (n >> 3) * 256 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15);
}

// ex[g] = max exponent over global row g (by_col = 0) / column g (by_col = 1):
// thread t of a 256-thread CTA: block 4 s' + t / 64, line (t % 64) / 2, half t % 2.
__global__ void __launch_bounds__(256) k_oz32_exponents(const double* __restrict__ data,
                                                        const int64_t* __restrict__ keys,
                                                        int64_t nblocks, int64_t G, int by_col,
                                                        int* __restrict__ ex) {
  pdl_wait();
  const int t = threadIdx.x, sub = t >> 6, line = (t & 63) >> 1, half = t & 1;
  for (int64_t s0 = (int64_t)blockIdx.x * 4; s0 < nblocks; s0 += (int64_t)gridDim.x * 4) {
    const int64_t s = s0 + sub;
    double mx = 0.0;
    int64_t key = 0;
    if (s < nblocks) {
      const double* b = data + s * (Z_NB * Z_NB);
      key = keys[s];
      if (by_col) {
#pragma unroll
        for (int i = 0; i < 16; ++i) mx = fmax(mx, oz_absf(b[(half * 16 + i) * Z_NB + line]));
      } else {
        // pairs half, half + 2, ...: a lane pair reads one whole sector per load
        const double2* q = reinterpret_cast<const double2*>(b + line * Z_NB) + half;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double2 v = q[2 * i];
          mx = fmax(mx, fmax(oz_absf(v.x), oz_absf(v.y)));
        }
      }
    }
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    if (s < nblocks && half == 0 && mx > 0.0)
      atomicMax(ex + (by_col ? key % G : key / G) * Z_NB + line, oz_exp_of(mx));
  }
}

// out + s * 8 KB: the 8 digit slices of block s (trans: B role, slice row n =
// block column n).  Thread t: block 4 s' + t / 64, slice row (t % 64) / 2,
// k = 16 (t % 2) .. +15.
__global__ void __launch_bounds__(256) k_oz32_split(const double* __restrict__ data,
                                                    const int64_t* __restrict__ keys,
                                                    int64_t nblocks, int64_t G, int trans,
                                                    const int* __restrict__ ex,
                                                    int8_t* __restrict__ out) {
  pdl_wait();
  const int t = threadIdx.x, sub = t >> 6, n = (t & 63) >> 1, kc = t & 1;
  for (int64_t s0 = (int64_t)blockIdx.x * 4; s0 < nblocks; s0 += (int64_t)gridDim.x * 4) {
    const int64_t s = s0 + sub;
    if (s >= nblocks) continue;
    const double* b = data + s * (Z_NB * Z_NB);
    double y[16];
    if (trans) {
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = b[(kc * 16 + i) * Z_NB + n];
    } else {
      // coalesced: lane pair (kc = 0, 1) loads pairs kc + 2i (one sector per
      // load), then swaps the halves the other lane needs -- lane kc ends
      // with pairs 8 kc .. 8 kc + 7 (k = 16 kc .. 16 kc + 15)
      const double2* q = reinterpret_cast<const double2*>(b + n * Z_NB) + kc;
      double2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = q[2 * i];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        // lane 0 keeps v[i] (pair 2i) and receives lane 1's v[i] (pair 2i + 1);
        // lane 1 keeps v[i + 4] (pair 2i + 9) and receives lane 0's v[i + 4] (pair 2i + 8)
        const double2 send = kc ? v[i] : v[i + 4];
        const double2 keep = kc ? v[i + 4] : v[i];
        double2 got;
        got.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
        got.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
        const double2 lo = kc ? got : keep, hi = kc ? keep : got;
        y[4 * i] = lo.x;
        y[4 * i + 1] = lo.y;
        y[4 * i + 2] = hi.x;
        y[4 * i + 3] = hi.y;
      }
    }
    const int64_t key = keys[s];
    const int e = oz_exp(ex[(trans ? key % G : key / G) * Z_NB + n]);
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint64_t d = oz_digits(y[i], e);
      hi[i] = (uint32_t)(d >> 32);
      lo[i] = (uint32_t)d;
    }
    int8_t* o = out + s * Z_BLOCK_BYTES + z_off(n, kc * 16);
#pragma unroll
    for (int p = 0; p < Z_SLICES; ++p) {
      const uint32_t* h = p < 4 ? hi : lo;
      const int byte = 3 - (p & 3);
      *reinterpret_cast<uint4*>(o + p * Z_SLICE_BYTES) =
          make_uint4(oz_gather4(h[0], h[1], h[2], h[3], byte),
                     oz_gather4(h[4], h[5], h[6], h[7], byte),
                     oz_gather4(h[8], h[9], h[10], h[11], byte),
                     oz_gather4(h[12], h[13], h[14], h[15], byte));
    }
  }
}

__constant__ int c_z_narrow = 0;  // 1: three N = 128 MMAs per product (SPAMM_K4Z_HINT bit 2)
__device__ __forceinline__ bool z_wide_mma() { return c_z_narrow == 0; }

template <class Idx, int NBUF, int Z_TPS, int Z_STAGES>
__global__ void __launch_bounds__(Z_THREADS, NBUF == 2 ? 1 : 2)
    k_leaf_ozaki32(int64_t n_seg, const int64_t* __restrict__ seg, const Idx* __restrict__ a_idx,
                   const Idx* __restrict__ b_idx, const int32_t* __restrict__ b_tr,
                   const int64_t* __restrict__ a_keys, const int64_t* __restrict__ b_keys,
                   int64_t G, const int8_t* __restrict__ As, const int8_t* __restrict__ Bs,
                   const int* __restrict__ ex_a, const int* __restrict__ ex_b,
                   const int64_t* __restrict__ c_out, const int64_t* __restrict__ c_mirror,
                   int accumulate, double* __restrict__ C, const int32_t* __restrict__ order,
                   int* __restrict__ next_block, const double* __restrict__ Ad,
                   const double* __restrict__ Bd, int* __restrict__ ex_out) {
  pdl_wait();
  constexpr int Z_STAGE = ZCfg<NBUF, Z_TPS, Z_STAGES>::STAGE;
  constexpr uint32_t TCOLS = 256u * NBUF;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + (Z_PAD - 1)) & ~(uint32_t)(Z_PAD - 1);
  uint8_t* gbase = smem_raw + (base - raw);
  long long* xh = reinterpret_cast<long long*>(gbase + Z_STAGES * Z_STAGE);
  long long* xl = xh + 4 * 8 * 32;
  const uint32_t bars = base + Z_STAGES * Z_STAGE + Z_XBUF;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (Z_STAGES + s); };
  auto tfull = [&](int b) { return bars + 8u * (2 * Z_STAGES + b); };
  auto tempty = [&](int b) { return bars + 8u * (2 * Z_STAGES + 2 + b); };
  int64_t* meta = reinterpret_cast<int64_t*>(gbase + Z_STAGES * Z_STAGE + Z_XBUF +
                                             8 * (2 * Z_STAGES + 4));
  int64_t* meta2 = meta + Z_STAGES;  // (bi << 32) | bj of the chunk starting in this stage
  int64_t* ring = meta2 + Z_STAGES;  // per accumulator buffer: meta, meta2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Z_STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull(b), 2);  // MMA completion (commit) + the ring entry
      mbar_init(tempty(b), Z_EPI / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)), "r"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 4) {
    // ---------------- producer: two 8-KB bulk copies per task, Z_TPS per stage ----------------
    int stage = 0, slot = 0, n_in = 0;
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
      const bool next = claim(mn, t0n, t1n);
      for (int64_t c0 = t0; c0 < t1; c0 += 32) {
        const int64_t t = c0 + lane;
        int64_t ra_l = 0, rb_l = 0;
        if (t < t1) {
          ra_l = (int64_t)a_idx[t];
          rb_l = (int64_t)b_idx[t];
          if (b_tr) rb_l = b_tr[rb_l];
        }
        const int cnt = t1 - c0 < 32 ? (int)(t1 - c0) : 32;
        for (int q = 0; q < cnt; ++q) {
          const int64_t ra = __shfl_sync(0xffffffffu, ra_l, q);
          const int64_t rb = __shfl_sync(0xffffffffu, rb_l, q);
          const int64_t tq = c0 + q, r = tq - t0;
          if (slot == 0) {  // open a stage: up to Z_TPS tasks of this chunk
            const int64_t cend = t0 + (r / Z_CHUNK + 1) * Z_CHUNK;
            const int64_t left = (cend < t1 ? cend : t1) - tq;
            n_in = left < Z_TPS ? (int)left : Z_TPS;
            mbar_wait(empty(stage), phase ^ 1u);
            if (lane == 0) {
              const bool first = r % Z_CHUNK == 0;
              const bool last = tq + n_in == t1 || (r + n_in) % Z_CHUNK == 0;
              const bool cont = r >= Z_CHUNK || accumulate;
              // bit 8: the chunk ends the C block's segment
              meta[stage] = (m << 9) | ((int64_t)n_in << 3) | (first ? 1 : 0) | (last ? 2 : 0) |
                            (cont ? 4 : 0) | (tq + n_in == t1 ? 256 : 0);
              if (first)
                meta2[stage] = ((a_keys[a_idx[tq]] / G) << 32) | (b_keys[b_idx[tq]] % G);
              mbar_expect_tx(full(stage), (uint32_t)(n_in * Z_TASK));
            }
          }
          if (lane == 0) {
            const uint32_t sa = base + stage * Z_STAGE + slot * Z_TASK;
            bulk_g2s(sa, As + ra * Z_BLOCK_BYTES, Z_BLOCK_BYTES, full(stage));
            bulk_g2s(sa + Z_BLOCK_BYTES, Bs + rb * Z_BLOCK_BYTES, Z_BLOCK_BYTES, full(stage));
          }
          __syncwarp();
          if (++slot == n_in) {
            slot = 0;
            if (++stage == Z_STAGES) {
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
  } else if (warp == 5) {
    // ---------------- MMA issuer: one thread, 3 MMAs per task ----------------
    if (lane == 0) {
      static_assert(Z_NB == 32, "");
      const bool wide = z_wide_mma();
      int stage = 0, nchunk = 0;
      uint32_t phase = 0, tph[2] = {0u, 0u};
      int64_t cur2 = 0;
      for (;;) {
        mbar_wait(full(stage), phase);
        tc_after();
        const int64_t md = meta[stage];
        const int b = NBUF == 2 ? (nchunk & 1) : 0;
        if (md < 0) {
          mbar_wait(tempty(b), tph[b] ^ 1u);  // the epilogue is done with this buffer
          ring[2 * b] = -1;
          mbar_arrive(tfull(b));
          oz_commit(tfull(b));
          break;
        }
        const bool first = md & 1;
        const int n_in = (int)((md >> 3) & 31);
        if (first) {
          cur2 = meta2[stage];
          mbar_wait(tempty(b), tph[b] ^ 1u);  // accumulator buffer b drained
          tph[b] ^= 1u;
          tc_after();
        }
        const uint32_t d0 = tbase + 256u * b;
        for (int q = 0; q < n_in; ++q) {
          const uint32_t sa = base + stage * Z_STAGE + q * Z_TASK, sb = sa + Z_BLOCK_BYTES;
          const uint32_t init = (first && q == 0) ? 0u : 1u;
          if (wide) {  // anchors (0,0) and (0,4) as one N = 256 MMA over tiles 0-1
            oz_mma(d0, oz_desc(sa, Z_SBO), oz_desc(sb, Z_SBO), init, OZ_IDESC_N256);
          } else {
            oz_mma(d0, oz_desc(sa, Z_SBO), oz_desc(sb, Z_SBO), init);
            oz_mma(d0 + 128u, oz_desc(sa, Z_SBO), oz_desc(sb + 4 * Z_SLICE_BYTES, Z_SBO), init);
          }
          oz_mma(d0 + 128u, oz_desc(sa + 4 * Z_SLICE_BYTES, Z_SBO), oz_desc(sb, Z_SBO), 1u);
        }
        oz_commit(empty(stage));
        if (md & 2) {
          ring[2 * b] = md;
          ring[2 * b + 1] = cur2;
          mbar_arrive(tfull(b));
          oz_commit(tfull(b));
          ++nchunk;
        }
        if (++stage == Z_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp w = TMEM lane quarter w = A slice offset ----------------
    const int w = warp, r = lane;
    const uint32_t lane_base = tbase + ((uint32_t)(w * 32) << 16);
    uint32_t eph[2] = {0u, 0u};
    for (int nchunk = 0;; ++nchunk) {
      const int b = NBUF == 2 ? (nchunk & 1) : 0;
      mbar_wait(tfull(b), eph[b]);
      eph[b] ^= 1u;
      tc_after();
      const int64_t md = ring[2 * b];
      if (md < 0) break;
      const int64_t bij = ring[2 * b + 1];
      const int64_t m = md >> 9;
      const bool cont = md & 4, seg_end = md & 256;
      const int64_t bi = bij >> 32, bj = bij & 0xffffffffLL;
      const int exr = ex_a[bi * Z_NB + r];
      const bool row_bad = exr == OZ_EXP_BAD;
      const int er = (row_bad ? 0 : oz_exp(exr)) - 14;
      double* Cb = C + (c_out ? c_out[m] : m) * (int64_t)(Z_NB * Z_NB);
      const int64_t mi = c_mirror ? c_mirror[m] : -1;
      double* Cm = mi >= 0 ? C + mi * (int64_t)(Z_NB * Z_NB) : nullptr;
      const uint32_t tb = lane_base + 256u * b;
      // ex_out: the product's own row exponents (see leaf_ozaki.cu)
      const bool want_ex = ex_out != nullptr && seg_end;
      unsigned rcode = 0u;
      unsigned cc0 = 0, cc1 = 0, cc2 = 0, cc3 = 0;  // per chunk: 2 column codes (registers)
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        int V[2][4][8];  // [tile][j][c8] of TMEM lane (w, r)
#pragma unroll
        for (int T = 0; T < 2; ++T)
#pragma unroll
          for (int j = 0; j < 4; ++j) tmem_ld8(tb + 128u * T + 32u * j + 8u * cc, V[T][j]);
        tmem_wait8(V[0][0]);
#pragma unroll
        for (int T = 0; T < 2; ++T)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (T || j) tmem_keep8(V[T][j]);
        if (cc == 3) {  // every TMEM read of this buffer is done: hand it back
          tc_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty(b));
        }
        // Fold this warp's 8 sub-blocks (digit sums d = 4T + w + j) of each
        // column into the exact integers Th = sum_{d<=4} S_d 2^(8(4-d)) and
        // Tl = sum_{d=5..8} S_d 2^(8(8-d)) before the exchange (|sub-block| <=
        // 2^26: |Th| < 2^62, |Tl| < 2^54, exact in int64; the by-product pairs
        // of digit sums 9 and 10 weigh < 2^-72 of the row x column scales and
        // are dropped -- a set closed under transposition, so S_d = S_d^T and
        // the symmetric-operand result stays bitwise symmetric).  The exchange
        // carries one (Th, Tl) pair per warp and element instead of 8 ints.
        // (each term is one 32 x 32 -> 64-bit multiply-add: the multiplier
        // 2^(8(4-d)) / 2^(8(8-d)) of a sub-block fits an int except 2^32 for
        // d = 0, which is a shift into the high word)
        int mh[2][4], ml[2][4];
#pragma unroll
        for (int T = 0; T < 2; ++T)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int d = 4 * T + w + j;  // (w is warp-uniform)
            mh[T][j] = (d >= 1 && d <= 4) ? 1 << (8 * (4 - d)) : 0;
            ml[T][j] = (d >= 5 && d <= 8) ? 1 << (8 * (8 - d)) : 0;
          }
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          long long ph = w == 0 ? (long long)V[0][0][c8] * 4294967296LL : 0LL, pl = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // T = 0: d = w + j in 0..6 (either part); T = 1: d = 4 + w + j in
            // 4..10 (Th only for d = 4)
            ph += (long long)V[0][j][c8] * (long long)mh[0][j];
            pl += (long long)V[0][j][c8] * (long long)ml[0][j];
            pl += (long long)V[1][j][c8] * (long long)ml[1][j];
          }
          ph += (long long)V[1][0][c8] * (long long)mh[1][0];  // (d = 4: w = 0, j = 0)
          xh[(w * 8 + c8) * 32 + r] = ph;
          xl[(w * 8 + c8) * 32 + r] = pl;
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        // this thread: row r, columns 2w, 2w+1 of the chunk
        double res[2];
        bool bad[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c8 = 2 * w + h;
          long long th = 0, tl = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            th += xh[(i * 8 + c8) * 32 + r];
            tl += xl[(i * 8 + c8) * 32 + r];
          }
          const double v = oz_round2(th, tl);  // 2^32 sum_d S_d 2^-8d, one rounding
          const int col = cc * 8 + c8;
          const int exc = ex_b[bj * Z_NB + col];
          bad[h] = row_bad || exc == OZ_EXP_BAD;
          const int k = er - 32 + (bad[h] ? 0 : oz_exp(exc));  // C = v 2^k
          res[h] = (k >= -1022 && k <= 1023)
                       ? __dmul_rn(v, __longlong_as_double((long long)(k + 1023) << 52))
                       : ldexp(v, k);
        }
        const int col0 = cc * 8 + 2 * w;
        double2* p = reinterpret_cast<double2*>(Cb + r * Z_NB + col0);
        if (bad[0] || bad[1]) {
          // non-finite operand entries: those elements are computed once, at
          // the segment's end, in FP64 in the reference's order (leaf_ozaki.cu)
          // (unrolled: a dynamically indexed res[] would live in local memory)
          double* rp = Cb + r * Z_NB + col0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double v = res[h];
            if (bad[h]) {
              if (!seg_end) continue;
              v = oz_exact_elem<Idx>(accumulate ? rp[h] : 0.0, Ad, Bd, a_idx, b_idx, seg[m],
                                     seg[m + 1], Z_NB, r, col0 + h);
            } else if (cont) {
              v = __dadd_rn(rp[h], v);
            }
            rp[h] = v;
            if (Cm) Cm[(col0 + h) * Z_NB + r] = v;
            res[h] = v;
          }
        } else {
          if (cont) {
            const double2 o = *p;
            res[0] = __dadd_rn(o.x, res[0]);
            res[1] = __dadd_rn(o.y, res[1]);
          }
          *p = make_double2(res[0], res[1]);
          if (Cm) {
            Cm[col0 * Z_NB + r] = res[0];
            Cm[(col0 + 1) * Z_NB + r] = res[1];
          }
        }
        if (want_ex) {
          const unsigned k0 = oz_ex_code(res[0]), k1 = oz_ex_code(res[1]);
          rcode = max(rcode, max(k0, k1));
          const unsigned wk = k0 | (k1 << 16);
          if (cc == 0) cc0 = wk;
          else if (cc == 1) cc1 = wk;
          else if (cc == 2) cc2 = wk;
          else cc3 = wk;
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
      }
      if (want_ex) {
        if (Cm) {  // lane = row: a column's max over the warp is the block's
          const unsigned cw[4] = {cc0, cc1, cc2, cc3};
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const unsigned mx = __reduce_max_sync(0xffffffffu, (cw[cc] >> (16 * h)) & 0xFFFFu);
              if (lane == 0 && mx) atomicMax(ex_out + bj * Z_NB + cc * 8 + 2 * w + h, oz_ex_decode(mx));
            }
        }
        if (rcode) atomicMax(ex_out + bi * Z_NB + r, oz_ex_decode(rcode));
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == 5)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase),
                 "r"(TCOLS)
                 : "memory");
}

}  // namespace

void oz32_operand_passes(const Mat& M, bool trans, int* ex, int8_t* out, cudaStream_t s,
                         bool exponents) {
  const int grid = grid_for((M.nblocks + 3) / 4, 1, (int64_t)multiprocessors() * 8);
  if (exponents) {
    launch_plain(k_oz32_exponents, grid, 256, 0, s, (const double*)M.data, (const int64_t*)M.keys,
                 M.nblocks, M.G, trans ? 1 : 0, ex);
    SPAMM_LAUNCH_CK();
  }
  if (exponents)
    launch_pdl(k_oz32_split, grid, 256, 0, s, (const double*)M.data, (const int64_t*)M.keys,
               M.nblocks, M.G, trans ? 1 : 0, (const int*)ex, out);
  else  // first launch after the caller's cross-stream wait: plain
    launch_plain(k_oz32_split, grid, 256, 0, s, (const double*)M.data, (const int64_t*)M.keys,
                 M.nblocks, M.G, trans ? 1 : 0, (const int*)ex, out);
  SPAMM_LAUNCH_CK();
}

void oz32_exponents(const Mat& M, bool by_col, int* ex, cudaStream_t s) {
  const int grid = grid_for((M.nblocks + 3) / 4, 1, (int64_t)multiprocessors() * 8);
  launch_plain(k_oz32_exponents, grid, 256, 0, s, (const double*)M.data, (const int64_t*)M.keys,
               M.nblocks, M.G, by_col ? 1 : 0, ex);
  SPAMM_LAUNCH_CK();
}

template <class Idx, int NBUF, int TPS, int STAGES>
void oz32_launch_cfg(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                     const int64_t* c_out, const int64_t* c_mirror, bool accumulate, const Mat& A,
                     const Mat& B, const OzakiOperands& op, double* C, cudaStream_t s,
                     const int32_t* order, int* counter, int* ex_out) {
  using Cfg = ZCfg<NBUF, TPS, STAGES>;
  auto kern = k_leaf_ozaki32<Idx, NBUF, TPS, STAGES>;
  static std::once_flag once;
  std::call_once(once, [&] {
    SPAMM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Cfg::SMEM));
    const char* v = getenv("SPAMM_K4Z_HINT");
    const int narrow = (v && (atoi(v) & 4)) ? 1 : 0;
    SPAMM_CK(cudaMemcpyToSymbol(c_z_narrow, &narrow, sizeof(int)));
  });
  int64_t grid = (int64_t)multiprocessors() * Cfg::CTAS;
  if (grid > n_seg) grid = n_seg;
  launch_plain(kern, (unsigned)grid, Z_THREADS, Cfg::SMEM, s, n_seg, seg, a_idx, b_idx,
               (const int32_t*)op.b_tr, (const int64_t*)A.keys, (const int64_t*)B.keys, op.G,
               (const int8_t*)op.as, (const int8_t*)op.bs, (const int*)op.ex_a,
               (const int*)op.ex_b, c_out, c_mirror, accumulate ? 1 : 0, C,
               order, counter, (const double*)A.data, (const double*)B.data, ex_out);
  SPAMM_LAUNCH_CK();
}

template <class Idx>
void oz32_launch(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                 const int64_t* c_out, const int64_t* c_mirror, bool accumulate, const Mat& A,
                 const Mat& B, const OzakiOperands& op, double* C, cudaStream_t s,
                 const int32_t* order, int* counter, int* ex_out) {
  // Two CTAs per SM (256 TMEM columns each): the kernel is latency-bound, and
  // a second CTA hides it better than double-buffered accumulators in one
  // (cfg3 K4z 8.0 vs 10.9 ms per solve; 1 task x 4 stages: 9.7 ms).  With the
  // 16-KB exchange buffer (int64 pairs) a CTA has room for 3 stages of 2
  // tasks -- the default (cfg3 solve 14.19 vs 14.71 ms with 2 stages; 2 stages
  // of 3 tasks: 14.21; 6 stages of 1 task: 16.2).  SPAMM_OZ32_SHAPE=2: 2
  // stages of 2 tasks; =1: one CTA per SM, double-buffered TMEM.
  static const int shape = [] {
    const char* v = getenv("SPAMM_OZ32_SHAPE");
    return v ? atoi(v) : 3;
  }();
  if (shape == 1)
    oz32_launch_cfg<Idx, 2, 4, 3>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B,
                                  op, C, s, order, counter, ex_out);
  else if (shape == 3)  // two CTAs per SM, 3 stages of 2 tasks (the 16-KB exchange buffer)
    oz32_launch_cfg<Idx, 1, 2, 3>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B,
                                  op, C, s, order, counter, ex_out);
  else if (shape == 4)  // two CTAs per SM, 2 stages of 3 tasks
    oz32_launch_cfg<Idx, 1, 3, 2>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B,
                                  op, C, s, order, counter, ex_out);
  else if (shape == 5)  // two CTAs per SM, 6 stages of 1 task
    oz32_launch_cfg<Idx, 1, 1, 6>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B,
                                  op, C, s, order, counter, ex_out);
  else
    oz32_launch_cfg<Idx, 1, 2, 2>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B,
                                  op, C, s, order, counter, ex_out);
}

template void oz32_launch<int32_t>(int64_t, const int64_t*, const int32_t*, const int32_t*,
                                   const int64_t*, const int64_t*, bool, const Mat&, const Mat&,
                                   const OzakiOperands&, double*, cudaStream_t, const int32_t*,
                                   int*, int*);
template void oz32_launch<int64_t>(int64_t, const int64_t*, const int64_t*, const int64_t*,
                                   const int64_t*, const int64_t*, bool, const Mat&, const Mat&,
                                   const OzakiOperands&, double*, cudaStream_t, const int32_t*,
                                   int*, int*);

}  // namespace spamm
