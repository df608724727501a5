// K4z (Nb = 64): the leaf products on the INT8 tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM) by exact digit slicing -- Ozaki scheme I.
//
// Reference: _gemm_acc / _gemm_batch (kernel.py:64-77); same contract as the
// DMMA kernel K4 (leaf_tma.cu): the tasks of one C block (k ascending) are
// reduced by one CTA, deterministically, no atomics.  The arithmetic differs:
//
//  * every operand row r (A) / column c (B) gets one power-of-two scale 2^E
//    (E: frexp exponent of the largest |x| in that global row / column over
//    all stored blocks, k_oz_exponents), and x 2^-E is written with 8 signed
//    int8 digits x = 2^E (s_0 2^-7 + sum_{p=1..7} s_p 2^-(7+8p)), s_p in
//    [-128, 127] (k_oz_split: floor digits of |x|, a carry pass from the
//    bottom, the sign applied last -- every step exact; 63 bits, the remainder
//    is < 2^(E-63));
//  * a digit product sum_k dA_p[r][k] dB_q[k][c] is computed EXACTLY in int32
//    on the tensor cores and summed exactly over the tasks of the C block
//    (|.| <= 64 x 2^14 = 2^20 per task and digit pair; a quadrant of tile t
//    accumulates the t + 1 <= 4 anchors of digit sum 2t and the epilogue adds
//    <= 2 quadrants per digit sum, so <= 8 pairs x OZ_CHUNK = 128 tasks x
//    2^20 = 2^30 -- int32 exact; longer segments flush per chunk to FP64, in
//    order);
//  * all digit pairs p + q <= 7 (and four of p + q = 8) are formed: A slices
//    stacked two per MMA along M (rows 0-63 = s_p, 64-127 = s_p+1), B slices
//    two per 128 columns along N: 10 slice-pair blocks per k-step into 4 TMEM
//    tiles of 128 columns (tile t holds the pairs of digit sums 2t, 2t+1,
//    2t+1, 2t+2 in its four quadrants) -- all 512 TMEM columns.  The blocks
//    sharing an A pair and two consecutive B pairs are one MMA of N = 256 over
//    two adjacent tiles: per k-step 4 MMAs of 128x256x32 + 2 of 128x128x32
//    (12 per task, 20 % less shared-memory operand traffic than 20 of N = 128);
//  * the epilogue adds the quadrants of equal digit sum d in int32 (exact),
//    so S_d[r][c] = S_d[c][r] bitwise for a symmetric operand, folds them
//    into two exact int64 (Th = sum_{d<=4} S_d 2^(8(4-d)), Tl = the rest)
//    while TMEM is held, hands TMEM back, and only then rounds Th + Tl 2^-32
//    (oz_round2) and scales: C = 2^(Er+Ec-46) (Th + Tl 2^-32) -- the FP64
//    work and the stores overlap the next C block's MMAs.
//
// Error: the dropped pairs (p + q >= 8) weigh <= 2^-64 K max|A_r| max|B_c|
// per element, below the FP64 rounding of the sum: measured 5-6e-17 relative
// Frobenius error against an extended-precision product, vs 4-6e-16 for a
// plain FP64 product (7-bit balanced digits, 4 tiles: 1e-14 -- the dropped
// pairs there weigh 2^-56 and add up systematically on the diagonal of X*X).
// Results are deterministic and exactly symmetric (diagonal blocks of X*X
// bitwise symmetric), not bitwise the DMMA kernel's.
//
// Operand traffic per task is the FP64 kernel's (8 slices x 4 KB = 32 KB per
// block), compute per task is the work of 20 tcgen05 MMAs of 128x128x32 =
// 1,333 tensor cycles versus ~4,100 cycles of DMMA at 64x64x64.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <cstdio>

#include "internal.h"
#include "ozaki_common.cuh"

namespace spamm {

namespace {

using namespace ozk;

constexpr int OZ_NB = 64;
constexpr int OZ_SLICES = 8;
constexpr int OZ_SLICE_BYTES = OZ_NB * OZ_NB;                  // 4 KB (int8)
constexpr int OZ_BLOCK_BYTES = OZ_SLICES * OZ_SLICE_BYTES;     // 32 KB
constexpr int OZ_STAGES = 3;
constexpr int OZ_STAGE = 2 * OZ_BLOCK_BYTES;                   // A + B slices of one task
constexpr int OZ_CHUNK = 128;       // tasks per TMEM accumulation (quadrant sums stay < 2^30)
// int32 bound: S_d adds <= 2 quadrants of <= 4 digit pairs each (tile 3 has
// anchors (0,6), (2,4), (4,2), (6,0)), each pair <= 64 products of |digit|^2
// <= 2^14 per task.
static_assert(8LL * OZ_NB * (1LL << 14) * OZ_CHUNK < (1LL << 31),
              "OZ_CHUNK too large for exact int32 digit sums");
// Epilogue: 8 warps in two groups of 4 (warp w reads TMEM lane quarter w % 4);
// group g converts the columns 32g..32g+31 of the C block.
constexpr int OZ_EPI = 256;
constexpr int OZ_GROUP = 128;
constexpr int OZ_PRODUCER = OZ_EPI / 32, OZ_MMA = OZ_PRODUCER + 1;  // warps 8, 9
constexpr int OZ_THREADS = OZ_EPI + 64;
constexpr int OZ_XBUF = 32 * OZ_EPI * 4;  // epilogue exchange: 32 ints per thread (32 KB)
constexpr size_t OZ_SMEM = 1024 + (size_t)OZ_STAGES * OZ_STAGE + OZ_XBUF + 256;

// Byte offset of element (n, k) of a 64x64 int8 slice in the UMMA K-major
// no-swizzle canonical layout: 8-row x 16-byte core matrices (128 B), the
// four k-chunks of an 8-row group adjacent (LBO = 128 B), row groups 512 B
// apart (SBO) -- so two consecutive slices form one 128-row operand.
__host__ __device__ constexpr int oz_off(int n, int k) {
  return (n >> 3) * 512 + (k >> 4) * 128 + (n & 7) * 16 + (k & 15);
}

// ex[g] = max frexp exponent of |x| over global row g (by_col = 0) or global
// column g (by_col = 1) of the stored blocks.
__global__ void __launch_bounds__(256) k_oz_exponents(const double* __restrict__ data,
                                                      const int64_t* __restrict__ keys,
                                                      int64_t nblocks, int64_t G, int by_col,
                                                      int* __restrict__ ex) {
  pdl_wait();
  __shared__ double red[4][OZ_NB];
  const int t = threadIdx.x;
  for (int64_t s = blockIdx.x; s < nblocks; s += gridDim.x) {
    const double* b = data + s * (OZ_NB * OZ_NB);
    const int64_t key = keys[s];
    if (by_col) {
      double mx = 0.0;
#pragma unroll 4
      for (int i = 0; i < 16; ++i) mx = fmax(mx, oz_absf(b[((t >> 6) + 4 * i) * OZ_NB + (t & 63)]));
      red[t >> 6][t & 63] = mx;
      __syncthreads();
      if (t < OZ_NB) {
        mx = fmax(fmax(red[0][t], red[1][t]), fmax(red[2][t], red[3][t]));
        if (mx > 0.0) atomicMax(ex + (key % G) * OZ_NB + t, oz_exp_of(mx));
      }
      __syncthreads();
    } else {
      // thread t: 16 elements of row t / 4, pairs t % 4, t % 4 + 4, ... (8
      // independent 16-byte loads; a quad reads 64 contiguous bytes per load,
      // so every sector a warp fetches is used whole)
      const double2* q = reinterpret_cast<const double2*>(b + (t >> 2) * OZ_NB) + (t & 3);
      double2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = q[4 * i];
      double mx = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) mx = fmax(mx, fmax(oz_absf(v[i].x), oz_absf(v[i].y)));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      if ((t & 3) == 0 && mx > 0.0) atomicMax(ex + (key / G) * OZ_NB + (t >> 2), oz_exp_of(mx));
    }
  }
}

// out + s * 32 KB: the 8 digit slices of block s.  trans = 0 (A role): slice
// row n = block row n, exponent of global row bi*64+n; trans = 1 (B role,
// K-major B^T): slice row n = block column n, exponent of global column bj*64+n.
// Thread t: slice row n = t / 4, k = 16 (t % 4) .. +15 (one 16-byte store per slice).
__global__ void __launch_bounds__(256) k_oz_split(const double* __restrict__ data,
                                                  const int64_t* __restrict__ keys,
                                                  int64_t nblocks, int64_t G, int trans,
                                                  const int* __restrict__ ex,
                                                  int8_t* __restrict__ out,
                                                  const int32_t* __restrict__ slot,
                                                  int32_t* __restrict__ tr) {
  pdl_wait();
  // Staged through shared memory in both roles (coalesced global loads):
  // trans: element (r, c) at r * 65 + c, read down column n;  !trans: at
  // r * 68 + c + c / 16, so a half-warp's reads (4 rows x 4 column groups)
  // fall in 16 distinct 8-byte banks.
  __shared__ double tile[OZ_NB * 68];
  const int t = threadIdx.x, n = t >> 2, kc = t & 3;
  for (int64_t s = blockIdx.x; s < nblocks; s += gridDim.x) {
    const double* b = data + s * (OZ_NB * OZ_NB);
    double y[16];
    if (trans) {
      for (int i = t; i < OZ_NB * OZ_NB; i += 256) tile[(i >> 6) * (OZ_NB + 1) + (i & 63)] = b[i];
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = tile[(kc * 16 + i) * (OZ_NB + 1) + n];
    } else {
      const double2* q = reinterpret_cast<const double2*>(b);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = t + 256 * j, c = (2 * i) & 63;
        const double2 v = q[i];
        double* d = tile + (i >> 5) * 68 + c + (c >> 4);
        d[0] = v.x;
        d[1] = v.y;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = tile[n * 68 + kc * 17 + i];
    }
    __syncthreads();
    const int64_t key = keys[s];
    // (symmetric operands) storage slot of the transposed block
    if (tr && t == 0) tr[s] = slot[(key % G) * G + key / G];
    const int e = oz_exp(ex[(trans ? key % G : key / G) * OZ_NB + n]);
    uint32_t hi[16], lo[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint64_t d = oz_digits(y[i], e);
      hi[i] = (uint32_t)(d >> 32);  // slices 0..3 = bytes 3..0
      lo[i] = (uint32_t)d;          // slices 4..7 = bytes 3..0
    }
    int8_t* o = out + s * OZ_BLOCK_BYTES + oz_off(n, kc * 16);
#pragma unroll
    for (int p = 0; p < OZ_SLICES; ++p) {
      const uint32_t* h = p < 4 ? hi : lo;
      const int byte = 3 - (p & 3);
      *reinterpret_cast<uint4*>(o + p * OZ_SLICE_BYTES) =
          make_uint4(oz_gather4(h[0], h[1], h[2], h[3], byte),
                     oz_gather4(h[4], h[5], h[6], h[7], byte),
                     oz_gather4(h[8], h[9], h[10], h[11], byte),
                     oz_gather4(h[12], h[13], h[14], h[15], byte));
    }
  }
}

// One full wave of `fn` (resident CTAs per SM x SMs): grids of the streaming
// pre-passes, which loop over the blocks, never leave a partial second wave.
template <typename F>
int resident_wave(F* fn, int threads) {
  int per_sm = 0;
  SPAMM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0));
  return (per_sm > 0 ? per_sm : 1) * multiprocessors();
}

// tr[s] = storage slot of the transposed block of s (symmetric operands).
__global__ void k_oz_trslot(const int64_t* __restrict__ keys, int64_t nblocks, int64_t G,
                            const int32_t* __restrict__ slot, int32_t* __restrict__ tr) {
  pdl_wait();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nblocks;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = keys[s];
    tr[s] = slot[(key % G) * G + key / G];
  }
}

// The 10 slice-pair MMAs of one task: A pair start p, B pair start q (tile (p + q) / 2).
__host__ __device__ constexpr int oz_p(int ci) {
  return ci == 0 ? 0 : ci == 1 ? 0 : ci == 2 ? 2 : ci == 3 ? 0 : ci == 4 ? 2 : ci == 5 ? 4
       : ci == 6 ? 0 : ci == 7 ? 2 : ci == 8 ? 4 : 6;
}
__host__ __device__ constexpr int oz_q(int ci) {
  return ci == 0 ? 0 : ci == 1 ? 2 : ci == 2 ? 0 : ci == 3 ? 4 : ci == 4 ? 2 : ci == 5 ? 0
       : ci == 6 ? 6 : ci == 7 ? 4 : ci == 8 ? 2 : 0;
}

// PROF (SPAMM_K4Z_PROF): per-CTA cycle counters; a separate instantiation so
// the counters cost the product kernel no registers.
template <class Idx, bool PROF>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_leaf_ozaki(int64_t n_seg, const int64_t* __restrict__ seg, const Idx* __restrict__ a_idx,
                 const Idx* __restrict__ b_idx, const int32_t* __restrict__ b_tr,
                 const int64_t* __restrict__ a_keys, const int64_t* __restrict__ b_keys, int64_t G,
                 const int8_t* __restrict__ As, const int8_t* __restrict__ Bs,
                 const int* __restrict__ ex_a, const int* __restrict__ ex_b,
                 const int64_t* __restrict__ c_out, const int64_t* __restrict__ c_mirror,
                 int accumulate, double* __restrict__ C, const int32_t* __restrict__ order,
                 int* __restrict__ next_block, int hint, long long* __restrict__ prof,
                 const double* __restrict__ Ad, const double* __restrict__ Bd,
                 int* __restrict__ ex_out) {
  auto gtime = []() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (long long)t;
  };
  if (PROF && threadIdx.x == 0) prof[blockIdx.x * 16 + 12] = gtime();
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  int* xb = reinterpret_cast<int*>(gbase + OZ_STAGES * OZ_STAGE);
  const uint32_t bars = base + OZ_STAGES * OZ_STAGE + OZ_XBUF;
  auto full = [&](int s) { return bars + 8u * s; };
  auto empty = [&](int s) { return bars + 8u * (OZ_STAGES + s); };
  const uint32_t tfull = bars + 8u * (2 * OZ_STAGES), tempty = tfull + 8u;
  int64_t* meta = reinterpret_cast<int64_t*>(gbase + OZ_STAGES * OZ_STAGE + OZ_XBUF +
                                             8 * (2 * OZ_STAGES + 2));
  int64_t* meta2 = meta + OZ_STAGES;  // (bi << 32) | bj of the chunk starting in this stage
  int64_t* ring = meta2 + OZ_STAGES;  // the chunk in TMEM: meta, meta2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    mbar_init(tfull, 2);   // MMA completion (commit) + the ring entry (MMA thread)
    mbar_init(tempty, OZ_EPI / 32);  // one arrive per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == OZ_MMA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == OZ_PRODUCER) {
    // ---------------- producer: two 32-KB bulk copies per task ----------------
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
    // Batches of 32 tasks (one index per lane).  The next batch's indices are
    // loaded while the current batch's copies are issued (its dependent
    // lookups -- transposed slot, the (i, j) of a chunk start -- one task
    // later), and the block after the current one is claimed during its
    // first batch: no chain of L2 round trips between two batches' copies.
    auto first_lookups = [&](int64_t c0_, int64_t t0_, int64_t t1_, int64_t& ra_, int64_t& rb_,
                             int64_t& kab_) {
      const int64_t t = c0_ + lane;
      kab_ = 0;
      if (t < t1_) {
        const int64_t rbo = rb_;
        if ((t - t0_) % OZ_CHUNK == 0)
          kab_ = ((a_keys[ra_] / G) << 32) | (b_keys[rbo] % G);
        if (b_tr) rb_ = b_tr[rbo];
      }
    };
    int64_t m = 0, t0 = 0, t1 = 0;
    bool have = claim(m, t0, t1);
    int64_t c0 = t0, ra_l = 0, rb_l = 0, kab_l = 0;
    if (have) {
      if (c0 + lane < t1) {
        ra_l = (int64_t)a_idx[c0 + lane];
        rb_l = (int64_t)b_idx[c0 + lane];
      }
      first_lookups(c0, t0, t1, ra_l, rb_l, kab_l);
    }
    int64_t mn = 0, t0n = 0, t1n = 0;  // the block claimed ahead
    bool hn = false, claimed = false;
    while (have) {
      const int cnt = t1 - c0 < 32 ? (int)(t1 - c0) : 32;
      int64_t nm = 0, nt0 = 0, nt1 = 0, nc0 = 0, nra = 0, nrb = 0, nkab = 0;
      bool hnext = false;
      for (int q = 0; q < cnt; ++q) {
        const int64_t ra = __shfl_sync(0xffffffffu, ra_l, q);
        const int64_t rb = __shfl_sync(0xffffffffu, rb_l, q);
        const int64_t kab = __shfl_sync(0xffffffffu, kab_l, q);
        mbar_wait(empty(stage), phase ^ 1u);
        if (lane == 0) {
          const int64_t tq = c0 + q, r = tq - t0;
          const bool first = r % OZ_CHUNK == 0;
          const bool last = tq + 1 == t1 || (r + 1) % OZ_CHUNK == 0;
          const bool cont = r >= OZ_CHUNK || accumulate;
          // bit 3: the chunk ends the C block's segment
          meta[stage] = (m << 4) | (first ? 1 : 0) | (last ? 2 : 0) | (cont ? 4 : 0) |
                        (tq + 1 == t1 ? 8 : 0);
          if (first) meta2[stage] = kab;
          mbar_expect_tx(full(stage), OZ_STAGE);
          const uint32_t sa = base + stage * OZ_STAGE;
          if (hint & 1) {  // operand slices evict_last (re-read by many C blocks)
            const uint64_t pol = pol_evict_last();
            bulk_g2s_pol(sa, As + ra * OZ_BLOCK_BYTES, OZ_BLOCK_BYTES, full(stage), pol);
            bulk_g2s_pol(sa + OZ_BLOCK_BYTES, Bs + rb * OZ_BLOCK_BYTES, OZ_BLOCK_BYTES,
                         full(stage), pol);
          } else {
            bulk_g2s(sa, As + ra * OZ_BLOCK_BYTES, OZ_BLOCK_BYTES, full(stage));
            bulk_g2s(sa + OZ_BLOCK_BYTES, Bs + rb * OZ_BLOCK_BYTES, OZ_BLOCK_BYTES,
                     full(stage));
          }
        }
        __syncwarp();
        if (++stage == OZ_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
        if (q == 0) {  // after this batch's first copy: claim ahead, load the next batch
          if (!claimed) {
            hn = claim(mn, t0n, t1n);
            claimed = true;
          }
          if (c0 + 32 < t1) {
            nm = m, nt0 = t0, nt1 = t1, nc0 = c0 + 32;
            hnext = true;
          } else {
            nm = mn, nt0 = t0n, nt1 = t1n, nc0 = t0n;
            hnext = hn;
          }
          if (hnext && nc0 + lane < nt1) {
            nra = (int64_t)a_idx[nc0 + lane];
            nrb = (int64_t)b_idx[nc0 + lane];
          }
        }
        if (hnext && (q == 1 || cnt == 1)) first_lookups(nc0, nt0, nt1, nra, nrb, nkab);
      }
      if (!hnext) break;
      if (nc0 == nt0) claimed = false;  // a new block: claim the one after it
      m = nm, t0 = nt0, t1 = nt1, c0 = nc0;
      ra_l = nra, rb_l = nrb, kab_l = nkab;
    }
    mbar_wait(empty(stage), phase ^ 1u);
    if (lane == 0) {
      meta[stage] = -1;
      mbar_arrive(full(stage));
    }
  } else if (warp == OZ_MMA) {
    // ---------------- MMA issuer: one thread ----------------
    if (lane == 0) {
      const bool wide = !(hint & 4);  // SPAMM_K4Z_HINT bit 2: the 10 x N = 128 MMA form
      int stage = 0;
      uint32_t phase = 0, tphase = 0;
      int64_t cur2 = 0;
      long long w_full = 0, w_tempty = 0, n_tasks = 0;
      const long long t_start = PROF ? clock64() : 0;
      for (;;) {
        long long t0 = PROF ? clock64() : 0;
        mbar_wait(full(stage), phase);
        if (PROF) w_full += clock64() - t0;
        tc_after();
        const int64_t md = meta[stage];
        if (md < 0) {
          mbar_wait(tempty, tphase ^ 1u);  // the epilogue is done with the last chunk
          ring[0] = -1;
          mbar_arrive(tfull);
          oz_commit(tfull);
          if (PROF) {
            long long* o = prof + blockIdx.x * 16;
            o[0] = clock64() - t_start;
            o[1] = w_full;
            o[2] = w_tempty;
            o[3] = n_tasks;
            o[13] = gtime();
          }
          break;
        }
        const bool first = md & 1;
        if (first) {
          cur2 = meta2[stage];
          t0 = PROF ? clock64() : 0;
          mbar_wait(tempty, tphase ^ 1u);  // TMEM drained by the epilogue
          if (PROF) w_tempty += clock64() - t0;
          tphase ^= 1u;
          tc_after();
        }
        const uint32_t sa = base + stage * OZ_STAGE, sb = sa + OZ_BLOCK_BYTES;
        if (wide) {
          // the same 10 slice-pair blocks as 4 MMAs of N = 256 (four B slices:
          // two adjacent tiles) + 2 of N = 128 per k-step: 20 % less shared-
          // memory operand traffic (the A pair is read once for two B pairs).
          // The first two open tiles 0-1 and 2-3; the rest accumulate.
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
            for (int mi = 0; mi < 6; ++mi) {
              const int p = mi == 0 ? 0 : mi == 1 ? 0 : mi == 2 ? 2 : mi == 3 ? 4 : mi == 4 ? 2 : 6;
              const int q = mi == 1 ? 4 : mi == 4 ? 4 : 0;
              const bool n256 = mi < 4;
              const bool opens = mi < 2;
              oz_mma(tbase + 128u * ((p + q) / 2), oz_desc(sa + p * OZ_SLICE_BYTES + ks * 256),
                     oz_desc(sb + q * OZ_SLICE_BYTES + ks * 256),
                     (first && opens && ks == 0) ? 0u : 1u, n256 ? OZ_IDESC_N256 : OZ_IDESC);
            }
          }
        } else {
#pragma unroll
        for (int ci = 0; ci < 10; ++ci) {
          const int p = oz_p(ci), q = oz_q(ci), t = (p + q) / 2;
          const bool opens = ci == 0 || ci == 1 || ci == 3 || ci == 6;  // first pair of tile t
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            oz_mma(tbase + 128u * t, oz_desc(sa + p * OZ_SLICE_BYTES + ks * 256),
                   oz_desc(sb + q * OZ_SLICE_BYTES + ks * 256),
                   (first && opens && ks == 0) ? 0u : 1u);
        }
        }
        oz_commit(empty(stage));  // stage free once these MMAs have read it
        ++n_tasks;
        if (md & 2) {
          ring[0] = md;
          ring[1] = cur2;
          mbar_arrive(tfull);
          oz_commit(tfull);  // accumulators complete
        }
        if (++stage == OZ_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warps 0-7, TMEM lane (warp % 4) * 32 + lane ----------------
    const int grp = warp >> 2;
    const int e = (warp & 3) * 32 + lane, r = e & 63, partner = e ^ 64;
    const bool top = e < 64;
    const int own0 = top ? 0 : 4;  // the 4 columns of each 8-column chunk this thread writes
    int* xg = xb + grp * (32 * OZ_GROUP);
    const uint32_t lane_base = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t ephase = 0;
    long long e_wait = 0, e_hold = 0, e_all = 0, n_blk = 0;
    long long e_ph[4] = {0, 0, 0, 0};  // chunk phases: TMEM read, exchange, convert+store, barrier
    for (;;) {
      long long te0 = PROF ? clock64() : 0;
      mbar_wait(tfull, ephase);
      if (PROF && threadIdx.x == 0) e_wait += clock64() - te0;
      te0 = PROF ? clock64() : 0;
      ephase ^= 1u;
      tc_after();
      const int64_t md = ring[0];
      if (md < 0) {
        if (PROF && threadIdx.x == 0) {
          prof[blockIdx.x * 16 + 4] = e_wait;
          prof[blockIdx.x * 16 + 5] = e_hold;
          prof[blockIdx.x * 16 + 6] = e_all;
          prof[blockIdx.x * 16 + 7] = n_blk;
          for (int i = 0; i < 4; ++i) prof[blockIdx.x * 16 + 8 + i] = e_ph[i];
          prof[blockIdx.x * 16 + 14] = gtime();
        }
        break;
      }
      const int64_t bij = ring[1];
      const int64_t m = md >> 4;
      const bool cont = md & 4, seg_end = md & 8;
      const int64_t bi = bij >> 32, bj = bij & 0xffffffffLL;
      const int exr = ex_a[bi * OZ_NB + r];
      const bool row_bad = exr == OZ_EXP_BAD;
      const int er = (row_bad ? 0 : oz_exp(exr)) - 14;
      double* Cb = C + (c_out ? c_out[m] : m) * (int64_t)(OZ_NB * OZ_NB);
      const int64_t mi = c_mirror ? c_mirror[m] : -1;
      double* Cm = mi >= 0 ? C + mi * (int64_t)(OZ_NB * OZ_NB) : nullptr;
      // ex_out (symmetric X^2): the K4z row exponents of the product itself,
      // so the next multiply skips its exponent pass -- this thread's row max
      // over its columns, and per column the max over the warp's 32 rows
      // (the rows of the mirror block)
      const bool want_ex = ex_out != nullptr && seg_end;
      unsigned rcode = 0u;  // row max (code, oz_ex_code)
      // Phase 1 (TMEM held): per 8-column chunk cl, read the four tiles, hand
      // the partner lane its 4 columns, and fold this thread's 4 columns into
      // the exact integers Th = sum_{d<=4} S_d 2^(8(4-d)) and
      // Tl = sum_{d=5..8} S_d 2^(8(8-d)) (|S_d| < 2^30: |Th| < 2^62.1, both
      // exact in int64; S_d = S_d^T for a symmetric operand, so Th / Tl are
      // too).  TMEM is handed back as soon as the last chunk's loads land.
      // Phase 2 (TMEM released, beside the next C block's MMAs): round
      // Th + Tl 2^-32 once, scale by 2^(Er + Ec - 46), accumulate, store.
      long long Th[4][4], Tl[4][4];
      int4* xg4 = reinterpret_cast<int4*>(xg);
      long long tp = (PROF && threadIdx.x == 0) ? clock64() : 0;
#pragma unroll
      for (int cl = 0; cl < 4; ++cl) {
        const int cc = grp * 4 + cl;
        int L[4][8], R[4][8];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          tmem_ld8(lane_base + 128u * t + cc * 8, L[t]);
          tmem_ld8(lane_base + 128u * t + 64 + cc * 8, R[t]);
        }
        tmem_wait8(L[0]);
        tmem_keep8(R[0]);
#pragma unroll
        for (int t = 1; t < 4; ++t) {
          tmem_keep8(L[t]);
          tmem_keep8(R[t]);
        }
        if (PROF && threadIdx.x == 0) {
          const long long t1 = clock64();
          e_ph[0] += t1 - tp;
          tp = t1;
        }
        if (cl == 3) {  // this warp's TMEM reads are complete: hand TMEM back
          tc_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty);
          if (PROF && threadIdx.x == 0) e_hold += clock64() - te0;
        }
        // hand the partner the 4 columns it owns: one 16-byte store per (tile, half)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          xg4[(t * 2) * OZ_GROUP + e] = top ? make_int4(L[t][4], L[t][5], L[t][6], L[t][7])
                                            : make_int4(L[t][0], L[t][1], L[t][2], L[t][3]);
          xg4[(t * 2 + 1) * OZ_GROUP + e] = top ? make_int4(R[t][4], R[t][5], R[t][6], R[t][7])
                                                : make_int4(R[t][0], R[t][1], R[t][2], R[t][3]);
        }
        asm volatile("bar.sync %0, 128;\n" ::"r"(1 + grp) : "memory");
        if (PROF && threadIdx.x == 0) {
          const long long t1 = clock64();
          e_ph[1] += t1 - tp;
          tp = t1;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int4 a = xg4[(t * 2) * OZ_GROUP + partner];
          const int4 b = xg4[(t * 2 + 1) * OZ_GROUP + partner];
          const int oa[4] = {a.x, a.y, a.z, a.w};
          const int ob[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            // quadrants (top / bottom A slice x left / right B slice) of tile t
            const int ml = top ? L[t][c] : L[t][4 + c];  // static register indices
            const int mr = top ? R[t][c] : R[t][4 + c];
            const int tl = top ? ml : oa[c], tr = top ? mr : ob[c];
            const int bl = top ? oa[c] : ml, br = top ? ob[c] : mr;
            // S_{2t} += tl, S_{2t+1} += tr + bl, S_{2t+2} += br
            if (t == 0) {
              Th[cl][c] = (long long)tl * 4294967296LL + (long long)(tr + bl) * 16777216LL;
              Tl[cl][c] = (long long)br * 65536LL;  // S_2 (Th), placed below
            } else if (t == 1) {
              Th[cl][c] += ((long long)Tl[cl][c] + (long long)tl * 65536LL) +
                           (long long)(tr + bl) * 256LL;
              Tl[cl][c] = br;  // S_4 part (Th)
            } else if (t == 2) {
              Th[cl][c] += (long long)Tl[cl][c] + (long long)tl;
              Tl[cl][c] = (long long)(tr + bl) * 16777216LL + (long long)br * 65536LL;
            } else {
              Tl[cl][c] += (long long)tl * 65536LL + (long long)(tr + bl) * 256LL + (long long)br;
            }
          }
        }
        if (PROF && threadIdx.x == 0) {
          const long long t1 = clock64();
          e_ph[2] += t1 - tp;
          tp = t1;
        }
        asm volatile("bar.sync %0, 128;\n" ::"r"(1 + grp) : "memory");
      }
      // ---- phase 2: TMEM is free; round, scale, accumulate, store ----
#pragma unroll
      for (int cl = 0; cl < 4; ++cl) {
        const int col0 = (grp * 4 + cl) * 8 + own0;
        const int4 ec4 = *reinterpret_cast<const int4*>(ex_b + bj * OZ_NB + col0);
        const int ecs[4] = {ec4.x, ec4.y, ec4.z, ec4.w};
        bool bad[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) bad[c] = row_bad || ecs[c] == OZ_EXP_BAD;
        double res[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double v = oz_round2(Th[cl][c], Tl[cl][c]);
          const int k = er - 32 + (bad[c] ? 0 : oz_exp(ecs[c]));  // C = v 2^k
          res[c] = (k >= -1022 && k <= 1023)
                       ? __dmul_rn(v, __longlong_as_double((long long)(k + 1023) << 52))
                       : ldexp(v, k);
        }
        double2* row = reinterpret_cast<double2*>(Cb + r * OZ_NB + col0);
        if (bad[0] || bad[1] || bad[2] || bad[3]) {
          // a non-finite operand entry in this row or one of these columns:
          // those elements are computed once, at the segment's end, in FP64
          // in the reference's order (earlier chunks leave them untouched)
          double* rp = Cb + r * OZ_NB + col0;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double v = res[c];
            if (bad[c]) {
              if (!seg_end) continue;
              v = oz_exact_elem<Idx>(accumulate ? rp[c] : 0.0, Ad, Bd, a_idx, b_idx, seg[m],
                                     seg[m + 1], OZ_NB, r, col0 + c);
            } else if (cont) {
              v = __dadd_rn(rp[c], v);
            }
            rp[c] = v;
            if (Cm) Cm[(col0 + c) * OZ_NB + r] = v;
            res[c] = v;
          }
        } else {
          double* rp = reinterpret_cast<double*>(row);
          if (cont) {
            double p0, p1, p2, p3;
            oz_ld4(rp, p0, p1, p2, p3);
            res[0] = __dadd_rn(p0, res[0]);
            res[1] = __dadd_rn(p1, res[1]);
            res[2] = __dadd_rn(p2, res[2]);
            res[3] = __dadd_rn(p3, res[3]);
          }
          if (hint & 2) {  // products streamed past L2 (evict_first)
            oz_st4_cs(rp, res[0], res[1], res[2], res[3]);
            if (Cm)
#pragma unroll
              for (int c = 0; c < 4; ++c) __stcs(Cm + (col0 + c) * OZ_NB + r, res[c]);
          } else if (hint & 8) {  // products kept in L2 for the norm pass that follows
            const unsigned long long pol = oz_policy_evict_last();
            oz_st4_hint(rp, res[0], res[1], res[2], res[3], pol);
            if (Cm)
#pragma unroll
              for (int c = 0; c < 4; ++c) oz_st1_hint(Cm + (col0 + c) * OZ_NB + r, res[c], pol);
          } else {
            oz_st4(rp, res[0], res[1], res[2], res[3]);
            if (Cm)
#pragma unroll
              for (int c = 0; c < 4; ++c) Cm[(col0 + c) * OZ_NB + r] = res[c];
          }
        }
        if (want_ex) {
          unsigned k4[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            k4[c] = oz_ex_code(res[c]);
            rcode = max(rcode, k4[c]);
          }
          if (Cm) {  // mirror rows: a column's max over this warp's 32 rows
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const unsigned mx = __reduce_max_sync(0xffffffffu, k4[c]);
              if (lane == 0 && mx)
                atomicMax(ex_out + bj * OZ_NB + col0 + c, oz_ex_decode(mx));
            }
          }
        }
      }
      if (want_ex && rcode) atomicMax(ex_out + bi * OZ_NB + r, oz_ex_decode(rcode));
      if (PROF && threadIdx.x == 0) e_ph[3] += clock64() - tp;
      if (PROF && threadIdx.x == 0) {
        e_all += clock64() - te0;
        ++n_blk;
      }
    }
  }
  tc_before();
  __syncthreads();
  tc_after();
  if (warp == OZ_MMA)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase)
                 : "memory");
}

}  // namespace

bool ozaki_supported(int nb) { return nb == OZ_NB || nb == 32; }

// The A slices of the SP2 loop's X*X (one size, every iteration): a buffer
// kept across multiplies per (host thread, device) instead of a pool round
// trip per product.  Reuse is ordered on the device: release records `done`
// on the stream that ran K4z, and the next prepare's stream waits on it (the
// caller may pass a different stream per multiply).
struct SliceCache {
  int8_t* p = nullptr;
  size_t bytes = 0;
  bool busy = false;           // handed out (host side: one multiply at a time)
  cudaEvent_t done = nullptr;  // recorded after the last K4z that read it
  bool pending = false;
};
static SliceCache& slice_cache() {
  thread_local SliceCache caches[64];
  int dev = 0;
  SPAMM_CK(cudaGetDevice(&dev));
  return caches[dev & 63];
}
static void slice_cache_release(cudaStream_t s) {
  SliceCache& c = slice_cache();
  if (!c.done) SPAMM_CK(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
  SPAMM_CK(cudaEventRecord(c.done, s));
  c.pending = true;
  c.busy = false;
}
void ozaki_cache_trim() {
  SliceCache& c = slice_cache();
  if (c.busy || !c.p) return;
  if (c.pending) SPAMM_CK(cudaEventSynchronize(c.done));
  SPAMM_CK(cudaFree(c.p));
  c.p = nullptr;
  c.bytes = 0;
  c.pending = false;
}

static void oz_dbg(const char* what, cudaStream_t s) {
  static const bool on = getenv("SPAMM_OZ_DEBUG") != nullptr;
  if (!on) return;
  const cudaError_t e = cudaStreamSynchronize(s);
  fprintf(stderr, "[oz] %s: %s\n", what, cudaGetErrorString(e));
}

bool ozaki_prepare(const Mat& A, const Mat& B, bool sym_b, cudaStream_t s, OzakiOperands& op,
                   bool try_only, bool defer_tr) {
  op = OzakiOperands();
  oz_dbg("enter", s);
  if (!ozaki_supported(A.nb) || B.nb != A.nb)
    throw CudaError("INT8-sliced leaf kernel needs block size 32 or 64");
  const int nb = A.nb;
  const int64_t G = A.G;
  op.G = G;
  op.nb = nb;
  op.sym_b = sym_b;
  const size_t blk_bytes = (size_t)OZ_SLICES * nb * nb;
  // The two big scratch buffers (the operands' size again) first; with
  // try_only an allocation failure returns false (nothing launched) so the
  // caller can fall back to the DMMA kernel.
  const size_t a_bytes = (size_t)A.nblocks * blk_bytes;
  const size_t b_bytes = sym_b ? 0 : (size_t)B.nblocks * blk_bytes;
  static const bool force_fail = getenv("SPAMM_OZ_FORCE_NOMEM") != nullptr;  // test hook
  if (try_only && force_fail) return false;
  // The A slices of the SP2 loop's X*X: the kept buffer (slice_cache) for
  // operands up to 1 GB.
  SliceCache& cache = slice_cache();
  // (sym: the row exponents and the transposed-slot map ride in the same buffer)
  const size_t extra = sym_b ? (size_t)G * nb * 4 + (size_t)(A.nblocks > 0 ? A.nblocks : 1) * 4 : 0;
  const size_t want = a_bytes + extra;
  if (a_bytes && want <= (size_t(1) << 30) && !cache.busy) {
    if (cache.pending) SPAMM_CK(cudaStreamWaitEvent(s, cache.done, 0));  // last K4z done with it
    if (cache.bytes < want) {
      if (cache.p) {
        if (cache.pending) SPAMM_CK(cudaEventSynchronize(cache.done));
        cudaFree(cache.p);
      }
      cache.pending = false;
      cache.p = nullptr;
      cache.bytes = 0;
      if (cudaMalloc(reinterpret_cast<void**>(&cache.p), want) == cudaSuccess) {
        cache.bytes = want;
      } else {
        cudaGetLastError();
        cache.p = nullptr;
      }
    }
    if (cache.p) {
      op.as = cache.p;
      op.as_cached = true;
      cache.busy = true;
    }
  }
  op.release_cache = slice_cache_release;
  if (op.as_cached) {
    if (!try_only) op.bs = static_cast<int8_t*>(dmalloc_bytes(b_bytes, s));
    else if (b_bytes &&
             cudaMallocAsync(reinterpret_cast<void**>(&op.bs), b_bytes, s) != cudaSuccess) {
      cudaGetLastError();
      op.bs = nullptr;
      cache.busy = false;
      op.as = nullptr;
      op.as_cached = false;
      return false;
    }
  } else if (try_only) {
    if (a_bytes && cudaMallocAsync(reinterpret_cast<void**>(&op.as), a_bytes, s) != cudaSuccess) {
      cudaGetLastError();
      op.as = nullptr;
      return false;
    }
    if (b_bytes && cudaMallocAsync(reinterpret_cast<void**>(&op.bs), b_bytes, s) != cudaSuccess) {
      cudaGetLastError();
      dfree(op.as, s);
      op.as = op.bs = nullptr;
      return false;
    }
  } else {
    op.as = static_cast<int8_t*>(dmalloc_bytes(a_bytes, s));
    op.bs = static_cast<int8_t*>(dmalloc_bytes(b_bytes, s));
  }
  // Row exponents installed on the matrix (spamm_mat_set_oz_exponents: the
  // multi-GPU driver all-reduces them so that a shard's extended operand
  // scales its rows exactly as the whole matrix would) are used as given.
  const bool ex_a_given = A.oz_ex_row != nullptr;
  if (op.as_cached && sym_b) {
    op.ex_a = reinterpret_cast<int*>(op.as + a_bytes);
    op.b_tr = op.ex_a + G * nb;
    op.tail_cached = true;
  } else if (!ex_a_given) {
    op.ex_a = dmalloc<int>(G * nb, s);
  }
  if (ex_a_given) {
    op.ex_a_ext = true;
    op.ex_a = A.oz_ex_row;
  } else {
    SPAMM_CK(cudaMemsetAsync(op.ex_a, 0x80, G * nb * sizeof(int), s));
  }
  const bool ex_b_given = !sym_b && B.oz_ex_col != nullptr;
  if (nb == 32) {
    oz32_operand_passes(A, false, op.ex_a, op.as, s, !ex_a_given);
    if (sym_b) {
      op.ex_b = op.ex_a;
      op.bs = op.as;
      if (!op.tail_cached) op.b_tr = dmalloc<int32_t>(A.nblocks > 0 ? A.nblocks : 1, s);
      if (defer_tr) {
        op.tr_pending = true;
      } else {
        launch_pdl(k_oz_trslot, grid_for(A.nblocks, 256), 256, 0, s, (const int64_t*)A.keys,
                   A.nblocks, G, (const int32_t*)A.slot, op.b_tr);
        SPAMM_LAUNCH_CK();
      }
    } else {
      if (ex_b_given) {
        op.ex_b_ext = true;
        op.ex_b = B.oz_ex_col;
      } else {
        op.ex_b = dmalloc<int>(G * nb, s);
        SPAMM_CK(cudaMemsetAsync(op.ex_b, 0x80, G * nb * sizeof(int), s));
      }
      oz32_operand_passes(B, true, op.ex_b, op.bs, s, !ex_b_given);
    }
    return true;
  }
  // CTAs per SM of the two passes: 2 of the 4 that fit, leaving room for the
  // latency-bound cull and finalisation kernels that run beside them on the
  // main stream (cfg4 solve, interleaved A/B: 2 per SM 30.7, a full wave
  // 30.9, 1 per SM 31.3 ms).  SPAMM_OZ_SPLIT_CTAS=n caps at n per SM (0: a
  // full wave; < 0: one CTA per block).
  static const int pass_ctas = [] {
    const char* v = getenv("SPAMM_OZ_SPLIT_CTAS");
    return v ? atoi(v) : 2;
  }();
  auto wave_of = [](int full) {
    return pass_ctas > 0 ? std::min(full, pass_ctas * multiprocessors())
                         : pass_ctas < 0 ? INT_MAX : full;
  };
  static const int wave_ex = wave_of(resident_wave(k_oz_exponents, 256));
  static const int wave_split = wave_of(resident_wave(k_oz_split, 256));
  const int gx = grid_for(A.nblocks, 1, wave_split);
  // symmetric: the transposed-slot map comes out of A's split
  if (sym_b && !op.tail_cached) op.b_tr = dmalloc<int32_t>(A.nblocks > 0 ? A.nblocks : 1, s);
  int32_t* tr = sym_b && !defer_tr ? op.b_tr : nullptr;
  op.tr_pending = sym_b && defer_tr;
  if (!ex_a_given) {
    launch_plain(k_oz_exponents, grid_for(A.nblocks, 1, wave_ex), 256, 0, s, A.data, A.keys,
                 A.nblocks, G, 0, op.ex_a);
    SPAMM_LAUNCH_CK();
    oz_dbg("exponents A", s);
    launch_pdl(k_oz_split, gx, 256, 0, s, A.data, A.keys, A.nblocks, G, 0, (const int*)op.ex_a,
               op.as, (const int32_t*)A.slot, tr);
  } else {  // (first launch after the cross-stream wait: plain)
    launch_plain(k_oz_split, gx, 256, 0, s, A.data, A.keys, A.nblocks, G, 0,
                 (const int*)op.ex_a, op.as, (const int32_t*)A.slot, tr);
  }
  SPAMM_LAUNCH_CK();
  oz_dbg("split A", s);
  if (sym_b) {
    op.ex_b = op.ex_a;
    op.bs = op.as;
  } else {
    const int gy = grid_for(B.nblocks, 1, wave_split);
    if (ex_b_given) {
      op.ex_b_ext = true;
      op.ex_b = B.oz_ex_col;
    } else {
      op.ex_b = dmalloc<int>(G * OZ_NB, s);
      SPAMM_CK(cudaMemsetAsync(op.ex_b, 0x80, G * OZ_NB * sizeof(int), s));
      launch_pdl(k_oz_exponents, grid_for(B.nblocks, 1, wave_ex), 256, 0, s, B.data, B.keys, B.nblocks, G, 1, op.ex_b);
      SPAMM_LAUNCH_CK();
    }
    launch_pdl(k_oz_split, gy, 256, 0, s, B.data, B.keys, B.nblocks, G, 1, (const int*)op.ex_b,
               op.bs, (const int32_t*)nullptr, (int32_t*)nullptr);
    SPAMM_LAUNCH_CK();
    oz_dbg("B passes", s);
  }
  return true;
}

void ozaki_finish_tr(const Mat& A, OzakiOperands& op, cudaStream_t s) {
  if (!op.tr_pending) return;
  launch_plain(k_oz_trslot, grid_for(A.nblocks, 256), 256, 0, s, (const int64_t*)A.keys,
               A.nblocks, A.G, (const int32_t*)A.slot, op.b_tr);
  SPAMM_LAUNCH_CK();
  op.tr_pending = false;
}

void ozaki_release(OzakiOperands& op, cudaStream_t s) {
  if (!op.tail_cached) dfree(op.b_tr, s);
  if (!op.sym_b) {
    if (!op.ex_b_ext) dfree(op.ex_b, s);
    dfree(op.bs, s);
  }
  if (!op.tail_cached && !op.ex_a_ext) dfree(op.ex_a, s);
  if (op.as_cached) {
    if (op.release_cache) op.release_cache(s);
  } else {
    dfree(op.as, s);
  }
  op = OzakiOperands();
}

void ozaki_exponents(const Mat& M, bool by_col, int* ex, cudaStream_t s) {
  if (!ozaki_supported(M.nb)) throw CudaError("INT8-sliced leaf kernel needs block size 32 or 64");
  SPAMM_CK(cudaMemsetAsync(ex, 0x80, M.G * M.nb * sizeof(int), s));
  if (M.nblocks == 0) return;
  if (M.nb == 32) {
    oz32_exponents(M, by_col, ex, s);
    return;
  }
  static const int wave_ex = resident_wave(k_oz_exponents, 256);
  launch_plain(k_oz_exponents, grid_for(M.nblocks, 1, wave_ex), 256, 0, s, (const double*)M.data, (const int64_t*)M.keys,
               M.nblocks, M.G, by_col ? 1 : 0, ex);
  SPAMM_LAUNCH_CK();
}

template <class Idx>
void ozaki_launch(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                  const int64_t* c_out, const int64_t* c_mirror, bool accumulate, const Mat& A,
                  const Mat& B, const OzakiOperands& op, double* C, cudaStream_t s,
                  LptSchedule lpt, int* ex_out) {
  if (n_seg <= 0) return;
  const int32_t* order = lpt.order;
  int* counter = lpt.counter;
  int* scratch = nullptr;
  // Nb = 64: C blocks are claimed in Morton order: neighbouring CTAs share
  // operand rows and columns in L2 (measured 28.2 vs 28.9 ms of K4z per cfg4
  // solve against the longest-first order, whose tail advantage the short,
  // uniform K4z blocks do not need).  Nb = 32: longest first -- a launch is
  // ~9 C blocks per CTA, so the last wave of a Morton-ordered launch (the long
  // diagonal blocks of the curve's end) leaves ~16 % of the launch to a tail,
  // and the whole slice set (41 MB at cfg3) sits in L2 whatever the order.
  // SPAMM_K4_ORDER=lpt / morton selects one order for both.
  static const int order_mode = [] {
    const char* v = getenv("SPAMM_K4_ORDER");
    return !v ? 0 : strcmp(v, "lpt") == 0 ? 1 : strcmp(v, "morton") == 0 ? 2 : 0;
  }();
  const bool morton = order_mode == 2 || (order_mode == 0 && op.nb != 32);
  if (morton) {
    scratch = dmalloc<int>(1, s);
    SPAMM_CK(cudaMemsetAsync(scratch, 0, sizeof(int), s));
    counter = scratch;
    order = nullptr;
  } else if (!order || !counter) {
    scratch = lpt_schedule(n_seg, seg, &order, &counter, s);
  }
  if (op.nb == 32) {
    oz32_launch<Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, op, C, s,
                     order, counter, ex_out);
    dfree(scratch, s);
    return;
  }
  static const int hint = [] {  // L2 policy experiment bits (see the kernel)
    const char* v = getenv("SPAMM_K4Z_HINT");
    return v ? atoi(v) : 0;
  }();
  static const bool want_prof = getenv("SPAMM_K4Z_PROF") != nullptr;
  long long* prof = nullptr;
  auto kern = want_prof ? k_leaf_ozaki<Idx, true> : k_leaf_ozaki<Idx, false>;
  static std::once_flag once;
  std::call_once(once, [&] {
    SPAMM_CK(cudaFuncSetAttribute(k_leaf_ozaki<Idx, true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_SMEM));
    SPAMM_CK(cudaFuncSetAttribute(k_leaf_ozaki<Idx, false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)OZ_SMEM));
  });
  int64_t grid = multiprocessors();
  if (grid > n_seg) grid = n_seg;
  if (want_prof) {
    prof = dmalloc<long long>((size_t)grid * 16, s);
    SPAMM_CK(cudaMemsetAsync(prof, 0, (size_t)grid * 128, s));
  }
  // (plain launch: K4z follows a wait on the pre-pass stream, see launch_plain)
  launch_plain(kern, (unsigned)grid, OZ_THREADS, OZ_SMEM, s, n_seg, seg, a_idx, b_idx,
             (const int32_t*)op.b_tr, (const int64_t*)A.keys, (const int64_t*)B.keys, op.G,
             (const int8_t*)op.as, (const int8_t*)op.bs, (const int*)op.ex_a, (const int*)op.ex_b,
             c_out, c_mirror, accumulate ? 1 : 0, C, order, counter, hint, prof,
             (const double*)A.data, (const double*)B.data, ex_out);
  SPAMM_LAUNCH_CK();
  oz_dbg("k4z", s);
  if (prof) {  // SPAMM_K4Z_PROF=1: per-launch cycle breakdown (diagnostics; syncs)
    std::vector<long long> h((size_t)grid * 16);
    SPAMM_CK(cudaMemcpyAsync(h.data(), prof, h.size() * 8, cudaMemcpyDeviceToHost, s));
    SPAMM_CK(cudaStreamSynchronize(s));
    double a[12] = {0}, lo = 1e300, hi = 0;
    for (int64_t b = 0; b < grid; ++b) {
      for (int i = 0; i < 12; ++i) a[i] += (double)h[b * 16 + i] / grid;
      lo = std::min(lo, (double)h[b * 16]);
      hi = std::max(hi, (double)h[b * 16]);
    }
    {  // globaltimer spans (us) from the first CTA's entry
      long long e0 = LLONG_MAX, e1 = 0, m1 = 0, x1 = 0;
      double mavg = 0;
      for (int64_t b = 0; b < grid; ++b) {
        e0 = std::min(e0, h[b * 16 + 12]);
        e1 = std::max(e1, h[b * 16 + 12]);
      }
      for (int64_t b = 0; b < grid; ++b) {
        m1 = std::max(m1, h[b * 16 + 13]);
        x1 = std::max(x1, h[b * 16 + 14]);
        mavg += (double)(h[b * 16 + 13] - e0) / grid;
      }
      fprintf(stderr,
              "[k4z-span] us: entries 0..%.2f mma end avg %.2f max %.2f epilogue end max %.2f "
              "(clock %.3f GHz)\n",
              (e1 - e0) / 1e3, mavg / 1e3, (m1 - e0) / 1e3, (x1 - e0) / 1e3,
              a[0] / (mavg > 0 ? mavg : 1));
    }
    fprintf(stderr,
            "[k4z] cycles %.0f (CTA min %.0f max %.0f): mma waits full %.0f tempty %.0f, "
            "tasks %.0f (%.0f cyc/task); epi wait %.0f hold %.0f all %.0f blocks %.0f; "
            "chunk phases tmem %.0f exchange %.0f convert+store %.0f barrier %.0f\n",
            a[0], lo, hi, a[1], a[2], a[3], a[0] / (a[3] > 0 ? a[3] : 1), a[4], a[5], a[6], a[7],
            a[8], a[9], a[10], a[11]);
    dfree(prof, s);
  }
  dfree(scratch, s);
}

template <class Idx>
bool leaf_products_ozaki(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                         const int64_t* c_out, const int64_t* c_mirror, bool accumulate,
                         const Mat& A, const Mat& B, bool sym_b, double* C, cudaStream_t s,
                         LptSchedule lpt, bool try_only, int* ex_out) {
  if (n_seg <= 0) return true;
  OzakiOperands op;
  if (!ozaki_prepare(A, B, sym_b, s, op, try_only)) return false;
  ozaki_launch<Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, op, C, s, lpt,
                    ex_out);
  ozaki_release(op, s);
  return true;
}

template void ozaki_launch<int32_t>(int64_t, const int64_t*, const int32_t*, const int32_t*,
                                    const int64_t*, const int64_t*, bool, const Mat&, const Mat&,
                                    const OzakiOperands&, double*, cudaStream_t, LptSchedule,
                                    int*);
template bool leaf_products_ozaki<int32_t>(int64_t, const int64_t*, const int32_t*,
                                           const int32_t*, const int64_t*, const int64_t*, bool,
                                           const Mat&, const Mat&, bool, double*, cudaStream_t,
                                           LptSchedule, bool, int*);
template bool leaf_products_ozaki<int64_t>(int64_t, const int64_t*, const int64_t*,
                                           const int64_t*, const int64_t*, const int64_t*, bool,
                                           const Mat&, const Mat&, bool, double*, cudaStream_t,
                                           LptSchedule, bool, int*);

}  // namespace spamm
