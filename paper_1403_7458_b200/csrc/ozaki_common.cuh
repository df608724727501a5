// Device helpers shared by the INT8-sliced leaf kernels (leaf_ozaki.cu for
// Nb = 64, leaf_ozaki32.cu for Nb = 32): the digit split, mbarrier / bulk-copy
// / tcgen05 PTX wrappers.  See leaf_ozaki.cu for the scheme.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace spamm {
namespace ozk {

constexpr int OZ_EXP_NONE = (int)0x80808080;  // memset pattern: "no nonzero seen"
// Row / column holding an Inf or NaN (atomicMax: dominates every exponent).
// Its digits are all zero, and the epilogue recomputes the C elements of that
// row / column in FP64 in the reference's order (oz_exact_elem), so non-finite
// operands give the reference's Inf / NaN pattern (kernel.py:64-77).
constexpr int OZ_EXP_BAD = 0x7fffffff;

__device__ __forceinline__ int oz_exp(int e) { return e == OZ_EXP_NONE ? 0 : e; }

// sum_d S_d 2^-8d (d = 0 .. NL-1) in the Horner order of the design --
// v = S_{NL-1}, then v = RN(v 2^-8 + S_d) for d = NL-2 .. 0 -- bitwise, with
// fewer FP64 operations: for |S_d| < 2^31 the first two steps are exact
// (<= 40 and 48 significant bits) and the third rounds the exact value
// T 2^-24, T = S_{NL-1} + 2^8 S_{NL-2} + 2^16 S_{NL-3} + 2^24 S_{NL-4}
// (|T| < 2^56, exact in int64), so those three steps are one int64
// conversion; the fourth folds the 2^-24 into its (exact) scaling.
template <int NL>
__device__ __forceinline__ double oz_horner(const int (&S)[NL]) {
  static_assert(NL >= 5, "oz_horner: at least 5 digit levels");
  const long long T = (long long)S[NL - 1] + (long long)S[NL - 2] * 256LL +
                      (long long)S[NL - 3] * 65536LL + (long long)S[NL - 4] * 16777216LL;
  double v = __fma_rn(__ll2double_rn(T), 0x1p-32, (double)S[NL - 5]);
#pragma unroll
  for (int d = NL - 6; d >= 0; --d) v = __fma_rn(v, 0x1p-8, (double)S[d]);
  return v;
}

// th + tl 2^-32 rounded to double (|th| < 2^62.1, |tl| < 2^54.1; the value of
// sum_d S_d 2^-8d scaled by 2^32): hi = RN(th) and its exact remainder
// th - hi (|.| <= 2^9, an integer), the remainder plus the low part in one
// FMA, then one final add -- within a few units of 2^-60 of the exactly
// rounded value, deterministic in (th, tl).
__device__ __forceinline__ double oz_round2(long long th, long long tl) {
  const double hi = __ll2double_rn(th);
  const long long rem = th - __double2ll_rz(hi);  // exact: hi is an integer < 2^63
  const double lo = __fma_rn(__ll2double_rn(tl), 0x1p-32, (double)rem);
  return __dadd_rn(hi, lo);
}

// 32-byte global accesses (sm_100: LDG/STG.256): one whole sector per lane
// for the four C elements an epilogue thread owns in a row.
__device__ __forceinline__ void oz_ld4(const double* p, double& a, double& b, double& c,
                                       double& d) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
__device__ __forceinline__ void oz_st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
__device__ __forceinline__ unsigned long long oz_policy_evict_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void oz_st4_hint(double* p, double a, double b, double c, double d,
                                            unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "d"(a),
               "d"(b), "d"(c), "d"(d), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void oz_st1_hint(double* p, double a, unsigned long long pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(a), "l"(pol) : "memory");
}
__device__ __forceinline__ void oz_st4_cs(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}
// |x| for the exponent passes, +Inf for a non-finite x (fmax would drop NaN).
__device__ __forceinline__ double oz_absf(double x) {
  return isfinite(x) ? fabs(x) : __longlong_as_double(0x7ff0000000000000LL);
}
// C element (r, c) of one C block over its tasks [t0, t1) in the reference's
// order (_gemm_acc, kernel.py:64-77: i-k-j loops, tasks k ascending, unfused
// multiply and add) starting from acc -- bitwise the exact leaf kernel.
template <class Idx>
__device__ __noinline__ double oz_exact_elem(double acc, const double* __restrict__ A,
                                             const double* __restrict__ B,
                                             const Idx* __restrict__ a_idx,
                                             const Idx* __restrict__ b_idx, int64_t t0, int64_t t1,
                                             int nb, int r, int c) {
  const int64_t nb2 = (int64_t)nb * nb;
  for (int64_t t = t0; t < t1; ++t) {
    const double* a = A + (int64_t)a_idx[t] * nb2 + (int64_t)r * nb;
    const double* b = B + (int64_t)b_idx[t] * nb2 + c;
    for (int k = 0; k < nb; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k], b[(int64_t)k * nb]));
  }
  return acc;
}
// Row / column exponent E: max |x| < 2^E, bumped when the mantissa is within
// 2^-7.5 of 1 so that |x 2^(7-E)| <= 127.25 -- the leading signed digit then
// stays in [-128, 127] after the carry from the tail.
__device__ __forceinline__ int oz_frexp(double mx) {
  int e;
  const double f = frexp(mx, &e);
  return f >= 0.994140625 ? e + 1 : e;
}
// The scale exponent of |x| as an unsigned code in the exponents' order (0:
// x == 0, 0xFFFF: Inf / NaN = OZ_EXP_BAD, else oz_frexp(|x|) + 0x8000), from
// the bit pattern with integer operations only (cheap enough for the K4z
// epilogue): frexp's exponent is the biased exponent - 1022 (subnormals: the
// bit length of the mantissa - 1074), bumped when the 8 mantissa bits after
// the leading one are >= 0xFD, i.e. frac >= 0.994140625 as in oz_frexp.
__device__ __forceinline__ unsigned oz_ex_code(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x) & 0x7FFFFFFFFFFFFFFFull;
  if (b == 0) return 0u;
  const unsigned E = (unsigned)(b >> 52);
  if (E == 0x7FFu) return 0xFFFFu;
  int e;
  if (E) {
    e = (int)E - 1022 + (((b >> 44) & 0xFF) >= 0xFD ? 1 : 0);
  } else {
    const int lz = __clzll((long long)b);
    e = (64 - lz) - 1074 + (((b << (lz + 1)) >> 56) >= 0xFD ? 1 : 0);
  }
  return (unsigned)(e + 0x8000);
}
__device__ __forceinline__ int oz_ex_decode(unsigned c) {
  return c == 0xFFFFu ? OZ_EXP_BAD : (int)c - 0x8000;
}
// The row / column exponent of a reduced max oz_absf (mx > 0).
__device__ __forceinline__ int oz_exp_of(double mx) {
  return isinf(mx) ? OZ_EXP_BAD : oz_frexp(mx);
}


// The 8 signed digits of x against the scale 2^E, packed as bytes (slice p =
// byte 7 - p): V = floor(|x| 2^(63-E)) from the bit pattern (|x| 2^-E < 1, so
// V < 2^63; the bytes of V are the floor digits), then the carry pass as one
// add -- W = V + 0x80 (0x7F for x < 0) in each of the 7 low bytes -- whose
// bytes XOR the same constant are the signed digits (negated for x < 0, the
// carry threshold 129 there keeping them in [-128, 127]).
__device__ __forceinline__ uint64_t oz_digits(double x, int e) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const bool neg = bits >> 63;
  int be = (int)((bits >> 52) & 0x7FF);
  uint64_t m = bits & 0xFFFFFFFFFFFFFull;
  if (be) m |= 1ull << 52;
  else be = 1;  // subnormal (or zero: m = 0)
  const int sh = be - 1012 - e;  // |x| 2^(63-E) = m 2^sh, sh <= 10
  const uint64_t v = sh >= 0 ? m << sh : (sh > -64 ? m >> -sh : 0ull);
  const uint64_t off = neg ? 0x007F7F7F7F7F7F7Full : 0x0080808080808080ull;
  const uint64_t w = v + off;
  const uint64_t top = neg ? (uint64_t)((-(int)(w >> 56)) & 0xFF) : (w >> 56);
  return ((w ^ off) & 0x00FFFFFFFFFFFFFFull) | (top << 56);
}

// Bytes `byte` of four packed digit words -> one 32-bit word (element order).
__device__ __forceinline__ uint32_t oz_gather4(uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                               int byte) {
  const uint32_t sel = (uint32_t)byte | ((uint32_t)(4 + byte) << 4);
  return __byte_perm(__byte_perm(a, b, sel), __byte_perm(c, d, sel), 0x5410);
}


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
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_pol(uint32_t dst, const void* src, uint32_t bytes,
                                             uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tc_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// Shared-memory matrix descriptor: K-major, no swizzle, LBO 128 B (the two
// 16-byte k-chunks of one MMA), SBO = stride of 8-row groups, version 1 (sm_100).
__device__ __forceinline__ uint64_t oz_desc(uint32_t addr, uint32_t sbo = 512) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
// Instruction descriptor: D s32, A/B signed int8, both K-major, N = 128, M = 128.
constexpr uint32_t OZ_IDESC =
    (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
// N = 256 (four B slices): the accumulator spans two adjacent 128-column tiles.
constexpr uint32_t OZ_IDESC_N256 =
    (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ void oz_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc,
                                       uint32_t idesc = OZ_IDESC) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void oz_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::
                   "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7])
      : "r"(taddr));
}
// tcgen05.wait::ld, with the loaded registers threaded through so no use of
// them can be scheduled above the wait.
__device__ __forceinline__ void tmem_wait8(int (&v)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7])
               :
               : "memory");
}
__device__ __forceinline__ void tmem_keep8(int (&v)[8]) {
  asm volatile(""
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]));
}


// K4z column exponents produced by a kernel that already streams a block
// warp-wide with lane l holding columns (2l, 2l + 1) mod Nb of every row it
// reads (K1, the SP2 update): m0 / m1 = the lane's max oz_absf over those
// columns; atomicMax into ex[bj * Nb + col] as k_oz_exponents(by_col = 1)
// would.  For a bitwise symmetric matrix these are its row exponents too.
template <int NB>
__device__ __forceinline__ void oz_col_exponents(double m0, double m1, int64_t bj, int* ex,
                                                 int lane) {
  if (NB == 32) {  // lanes l and l ^ 16 hold the same column pair
    m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, 16));
    m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, 16));
    if (lane >= 16) return;
  }
  const int c = (2 * lane) % NB;
  if (m0 > 0.0) atomicMax(ex + bj * NB + c, oz_exp_of(m0));
  if (m1 > 0.0) atomicMax(ex + bj * NB + c + 1, oz_exp_of(m1));
}

}  // namespace ozk
}  // namespace spamm
