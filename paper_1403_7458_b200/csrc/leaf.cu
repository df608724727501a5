// K4: batched leaf products with a task-sorted segmented reduction.
//
// Reference: _gemm_acc / _gemm_batch (kernel.py:64-77).  For every C block
// (one segment of the task list, tasks k-ascending) C_ij = sum_k A_ik B_kj.
// One CTA owns one C block for its whole segment, so the reduction over k
// happens in registers in task order -- no atomics, bitwise run-to-run
// deterministic.
//
// LEAF_DMMA: sm_100a has no f64 tcgen05 kind; FP64 tensor math is
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, measured 37.1 TF/s peak on B200,
// profiles/fp64_peak_r01.json).  A/B blocks are staged through a
// STAGES-deep cp.async ring in shared memory (rows padded by 4 doubles:
// conflict-free fragment loads), accumulators live in registers.
// LEAF_EXACT: CUDA-core DMUL+DADD in the reference's exact order (i-k-j,
// k ascending, unfused): bitwise identical to the reference.
#include "internal.h"

namespace spamm {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int NB, int WARPS_M, int WARPS_N, int STAGES>
struct DmmaCfg {
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int LD = NB + 4;
  static constexpr int TILE = NB * LD;
  static constexpr size_t SMEM = (size_t)STAGES * 2 * TILE * sizeof(double);
};

template <int NB, int WARPS_M, int WARPS_N, int STAGES, class Idx>
__global__ void __launch_bounds__(32 * WARPS_M* WARPS_N)
    k_leaf_dmma(const int64_t* __restrict__ seg, const Idx* __restrict__ a_idx,
                const Idx* __restrict__ b_idx, const int64_t* __restrict__ c_out,
                const int64_t* __restrict__ c_mirror, int accumulate,
                const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C) {
  using Cfg = DmmaCfg<NB, WARPS_M, WARPS_N, STAGES>;
  constexpr int NTHR = Cfg::THREADS, LD = Cfg::LD, TILE = Cfg::TILE;
  constexpr int WTM = NB / WARPS_M, WTN = NB / WARPS_N, MT = WTM / 8, NT = WTN / 8;
  constexpr int CHUNKS = NB * NB / 2;  // 16-byte chunks per block
  extern __shared__ __align__(16) double smem[];

  const int64_t m = blockIdx.x;
  const int64_t s0 = seg[m];
  const int n = (int)(seg[m + 1] - s0);
  double* Cb = C + (c_out ? c_out[m] : m) * (int64_t)(NB * NB);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / WARPS_N, wn = warp % WARPS_N;
  const int r8 = lane >> 2, c4 = lane & 3;

  double acc[MT][NT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      if (accumulate) {
        const double2 v = *reinterpret_cast<const double2*>(
            Cb + (wm * WTM + mt * 8 + r8) * NB + wn * WTN + nt * 8 + 2 * c4);
        acc[mt][nt][0] = v.x;
        acc[mt][nt][1] = v.y;
      } else {
        acc[mt][nt][0] = 0.0;
        acc[mt][nt][1] = 0.0;
      }
    }

  auto load = [&](int t, int st) {
    const double* a = A + (int64_t)a_idx[s0 + t] * (NB * NB);
    const double* b = B + (int64_t)b_idx[s0 + t] * (NB * NB);
    double* sa = smem + st * 2 * TILE;
    double* sb = sa + TILE;
#pragma unroll
    for (int c = threadIdx.x; c < CHUNKS; c += NTHR) {
      const int r = (2 * c) / NB, col = (2 * c) % NB;
      cp_async16(sa + r * LD + col, a + 2 * c);
      cp_async16(sb + r * LD + col, b + 2 * c);
    }
  };

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < n) load(st, st);
    cp_async_commit();
  }
  int st_use = 0, st_load = STAGES - 1;
  for (int it = 0; it < n; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (it + STAGES - 1 < n) load(it + STAGES - 1, st_load);
    cp_async_commit();
    const double* sa = smem + st_use * 2 * TILE;
    const double* sb = sa + TILE;
#pragma unroll
    for (int kk = 0; kk < NB; kk += 4) {
      double af[MT], bf[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) af[mt] = sa[(wm * WTM + mt * 8 + r8) * LD + kk + c4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[nt] = sb[(kk + c4) * LD + wn * WTN + nt * 8 + r8];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma884(acc[mt][nt], af[mt], bf[nt]);
    }
    st_use = st_use + 1 == STAGES ? 0 : st_use + 1;
    st_load = st_load + 1 == STAGES ? 0 : st_load + 1;
  }
  cp_async_wait<0>();

#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double2 v;
      v.x = acc[mt][nt][0];
      v.y = acc[mt][nt][1];
      *reinterpret_cast<double2*>(Cb + (wm * WTM + mt * 8 + r8) * NB + wn * WTN + nt * 8 + 2 * c4) = v;
    }
  const int64_t mi = c_mirror ? c_mirror[m] : -1;
  if (mi >= 0) {
    double* Cm = C + mi * (int64_t)(NB * NB);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int r = wm * WTM + mt * 8 + r8, c = wn * WTN + nt * 8 + 2 * c4;
        Cm[c * NB + r] = acc[mt][nt][0];
        Cm[(c + 1) * NB + r] = acc[mt][nt][1];
      }
  }
}

// Exact path, nb <= 64: blocks staged in smem, each thread owns EPT elements.
template <class Idx, int EPT>
__global__ void __launch_bounds__(256)
    k_leaf_exact_smem(const int64_t* __restrict__ seg, const Idx* __restrict__ a_idx,
                      const Idx* __restrict__ b_idx, const int64_t* __restrict__ c_out,
                      const int64_t* __restrict__ c_mirror, int accumulate,
                      const double* __restrict__ A, const double* __restrict__ B,
                      double* __restrict__ C, int nb) {
  extern __shared__ __align__(16) double sm[];
  const int nb2 = nb * nb;
  double* sa = sm;
  double* sb = sm + nb2;
  const int64_t m = blockIdx.x;
  const int64_t s0 = seg[m], s1 = seg[m + 1];
  double* Cb = C + (c_out ? c_out[m] : m) * (int64_t)nb2;
  double acc[EPT];
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int e = threadIdx.x + r * blockDim.x;
    acc[r] = (accumulate && e < nb2) ? Cb[e] : 0.0;
  }
  for (int64_t t = s0; t < s1; ++t) {
    __syncthreads();
    const double* a = A + (int64_t)a_idx[t] * nb2;
    const double* b = B + (int64_t)b_idx[t] * nb2;
    for (int e = threadIdx.x; e < nb2; e += blockDim.x) {
      sa[e] = a[e];
      sb[e] = b[e];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < EPT; ++r) {
      const int e = threadIdx.x + r * blockDim.x;
      if (e < nb2) {
        const int i = e / nb, j = e % nb;
        double c = acc[r];
        for (int kk = 0; kk < nb; ++kk) c = __dadd_rn(c, __dmul_rn(sa[i * nb + kk], sb[kk * nb + j]));
        acc[r] = c;
      }
    }
  }
  const int64_t mi = c_mirror ? c_mirror[m] : -1;
  double* Cm = mi >= 0 ? C + mi * (int64_t)nb2 : nullptr;
#pragma unroll
  for (int r = 0; r < EPT; ++r) {
    const int e = threadIdx.x + r * blockDim.x;
    if (e < nb2) {
      Cb[e] = acc[r];
      if (Cm) Cm[(e % nb) * nb + e / nb] = acc[r];
    }
  }
}

// Exact path, any nb: one thread per C element, operands read through L1/L2.
template <class Idx>
__global__ void __launch_bounds__(256)
    k_leaf_exact_global(const int64_t* __restrict__ seg, const Idx* __restrict__ a_idx,
                        const Idx* __restrict__ b_idx, const int64_t* __restrict__ c_out,
                        const int64_t* __restrict__ c_mirror, int accumulate,
                        const double* __restrict__ A, const double* __restrict__ B,
                        double* __restrict__ C, int nb) {
  const int64_t nb2 = (int64_t)nb * nb;
  const int64_t m = blockIdx.x;
  const int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  if (e >= nb2) return;
  const int64_t i = e / nb, j = e % nb;
  double* Cb = C + (c_out ? c_out[m] : m) * nb2;
  double c = accumulate ? Cb[e] : 0.0;
  for (int64_t t = seg[m]; t < seg[m + 1]; ++t) {
    const double* a = A + (int64_t)a_idx[t] * nb2 + i * nb;
    const double* b = B + (int64_t)b_idx[t] * nb2 + j;
    for (int kk = 0; kk < nb; ++kk) c = __dadd_rn(c, __dmul_rn(__ldg(a + kk), __ldg(b + (int64_t)kk * nb)));
  }
  Cb[e] = c;
  const int64_t mi = c_mirror ? c_mirror[m] : -1;
  if (mi >= 0) C[mi * nb2 + j * nb + i] = c;
}

template <int NB, int WM, int WN, int ST, class Idx>
void launch_dmma(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                 const int64_t* c_out, const int64_t* c_mirror, bool acc, const double* A,
                 const double* B, double* C, cudaStream_t s) {
  using Cfg = DmmaCfg<NB, WM, WN, ST>;
  auto kern = k_leaf_dmma<NB, WM, WN, ST, Idx>;
  static bool attr_set = false;
  if (!attr_set) {
    SPAMM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
    attr_set = true;
  }
  kern<<<(unsigned)n_seg, Cfg::THREADS, Cfg::SMEM, s>>>(seg, a_idx, b_idx, c_out, c_mirror,
                                                        acc ? 1 : 0, A, B, C);
  SPAMM_LAUNCH_CK();
}

}  // namespace

bool dmma_supported(int nb) { return nb == 8 || nb == 16 || nb == 32 || nb == 64; }

template <class Idx>
void leaf_products(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                   const int64_t* c_out, const int64_t* c_mirror, bool accumulate,
                   const double* A, int64_t a_blocks, const double* B, int64_t b_blocks,
                   double* C, int nb, int kernel, cudaStream_t s, LptSchedule lpt) {
  if (n_seg <= 0) return;
  if (n_seg > 0x7fffffffLL) throw CudaError("too many C blocks for one launch");
  if (kernel == LEAF_OZAKI)
    throw CudaError("the INT8-sliced leaf kernel needs matrix operands (row/column exponents)");
  if ((kernel == LEAF_AUTO || kernel == LEAF_DMMA) && tma_leaf_supported(nb)) {
    leaf_products_tma<Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, a_blocks, B,
                           b_blocks, C, nb, s, lpt);
    return;
  }
  const bool dmma = kernel != LEAF_EXACT && dmma_supported(nb);
  if ((kernel == LEAF_DMMA || kernel == LEAF_DMMA_CPASYNC) && !dmma_supported(nb))
    throw CudaError("DMMA leaf kernel needs block size 8, 16, 32 or 64");
  if (dmma) {
    switch (nb) {
      case 8: launch_dmma<8, 1, 1, 4, Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, s); break;
      case 16: launch_dmma<16, 1, 1, 4, Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, s); break;
      case 32: launch_dmma<32, 2, 2, 4, Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, s); break;
      case 64: launch_dmma<64, 2, 2, 3, Idx>(n_seg, seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, s); break;
    }
    return;
  }
  const int nb2 = nb * nb;
  if (nb <= 64) {
    const int threads = nb2 < 256 ? ((nb2 + 31) / 32) * 32 : 256;
    const int ept = (nb2 + threads - 1) / threads;
    const size_t smem = 2 * (size_t)nb2 * sizeof(double);
    if (ept <= 1) {
      k_leaf_exact_smem<Idx, 1><<<(unsigned)n_seg, threads, smem, s>>>(seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, nb);
    } else if (ept <= 4) {
      k_leaf_exact_smem<Idx, 4><<<(unsigned)n_seg, threads, smem, s>>>(seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, nb);
    } else {
      auto kern = k_leaf_exact_smem<Idx, 16>;
      static bool attr = false;
      if (!attr) {
        SPAMM_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 64 * 8));
        attr = true;
      }
      kern<<<(unsigned)n_seg, threads, smem, s>>>(seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, nb);
    }
  } else {
    dim3 grid((unsigned)n_seg, (unsigned)((nb2 + 255) / 256));
    k_leaf_exact_global<Idx><<<grid, 256, 0, s>>>(seg, a_idx, b_idx, c_out, c_mirror, accumulate, A, B, C, nb);
  }
  SPAMM_LAUNCH_CK();
}

template void leaf_products<int32_t>(int64_t, const int64_t*, const int32_t*, const int32_t*,
                                     const int64_t*, const int64_t*, bool, const double*, int64_t,
                                     const double*, int64_t, double*, int, int, cudaStream_t,
                                     LptSchedule);
template void leaf_products<int64_t>(int64_t, const int64_t*, const int64_t*, const int64_t*,
                                     const int64_t*, const int64_t*, bool, const double*, int64_t,
                                     const double*, int64_t, double*, int, int, cudaStream_t,
                                     LptSchedule);

}  // namespace spamm
