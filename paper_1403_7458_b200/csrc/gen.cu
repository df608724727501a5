// K8: on-device generator of the counter-based cluster Hamiltonian (config 5).
//
// BASELINE config 5 (4096 molecules, N = 102,400, Nb = 64) is 84 GB dense:
// it cannot be built on the host.  synth.cluster_dense_cb defines the matrix
// as a pure function of (site positions, original row index, seed); this
// kernel evaluates the same expression with the same IEEE operation sequence
// (SplitMix64 counter hash, Cody-Waite/Horner exp, sqrt, division), so every
// block is bitwise equal to the host reference (tests/test_gpu_gen.py), and
// writes the blocks straight into the Morton-ordered storage.
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.h"

namespace spamm {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double sym_uniform(uint64_t a, uint64_t b, uint64_t n, uint64_t seed) {
  const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
  const uint64_t key = (seed * 0xBF58476D1CE4E5B9ull) ^ (lo * n + hi);
  const double u = __dmul_rn((double)(splitmix64(key) >> 11), 1.0 / 9007199254740992.0);
  return __dadd_rn(__dmul_rn(2.0, u), -1.0);
}

// synth.det_exp: k = rint(x / ln2), r = (x - k ln2_hi) - k ln2_lo, degree-13
// Horner with coefficients 1/n! (each the correctly rounded reciprocal).
__device__ __forceinline__ double det_exp(double x) {
  const double k = rint(__dmul_rn(x, 1.44269504088896338700e+00));
  const double r = __dadd_rn(__dadd_rn(x, -__dmul_rn(k, 6.93147180369123816490e-01)),
                             -__dmul_rn(k, 1.90821492927058770002e-10));
  double p = __ddiv_rn(1.0, 6227020800.0);
  double fact = 6227020800.0;
#pragma unroll
  for (int n = 12; n >= 0; --n) {
    fact = __ddiv_rn(fact, (double)(n + 1));
    p = __dadd_rn(__dmul_rn(p, r), __ddiv_rn(1.0, fact));
  }
  return ldexp(p, (int)k);
}

// H_ab of the counter-based cluster (the expression of k_cluster_blocks, in
// the same operation order), straight from the site arrays.
__device__ __forceinline__ double cluster_elem(const double* __restrict__ pos,
                                               const int64_t* __restrict__ orig,
                                               const double* __restrict__ diag, int64_t n,
                                               double amp, double decay, uint64_t seed, int64_t a,
                                               int64_t b) {
  if (a == b) return diag[a];
  double r2 = 0.0;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const double dd = __dadd_rn(pos[3 * a + ax], -pos[3 * b + ax]);
    r2 = __dadd_rn(r2, __dmul_rn(dd, dd));
  }
  const double x = __ddiv_rn(-__dsqrt_rn(r2), decay);
  const double s = sym_uniform((uint64_t)orig[a], (uint64_t)orig[b], (uint64_t)n, seed);
  return __dmul_rn(__dmul_rn(amp, det_exp(x)), s);
}

// Gershgorin discs of rows [row0, row1) of the cluster H without building it
// (multi-GPU config 5: each rank takes a row range): numpy's pairwise sum of
// |H_row| (the same leaf / fold schedule as ops.cu k_gersh_rows_warp, so the
// bounds are bitwise those of gershgorin() on the stored matrix), one warp
// per row, lanes on the <= 128-element leaves, lane 0 folds them in order.
__global__ void __launch_bounds__(256)
    k_gersh_cluster(const double* __restrict__ pos, const int64_t* __restrict__ orig,
                    const double* __restrict__ diag, int64_t n, double amp, double decay,
                    uint64_t seed, int64_t row0, int64_t row1, const int64_t* __restrict__ leaf_lo,
                    const int32_t* __restrict__ leaf_len, int n_leaves,
                    const int32_t* __restrict__ ops, int n_ops, double* __restrict__ lo,
                    double* __restrict__ hi) {
  extern __shared__ double leafv[];  // [8 warps][n_leaves]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* lv = leafv + (int64_t)warp * n_leaves;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = row0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < row1;
       i += nw) {
    auto at = [&](int64_t c) { return fabs(cluster_elem(pos, orig, diag, n, amp, decay, seed, i, c)); };
    for (int k = lane; k < n_leaves; k += 32) {
      const int64_t l0 = leaf_lo[k];
      const int ln = leaf_len[k];
      double res;
      if (ln < 8) {
        res = 0.0;
        for (int q = 0; q < ln; ++q) res = __dadd_rn(res, at(l0 + q));
      } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = at(l0 + j);
        int q = 8;
        for (; q < ln - (ln % 8); q += 8)
          for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], at(l0 + q + j));
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; q < ln; ++q) res = __dadd_rn(res, at(l0 + q));
      }
      lv[k] = res;
    }
    __syncwarp();
    if (lane == 0) {
      double st[48];
      int sp = 0;
      for (int o = 0; o < n_ops; ++o) {
        const int op = ops[o];
        if (op >= 0) {
          st[sp++] = lv[op];
        } else {
          const double r = st[--sp];
          st[sp - 1] = __dadd_rn(st[sp - 1], r);
        }
      }
      const double d = diag[i];
      const double radius = __dadd_rn(st[0], -fabs(d));
      lo[i - row0] = __dadd_rn(d, -radius);
      hi[i - row0] = __dadd_rn(d, radius);
    }
    __syncwarp();
  }
}

__global__ void k_native_flags(int depth, int64_t nbn, int64_t lo, int64_t hi,
                               uint8_t* __restrict__ flags) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npos;
       p += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    flags[p] = (bi < nbn && bj < nbn && p >= lo && p < hi) ? 1 : 0;
  }
}

__global__ void __launch_bounds__(256)
    k_cluster_blocks(const double* __restrict__ pos, const int64_t* __restrict__ orig,
                     const double* __restrict__ diag, int64_t n, int nb, int depth,
                     const uint8_t* __restrict__ flags, const int64_t* __restrict__ off,
                     double amp, double decay, uint64_t seed, double* __restrict__ data,
                     int64_t* __restrict__ keys) {
  extern __shared__ double sh[];  // rows: x,y,z,orig (4 nb), cols: 4 nb
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int nb2 = nb * nb;
  double* rx = sh;
  double* cx = sh + 4 * nb;
  for (int64_t p = blockIdx.x; p < npos; p += gridDim.x) {
    if (!flags[p]) continue;
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    const int64_t d = off[p];
    __syncthreads();
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
      const int64_t a = (int64_t)bi * nb + t, b = (int64_t)bj * nb + t;
      if (a < n) {
        rx[t] = pos[3 * a];
        rx[nb + t] = pos[3 * a + 1];
        rx[2 * nb + t] = pos[3 * a + 2];
        rx[3 * nb + t] = __longlong_as_double(orig[a]);
      }
      if (b < n) {
        cx[t] = pos[3 * b];
        cx[nb + t] = pos[3 * b + 1];
        cx[2 * nb + t] = pos[3 * b + 2];
        cx[3 * nb + t] = __longlong_as_double(orig[b]);
      }
    }
    __syncthreads();
    double* out = data + d * nb2;
    for (int e = threadIdx.x; e < nb2; e += blockDim.x) {
      const int r = e / nb, c = e % nb;
      const int64_t a = (int64_t)bi * nb + r, b = (int64_t)bj * nb + c;
      double v = 0.0;
      if (a < n && b < n) {
        if (a == b) {
          v = diag[a];
        } else {
          // r2 = sum over axes of (p_a - p_b)^2 in axis order (synth.cluster_dense_cb)
          double r2 = 0.0;
#pragma unroll
          for (int ax = 0; ax < 3; ++ax) {
            const double dd = __dadd_rn(rx[ax * nb + r], -cx[ax * nb + c]);
            r2 = __dadd_rn(r2, __dmul_rn(dd, dd));
          }
          const double x = __ddiv_rn(-__dsqrt_rn(r2), decay);
          const double s = sym_uniform((uint64_t)__double_as_longlong(rx[3 * nb + r]),
                                       (uint64_t)__double_as_longlong(cx[3 * nb + c]),
                                       (uint64_t)n, seed);
          v = __dmul_rn(__dmul_rn(amp, det_exp(x)), s);
        }
      }
      out[e] = v;
    }
    if (threadIdx.x == 0) keys[d] = (int64_t)bi * G + bj;
  }
}

}  // namespace

void cluster_gershgorin(const double* pos, const int64_t* orig, const double* diag, int64_t n,
                        double amp, double decay, uint64_t seed, int64_t row0, int64_t row1,
                        double* eps_min, double* eps_max, cudaStream_t s) {
  std::vector<int64_t> leaf_lo;
  std::vector<int32_t> leaf_len, ops;
  pairwise_schedule(n, leaf_lo, leaf_len, ops);
  const int nl = (int)leaf_lo.size(), no = (int)ops.size();
  const size_t smem = 8 * (size_t)nl * sizeof(double);
  if (smem > 200 * 1024) throw CudaError("cluster Gershgorin: row too long for the leaf buffer");
  const int64_t rows = row1 - row0;
  if (rows <= 0) {
    *eps_min = INFINITY;
    *eps_max = -INFINITY;
    return;
  }
  double* buf = dmalloc<double>(2 * rows + 2, s);
  int64_t* d_lo = dmalloc<int64_t>(nl, s);
  int32_t* d_len = dmalloc<int32_t>(nl, s);
  int32_t* d_ops = dmalloc<int32_t>(no, s);
  SPAMM_CK(cudaMemcpyAsync(d_lo, leaf_lo.data(), nl * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  SPAMM_CK(cudaMemcpyAsync(d_len, leaf_len.data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  SPAMM_CK(cudaMemcpyAsync(d_ops, ops.data(), no * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (smem > 48 * 1024)
    SPAMM_CK(cudaFuncSetAttribute(k_gersh_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  k_gersh_cluster<<<grid_for(rows * 32, 256, 148LL * 16), 256, smem, s>>>(
      pos, orig, diag, n, amp, decay, seed, row0, row1, d_lo, d_len, nl, d_ops, no, buf,
      buf + rows);
  SPAMM_LAUNCH_CK();
  minmax_launch(buf, buf + rows, rows, buf + 2 * rows, s);
  int64_t bits[2];
  d2h_sync(bits, reinterpret_cast<const int64_t*>(buf + 2 * rows), 2, s);
  memcpy(eps_min, &bits[0], 8);
  memcpy(eps_max, &bits[1], 8);
  dfree(buf, s);
  dfree(d_lo, s);
  dfree(d_len, s);
  dfree(d_ops, s);
}

void cluster_build(const double* pos, const int64_t* orig, const double* diag, double amp,
                   double decay, uint64_t seed, Mat& m, cudaStream_t s, int64_t lo,
                   int64_t hi) {
  const int64_t G = int64_t(1) << m.depth, npos = G * G;
  const int64_t nbn = (m.n_native + m.nb - 1) / m.nb;
  const bool whole = lo <= 0 && (hi < 0 || hi >= npos);
  if (hi < 0) hi = npos;
  uint8_t* flags = dmalloc<uint8_t>(npos, s);
  int64_t* off = dmalloc<int64_t>(npos + 1, s);
  k_native_flags<<<grid_for(npos, 256), 256, 0, s>>>(m.depth, nbn, lo, hi, flags);
  SPAMM_LAUNCH_CK();
  scan_exclusive_u8(flags, npos, off, s);
  if (whole) {
    m.nblocks = nbn * nbn;
  } else {
    d2h_sync(&m.nblocks, off + npos, 1, s);
  }
  m.data = dmalloc<double>((size_t)m.nblocks * m.nb * m.nb, s);
  m.keys = dmalloc<int64_t>(m.nblocks, s);
  if (m.nblocks > 0) {
    k_cluster_blocks<<<grid_for(m.nblocks, 1, 148LL * 32), 256, 8 * m.nb * sizeof(double), s>>>(
        pos, orig, diag, m.n_native, m.nb, m.depth, flags, off, amp, decay, seed, m.data, m.keys);
    SPAMM_LAUNCH_CK();
  }
  dfree(flags, s);
  dfree(off, s);
  finalize(m, s);
  // r2, s and the diagonal are exactly symmetric by construction (a Morton
  // shard holds part of a symmetric matrix: the caller sets the flag with the
  // global pyramid, spamm_mat_set_pyramid)
  m.sym = whole;
}

}  // namespace spamm
