// Element-wise builders and reductions on device-resident quadtree matrices.
//
// Reference call sites (each restated with the reference's exact rounding):
//  * build_from_dense   quadtree.py:208-242 (pad, block, keep non-zero blocks)
//  * to_dense           quadtree.py:245-252
//  * identity           quadtree.py:308-323
//  * add_scaled         quadtree.py:281-293: fl(fl(alpha*a) + fl(beta*b)) on the
//                       key union, absent operand = no term
//  * trace              quadtree.py:296-305: einsum("tii->") = sequential sum inside
//                       each diagonal block, then sequential over blocks (key order)
//  * gershgorin_bounds  sp2.py:68-76: numpy pairwise row sums of |F| (block 128,
//                       8 accumulators), radius = rowsum - |diag|
#include <algorithm>
#include <vector>

#include "internal.h"

namespace spamm {

namespace {

constexpr int WARPS_PER_CTA = 8;

__global__ void k_dense_block_flags(const double* __restrict__ dense, int64_t n, int64_t ld, int nb,
                                    int depth, uint8_t* __restrict__ flags) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nb2 = nb * nb;
  for (int64_t p = gw; p < npos; p += nw) {
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    bool any = false;
    for (int e = lane; e < nb2; e += 32) {
      const int64_t r = (int64_t)bi * nb + e / nb, c = (int64_t)bj * nb + e % nb;
      if (r < n && c < n) any |= dense[r * ld + c] != 0.0;
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) flags[p] = any ? 1 : 0;
  }
}

__global__ void k_dense_block_copy(const double* __restrict__ dense, int64_t n, int64_t ld, int nb,
                                   int depth, const uint8_t* __restrict__ flags,
                                   const int64_t* __restrict__ off, double* __restrict__ data,
                                   int64_t* __restrict__ keys) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nb2 = nb * nb;
  for (int64_t p = gw; p < npos; p += nw) {
    if (!flags[p]) continue;
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    const int64_t d = off[p];
    double* out = data + d * nb2;
    for (int e = lane; e < nb2; e += 32) {
      const int64_t r = (int64_t)bi * nb + e / nb, c = (int64_t)bj * nb + e % nb;
      out[e] = (r < n && c < n) ? dense[r * ld + c] : 0.0;
    }
    if (lane == 0) keys[d] = (int64_t)bi * G + bj;
  }
}

__global__ void k_block_store_dense(const double* __restrict__ data, const int64_t* __restrict__ keys,
                                    int64_t m, int nb, int64_t G, int64_t n, int64_t ld,
                                    double* __restrict__ dense) {
  const int nb2 = nb * nb;
  for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
    const int64_t key = keys[b], bi = key / G, bj = key % G;
    for (int e = threadIdx.x; e < nb2; e += blockDim.x) {
      const int64_t r = bi * nb + e / nb, c = bj * nb + e % nb;
      if (r < n && c < n) dense[r * ld + c] = data[b * nb2 + e];
    }
  }
}

__global__ void k_identity(int64_t n, int nb, int64_t G, int64_t n_diag, double* __restrict__ data,
                           int64_t* __restrict__ keys) {
  const int64_t nb2 = (int64_t)nb * nb;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n_diag;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fill = min((int64_t)nb, n - b * nb);
    for (int64_t d = 0; d < fill; ++d) data[b * nb2 + d * nb + d] = 1.0;
    keys[b] = b * G + b;
  }
}

__global__ void k_union_flags(const int32_t* __restrict__ sa, const int32_t* __restrict__ sb,
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

__global__ void k_add_scaled(double alpha, const double* __restrict__ A, const int32_t* __restrict__ sa,
                             double beta, const double* __restrict__ B, const int32_t* __restrict__ sb,
                             int depth, int nb, const uint8_t* __restrict__ flags,
                             const int64_t* __restrict__ off, double* __restrict__ out,
                             int64_t* __restrict__ keys) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  const int nb2 = nb * nb;
  for (int64_t p = blockIdx.x; p < npos; p += gridDim.x) {
    if (!flags[p]) continue;
    uint32_t bi, bj;
    morton_decode((uint64_t)p, bi, bj);
    const int64_t key = (int64_t)bi * G + bj;
    const int32_t ia = sa[key], ib = sb[key];
    const int64_t d = off[p];
    const double* a = ia >= 0 ? A + (int64_t)ia * nb2 : nullptr;
    const double* b = ib >= 0 ? B + (int64_t)ib * nb2 : nullptr;
    double* o = out + d * nb2;
    for (int e = threadIdx.x; e < nb2; e += blockDim.x) {
      double v = a ? __dmul_rn(alpha, a[e]) : 0.0;
      if (b) v = __dadd_rn(v, __dmul_rn(beta, b[e]));
      o[e] = v;
    }
    if (threadIdx.x == 0) keys[d] = key;
  }
}

// Per diagonal block: warp-parallel loads of the diagonal, then a sequential
// sum (lane 0 pulls element d from lane d % 32) -- einsum's inner loop order.
__global__ void k_trace_blocks(const int32_t* __restrict__ slot, const double* __restrict__ data,
                               int64_t G, int nb, double* __restrict__ partial,
                               uint8_t* __restrict__ present) {
  const int64_t nb2 = (int64_t)nb * nb;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < G; b += nw) {
    const int32_t s = slot[b * G + b];
    if (lane == 0) present[b] = s >= 0;
    if (s < 0) continue;
    const double* x = data + (int64_t)s * nb2;
    double acc = 0.0;
    for (int d0 = 0; d0 < nb; d0 += 32) {
      const int d = d0 + lane;
      const double v = d < nb ? x[(int64_t)d * nb + d] : 0.0;
      const int cnt = min(32, nb - d0);
      for (int i = 0; i < cnt; ++i) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, v, i));
    }
    if (lane == 0) partial[b] = acc;
  }
}

__global__ void k_trace(const int32_t* __restrict__ slot, const double* __restrict__ data, int64_t G,
                        int nb, double* __restrict__ partial, uint8_t* __restrict__ present,
                        double* __restrict__ out) {
  (void)slot;
  (void)data;
  if (threadIdx.x != 0) return;
  if (nb == 1) {
    // Nb = 1: einsum sees one contiguous run of diagonal values and uses its
    // two-lane sum_of_arr: per 8 values ((x0+x2)+(x4+x6)) into lane 0, odd
    // ones into lane 1, tail two at a time, then lane0 + lane1.
    double l0 = 0.0, l1 = 0.0, v[8];
    int nv = 0;
    for (int64_t b = 0; b < G; ++b) {
      if (!present[b]) continue;
      v[nv++] = partial[b];
      if (nv == 8) {
        l0 = __dadd_rn(__dadd_rn(__dadd_rn(v[0], v[2]), __dadd_rn(v[4], v[6])), l0);
        l1 = __dadd_rn(__dadd_rn(__dadd_rn(v[1], v[3]), __dadd_rn(v[5], v[7])), l1);
        nv = 0;
      }
    }
    for (int i = 0; i < nv; i += 2) {
      l0 = __dadd_rn(v[i], l0);
      if (i + 1 < nv) l1 = __dadd_rn(v[i + 1], l1);
    }
    out[0] = __dadd_rn(l0, l1);
    return;
  }
  double tot = 0.0;
  for (int64_t b = 0; b < G; ++b)
    if (present[b]) tot = __dadd_rn(tot, partial[b]);
  out[0] = tot;
}

// max |F - F^T| over native entries; non-negative doubles order like their bits.
__global__ void k_asym(const double* __restrict__ data, const int64_t* __restrict__ keys,
                       const int32_t* __restrict__ slot, int64_t m, int nb, int64_t G, int64_t n,
                       unsigned long long* __restrict__ out) {
  const int nb2 = nb * nb;
  double mx = 0.0;
  for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
    const int64_t key = keys[b], bi = key / G, bj = key % G;
    const int32_t t = slot[bj * G + bi];
    for (int e = threadIdx.x; e < nb2; e += blockDim.x) {
      const int r = e / nb, c = e % nb;
      if (bi * nb + r >= n || bj * nb + c >= n) continue;
      const double x = data[b * nb2 + e];
      const double y = t >= 0 ? data[(int64_t)t * nb2 + c * nb + r] : 0.0;
      mx = fmax(mx, fabs(__dadd_rn(x, -y)));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(mx));
}

// |F| row element, walking one native row through the block storage.
struct RowReader {
  const double* data;
  const int32_t* slot;
  int64_t G, row;
  int nb;
  __device__ double at(int64_t c) const {
    const int32_t s = slot[(row / nb) * G + c / nb];
    if (s < 0) return 0.0;
    return fabs(data[(int64_t)s * nb * nb + (row % nb) * nb + (c % nb)]);
  }
};

// numpy pairwise_sum leaf (n <= 128): 8 accumulators, or sequential for n < 8.
__device__ double pw_leaf(const RowReader& rr, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, rr.at(lo + i));
    return res;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = rr.at(lo + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], rr.at(lo + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, rr.at(lo + i));
  return res;
}

// numpy pairwise_sum recursion, iterative (explicit stack).
__device__ double pairwise(const RowReader& rr, int64_t n) {
  struct Frame {
    int64_t lo, n, n2;
    int state;
    double left;
  };
  Frame st[40];
  int sp = 0;
  st[0] = {0, n, 0, 0, 0.0};
  double ret = 0.0;
  while (true) {
    Frame& f = st[sp];
    if (f.state == 0) {
      if (f.n <= 128) {
        ret = pw_leaf(rr, f.lo, f.n);
        if (sp == 0) return ret;
        --sp;
        continue;
      }
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      f.n2 = n2;
      f.state = 1;
      st[sp + 1] = {f.lo, n2, 0, 0, 0.0};
      ++sp;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      st[sp + 1] = {f.lo + f.n2, f.n - f.n2, 0, 0, 0.0};
      ++sp;
    } else {
      ret = __dadd_rn(f.left, ret);
      if (sp == 0) return ret;
      --sp;
    }
  }
}

__global__ void k_gersh_rows(const double* __restrict__ data, const int32_t* __restrict__ slot,
                             int64_t G, int nb, int64_t n, double* __restrict__ lo,
                             double* __restrict__ hi) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    RowReader rr{data, slot, G, i, nb};
    const double rowsum = pairwise(rr, n);
    const int32_t s = slot[(i / nb) * G + i / nb];
    const double d = s >= 0 ? data[(int64_t)s * nb * nb + (i % nb) * nb + (i % nb)] : 0.0;
    const double radius = __dadd_rn(rowsum, -fabs(d));
    lo[i] = __dadd_rn(d, -radius);
    hi[i] = __dadd_rn(d, radius);
  }
}

// Warp per row: numpy's pairwise tree for length n is the same for every row,
// so the host flattens it once into leaves (lo, len) and a post-order op list
// (k >= 0: push leaf k, -1: pop r, pop l, push l + r).  Lanes evaluate leaves
// in parallel (each leaf is a <=128-element run, 8 accumulators), lane 0 then
// folds them in tree order -- the identical sequence of additions.
__global__ void __launch_bounds__(256)
    k_gersh_rows_warp(const double* __restrict__ data, const int32_t* __restrict__ slot, int64_t G,
                      int nb, int64_t n, const int64_t* __restrict__ leaf_lo,
                      const int32_t* __restrict__ leaf_len, int n_leaves,
                      const int32_t* __restrict__ ops, int n_ops, double* __restrict__ lo,
                      double* __restrict__ hi) {
  extern __shared__ double leafv[];  // [8 warps][n_leaves]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* lv = leafv + (int64_t)warp * n_leaves;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    RowReader rr{data, slot, G, i, nb};
    for (int k = lane; k < n_leaves; k += 32) lv[k] = pw_leaf(rr, leaf_lo[k], leaf_len[k]);
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
      const double rowsum = st[0];
      const int32_t s = slot[(i / nb) * G + i / nb];
      const double d = s >= 0 ? data[(int64_t)s * nb * nb + (i % nb) * nb + (i % nb)] : 0.0;
      const double radius = __dadd_rn(rowsum, -fabs(d));
      lo[i] = __dadd_rn(d, -radius);
      hi[i] = __dadd_rn(d, radius);
    }
    __syncwarp();
  }
}

__global__ void k_minmax(const double* __restrict__ lo, const double* __restrict__ hi, int64_t n,
                         double* __restrict__ out) {
  double mn = lo[0], mx = hi[0];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    mn = fmin(mn, lo[i]);
    mx = fmax(mx, hi[i]);
  }
  __shared__ double smn[32], smx[32];
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_down_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    out[0] = mn;
    out[1] = mx;
  }
}

int warp_grid(int64_t nwarps) { return grid_for(nwarps * 32, 32 * WARPS_PER_CTA, 148LL * 64); }

// Exact symmetry: every stored block (i,j) equals the transpose of block (j,i).
__global__ void k_symmetric(const double* __restrict__ data, const int64_t* __restrict__ keys,
                            const int32_t* __restrict__ slot, int64_t m, int nb, int64_t G,
                            int* __restrict__ bad) {
  const int nb2 = nb * nb;
  for (int64_t b = blockIdx.x; b < m; b += gridDim.x) {
    const int64_t key = keys[b], bi = key / G, bj = key % G;
    const int32_t t = slot[bj * G + bi];
    bool ok = t >= 0;
    if (ok)
      for (int e = threadIdx.x; e < nb2; e += blockDim.x) {
        const int r = e / nb, c = e % nb;
        ok &= data[b * nb2 + e] == data[(int64_t)t * nb2 + c * nb + r];
      }
    if (!__syncthreads_and(ok) && threadIdx.x == 0) *bad = 1;
  }
}

}  // namespace

bool is_symmetric(const Mat& m, cudaStream_t s) {
  if (m.nblocks == 0) return true;
  int64_t* flag = dmalloc<int64_t>(1, s);
  SPAMM_CK(cudaMemsetAsync(flag, 0, sizeof(int64_t), s));
  k_symmetric<<<grid_for(m.nblocks, 1, 148LL * 16), 256, 0, s>>>(
      m.data, m.keys, m.slot, m.nblocks, m.nb, m.G, reinterpret_cast<int*>(flag));
  SPAMM_LAUNCH_CK();
  int64_t h = 0;
  d2h_sync(&h, flag, 1, s);
  dfree(flag, s);
  return h == 0;
}

void from_dense(const double* dense, int64_t n, int64_t ld, Mat& m, cudaStream_t s) {
  const int64_t G = int64_t(1) << m.depth, npos = G * G;
  uint8_t* flags = dmalloc<uint8_t>(npos, s);
  int64_t* off = dmalloc<int64_t>(npos + 1, s);
  k_dense_block_flags<<<warp_grid(npos), 32 * WARPS_PER_CTA, 0, s>>>(dense, n, ld, m.nb, m.depth, flags);
  SPAMM_LAUNCH_CK();
  scan_exclusive_u8(flags, npos, off, s);
  int64_t S = 0;
  d2h_sync(&S, off + npos, 1, s);
  m.nblocks = S;
  m.data = dmalloc<double>((size_t)S * m.nb * m.nb, s);
  m.keys = dmalloc<int64_t>(S, s);
  if (S > 0) {
    k_dense_block_copy<<<warp_grid(npos), 32 * WARPS_PER_CTA, 0, s>>>(dense, n, ld, m.nb, m.depth,
                                                                       flags, off, m.data, m.keys);
    SPAMM_LAUNCH_CK();
  }
  dfree(flags, s);
  dfree(off, s);
  finalize(m, s);
  m.sym = is_symmetric(m, s);
}

void to_dense(const Mat& m, double* dense, int64_t ld, cudaStream_t s) {
  SPAMM_CK(cudaMemsetAsync(dense, 0, (size_t)m.n_native * ld * sizeof(double), s));
  if (m.nblocks > 0) {
    k_block_store_dense<<<grid_for(m.nblocks, 1, 148LL * 32), 256, 0, s>>>(
        m.data, m.keys, m.nblocks, m.nb, m.G, m.n_native, ld, dense);
    SPAMM_LAUNCH_CK();
  }
}

void identity(Mat& m, cudaStream_t s) {
  const int64_t G = int64_t(1) << m.depth;
  const int64_t n_diag = (m.n_native + m.nb - 1) / m.nb;
  m.nblocks = n_diag;
  m.data = dmalloc<double>((size_t)n_diag * m.nb * m.nb, s);
  m.keys = dmalloc<int64_t>(n_diag, s);
  SPAMM_CK(cudaMemsetAsync(m.data, 0, (size_t)n_diag * m.nb * m.nb * sizeof(double), s));
  k_identity<<<grid_for(n_diag, 128), 128, 0, s>>>(m.n_native, m.nb, G, n_diag, m.data, m.keys);
  SPAMM_LAUNCH_CK();
  finalize(m, s);
  m.sym = true;
}

void add_scaled(double alpha, const Mat& a, double beta, const Mat& b, Mat& out, cudaStream_t s) {
  const int64_t G = int64_t(1) << a.depth, npos = G * G;
  uint8_t* flags = dmalloc<uint8_t>(npos, s);
  int64_t* off = dmalloc<int64_t>(npos + 1, s);
  k_union_flags<<<grid_for(npos, 256), 256, 0, s>>>(a.slot, b.slot, a.depth, flags);
  SPAMM_LAUNCH_CK();
  scan_exclusive_u8(flags, npos, off, s);
  int64_t U = 0;
  d2h_sync(&U, off + npos, 1, s);
  out.n_native = a.n_native;
  out.nb = a.nb;
  out.chunk_size = a.chunk_size;
  out.depth = a.depth;
  out.nblocks = U;
  out.data = dmalloc<double>((size_t)U * a.nb * a.nb, s);
  out.keys = dmalloc<int64_t>(U, s);
  if (U > 0) {
    k_add_scaled<<<grid_for(npos, 1, 148LL * 32), 256, 0, s>>>(alpha, a.data, a.slot, beta, b.data,
                                                                b.slot, a.depth, a.nb, flags, off,
                                                                out.data, out.keys);
    SPAMM_LAUNCH_CK();
  }
  dfree(flags, s);
  dfree(off, s);
  finalize(out, s);
  out.sym = a.sym && b.sym;
}

void trace_launch(const Mat& m, double* dev_out, cudaStream_t s) {
  if (m.tr_dev) {  // computed by the single-CTA finalisation
    SPAMM_CK(cudaMemcpyAsync(dev_out, m.tr_dev, sizeof(double), cudaMemcpyDeviceToDevice, s));
    return;
  }
  double* partial = dmalloc<double>(m.G, s);
  uint8_t* present = dmalloc<uint8_t>(m.G, s);
  k_trace_blocks<<<grid_for(m.G * 32, 256), 256, 0, s>>>(m.slot, m.data, m.G, m.nb, partial,
                                                          present);
  SPAMM_LAUNCH_CK();
  k_trace<<<1, 32, 0, s>>>(m.slot, m.data, m.G, m.nb, partial, present, dev_out);
  SPAMM_LAUNCH_CK();
  dfree(partial, s);
  dfree(present, s);
}

void diag_traces(const Mat& m, double* out, cudaStream_t s) {
  SPAMM_CK(cudaMemsetAsync(out, 0, m.G * sizeof(double), s));  // absent blocks: +0.0
  uint8_t* present = dmalloc<uint8_t>(m.G, s);
  k_trace_blocks<<<grid_for(m.G * 32, 256), 256, 0, s>>>(m.slot, m.data, m.G, m.nb, out, present);
  SPAMM_LAUNCH_CK();
  dfree(present, s);
}

double trace(const Mat& m, cudaStream_t s) {
  if (m.tr_valid) return m.tr;
  int64_t* buf = dmalloc<int64_t>(1, s);
  trace_launch(m, reinterpret_cast<double*>(buf), s);
  int64_t bits = 0;
  d2h_sync(&bits, buf, 1, s);
  dfree(buf, s);
  double v;
  memcpy(&v, &bits, sizeof(v));
  m.tr = v;
  m.tr_valid = true;
  return v;
}

void pairwise_schedule(int64_t n, std::vector<int64_t>& leaf_lo, std::vector<int32_t>& leaf_len,
                       std::vector<int32_t>& ops) {
  struct Sched {
    std::vector<int64_t>& lo;
    std::vector<int32_t>& len;
    std::vector<int32_t>& ops;
    void build(int64_t a, int64_t m) {
      if (m <= 128) {
        ops.push_back((int32_t)lo.size());
        lo.push_back(a);
        len.push_back((int32_t)m);
        return;
      }
      int64_t m2 = m / 2;
      m2 -= m2 % 8;
      build(a, m2);
      build(a + m2, m - m2);
      ops.push_back(-1);
    }
  } sched{leaf_lo, leaf_len, ops};
  sched.build(0, n);
}

void minmax_launch(const double* lo, const double* hi, int64_t n, double* out, cudaStream_t s) {
  k_minmax<<<1, 1024, 0, s>>>(lo, hi, n, out);
  SPAMM_LAUNCH_CK();
}

void gershgorin(const Mat& f, double* eps_min, double* eps_max, double* asym, cudaStream_t s) {
  const int64_t n = f.n_native;
  double* buf = dmalloc<double>(2 * n + 3, s);
  double* lo = buf;
  double* hi = buf + n;
  double* res = buf + 2 * n;
  SPAMM_CK(cudaMemsetAsync(res + 2, 0, sizeof(double), s));
  if (f.nblocks > 0) {
    k_asym<<<grid_for(f.nblocks, 1, 148LL * 16), 256, 0, s>>>(
        f.data, f.keys, f.slot, f.nblocks, f.nb, f.G, n,
        reinterpret_cast<unsigned long long*>(res + 2));
    SPAMM_LAUNCH_CK();
  }
  // numpy pairwise_sum tree for a row of length n, flattened (same for all rows)
  std::vector<int64_t> leaf_lo;
  std::vector<int32_t> leaf_len, ops;
  pairwise_schedule(n, leaf_lo, leaf_len, ops);
  const int nl = (int)leaf_lo.size(), no = (int)ops.size();
  const size_t smem = 8 * (size_t)nl * sizeof(double);
  if (smem <= 200 * 1024) {
    int64_t* d_lo = dmalloc<int64_t>(nl, s);
    int32_t* d_len = dmalloc<int32_t>(nl, s);
    int32_t* d_ops = dmalloc<int32_t>(no, s);
    SPAMM_CK(cudaMemcpyAsync(d_lo, leaf_lo.data(), nl * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    SPAMM_CK(cudaMemcpyAsync(d_len, leaf_len.data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    SPAMM_CK(cudaMemcpyAsync(d_ops, ops.data(), no * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    if (smem > 48 * 1024)
      SPAMM_CK(cudaFuncSetAttribute(k_gersh_rows_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    k_gersh_rows_warp<<<grid_for(n * 32, 256, 148LL * 16), 256, smem, s>>>(
        f.data, f.slot, f.G, f.nb, n, d_lo, d_len, nl, d_ops, no, lo, hi);
    SPAMM_LAUNCH_CK();
    dfree(d_lo, s);
    dfree(d_len, s);
    dfree(d_ops, s);
  } else {
    k_gersh_rows<<<grid_for(n, 64), 64, 0, s>>>(f.data, f.slot, f.G, f.nb, n, lo, hi);
    SPAMM_LAUNCH_CK();
  }
  k_minmax<<<1, 1024, 0, s>>>(lo, hi, n, res);
  SPAMM_LAUNCH_CK();
  int64_t bits[3];
  d2h_sync(bits, reinterpret_cast<const int64_t*>(res), 3, s);
  dfree(buf, s);
  memcpy(eps_min, &bits[0], 8);
  memcpy(eps_max, &bits[1], 8);
  memcpy(asym, &bits[2], 8);
}

}  // namespace spamm
