// Multi-GPU shard plumbing for the distributed SP2 (dist.py):
// the halo plan of a rank's C segment, the block gather for other ranks, and
// the rank's operand (own blocks + fetched halo) with the whole matrix's
// pyramid.  The collectives themselves stay with the caller.
#include <algorithm>
#include <cstring>

#include "internal.h"

namespace spamm {

namespace {

// Operand keys the tasks of one cull read: A_ik, B_kj and, on the symmetric
// path, X_jk (the transposed block K4z takes B's digit slices from).
__global__ void k_need_flags(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                             const int64_t* __restrict__ seg, const int32_t* __restrict__ K,
                             int64_t n_c, int64_t G, int sym, uint8_t* __restrict__ need) {
  for (int64_t c = blockIdx.x; c < n_c; c += gridDim.x) {
    const int64_t i = ci[c], j = cj[c];
    for (int64_t t = seg[c] + threadIdx.x; t < seg[c + 1]; t += blockDim.x) {
      const int64_t k = K[t];
      need[i * G + k] = 1;
      need[k * G + j] = 1;
      if (sym) need[j * G + k] = 1;
    }
  }
}

__device__ __forceinline__ int owner_of(int64_t key, int64_t G, const int64_t* __restrict__ cuts,
                                        int world, int upper) {
  uint32_t i = (uint32_t)(key / G), j = (uint32_t)(key % G);
  if (upper && i > j) {
    const uint32_t t = i;
    i = j;
    j = t;
  }
  const int64_t pos = (int64_t)morton_encode(i, j);
  int o = 0;  // the segment [cuts[o], cuts[o+1]) holding pos
  while (o + 1 < world && pos >= cuts[o + 1]) ++o;
  return o;
}

// Remote needed keys: histogram per owner (pass 0), placement (pass 1).
template <bool PLACE>
__global__ void k_remote_keys(const uint8_t* __restrict__ need, int64_t G,
                              const int64_t* __restrict__ cuts, int world, int upper, int rank,
                              unsigned long long* __restrict__ cnt, int64_t* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < G * G;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!need[p]) continue;
    const int o = owner_of(p, G, cuts, world, upper);
    if (o == rank) continue;
    const unsigned long long q = atomicAdd(cnt + o, 1ull);
    if (PLACE) out[q] = p;  // cnt holds the group offsets in this pass
  }
}

__global__ void k_group_offsets(const unsigned long long* __restrict__ hist, int world,
                                unsigned long long* __restrict__ cursor,
                                int64_t* __restrict__ out_counts) {
  if (threadIdx.x != 0) return;
  unsigned long long a = 0;
  for (int o = 0; o < world; ++o) {
    cursor[o] = a;
    out_counts[o] = (int64_t)hist[o];
    a += hist[o];
  }
  out_counts[world] = (int64_t)a;
}

__global__ void k_gather_blocks(const double* __restrict__ data, const int32_t* __restrict__ slot,
                                const int64_t* __restrict__ keys, int64_t n, int nb2,
                                double* __restrict__ out, int* __restrict__ missing) {
  for (int64_t b = blockIdx.x; b < n; b += gridDim.x) {
    const int32_t sl = slot[keys[b]];
    if (sl < 0 && threadIdx.x == 0) atomicExch(missing, 1);
    const double2* src = reinterpret_cast<const double2*>(data + (int64_t)sl * nb2);
    double2* dst = reinterpret_cast<double2*>(out + b * nb2);
    for (int e = threadIdx.x; e < nb2 / 2; e += blockDim.x)
      dst[e] = sl >= 0 ? src[e] : make_double2(0.0, 0.0);
  }
}

__global__ void k_ext_flags(const int64_t* __restrict__ k0, int64_t n0,
                            const int64_t* __restrict__ k1, int64_t n1, int64_t G,
                            uint8_t* __restrict__ flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t key = i < n0 ? k0[i] : k1[i - n0];
    flags[morton_encode((uint32_t)(key / G), (uint32_t)(key % G))] = 1;
  }
}

// Scatter the blocks of both sources to their Morton-ordered storage slots.
__global__ void k_ext_scatter(const double* __restrict__ d0, const int64_t* __restrict__ k0,
                              int64_t n0, const double* __restrict__ d1,
                              const int64_t* __restrict__ k1, int64_t n1, int64_t G, int nb2,
                              const int64_t* __restrict__ off, double* __restrict__ data,
                              int64_t* __restrict__ keys, int32_t* __restrict__ slot) {
  for (int64_t b = blockIdx.x; b < n0 + n1; b += gridDim.x) {
    const bool first = b < n0;
    const int64_t key = first ? k0[b] : k1[b - n0];
    const int64_t d = off[morton_encode((uint32_t)(key / G), (uint32_t)(key % G))];
    const double2* src =
        reinterpret_cast<const double2*>(first ? d0 + b * nb2 : d1 + (b - n0) * nb2);
    double2* dst = reinterpret_cast<double2*>(data + d * nb2);
    for (int e = threadIdx.x; e < nb2 / 2; e += blockDim.x) dst[e] = src[e];
    if (threadIdx.x == 0) {
      keys[d] = key;
      slot[key] = (int32_t)d;
    }
  }
}

}  // namespace

void shard_plan(const Mat& x, double tau, int64_t lo, int64_t hi, bool sym_try, int rank,
                int world, const int64_t* cuts_host, bool upper, int64_t* out_keys,
                int64_t* counts_host, bool* sym_ok, int64_t* n_tasks, cudaStream_t s) {
  CullResult r;
  bool sym = sym_try;
  if (sym && !cull(x, x, tau, true, r, s, true, lo, hi)) sym = false;
  if (!sym) cull(x, x, tau, true, r, s, false, lo, hi);
  *sym_ok = sym;
  *n_tasks = r.n_tasks;
  const int64_t G = x.G, npos = G * G;
  uint8_t* need = dmalloc<uint8_t>(npos, s);
  SPAMM_CK(cudaMemsetAsync(need, 0, npos, s));
  if (r.n_tasks > 0 && r.n_c > 0) {
    k_need_flags<<<grid_for(r.n_c, 1, 148LL * 32), 128, 0, s>>>(r.ci, r.cj, r.seg, r.k, r.n_c, G,
                                                               sym ? 1 : 0, need);
    SPAMM_LAUNCH_CK();
  }
  r.release(s);
  // cuts to the device (one small copy), histogram, offsets, placement
  int64_t* cuts = dmalloc<int64_t>(world + 1, s);
  int64_t* stage = static_cast<int64_t*>(pinned_scratch((world + 1) * sizeof(int64_t)));
  std::memcpy(stage, cuts_host, (world + 1) * sizeof(int64_t));
  SPAMM_CK(cudaMemcpyAsync(cuts, stage, (world + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
  auto* hist = dmalloc<unsigned long long>(2 * world, s);
  int64_t* counts = dmalloc<int64_t>(world + 1, s);
  SPAMM_CK(cudaMemsetAsync(hist, 0, 2 * world * sizeof(unsigned long long), s));
  const int grid = grid_for(npos, 256);
  k_remote_keys<false><<<grid, 256, 0, s>>>(need, G, cuts, world, upper ? 1 : 0, rank, hist,
                                            nullptr);
  SPAMM_LAUNCH_CK();
  k_group_offsets<<<1, 32, 0, s>>>(hist, world, hist + world, counts);
  SPAMM_LAUNCH_CK();
  k_remote_keys<true><<<grid, 256, 0, s>>>(need, G, cuts, world, upper ? 1 : 0, rank,
                                           hist + world, out_keys);
  SPAMM_LAUNCH_CK();
  d2h_sync(counts_host, counts, world + 1, s);
  // (the pinned staging of the cuts is only reused after this sync)
  dfree(need, s);
  dfree(cuts, s);
  dfree(hist, s);
  dfree(counts, s);
}

void gather_blocks(const Mat& x, const int64_t* keys, int64_t n, double* out, cudaStream_t s) {
  if (n <= 0) return;
  int* missing = dmalloc<int>(1, s);
  SPAMM_CK(cudaMemsetAsync(missing, 0, sizeof(int), s));
  k_gather_blocks<<<grid_for(n, 1, 148LL * 32), 256, 0, s>>>(x.data, x.slot, keys, n,
                                                             x.nb * x.nb, out, missing);
  SPAMM_LAUNCH_CK();
  dfree(missing, s);  // (diagnostic flag; the caller's plan guarantees ownership)
}

void shard_extend(const Mat& x, const int64_t* keys, const double* blocks, int64_t n, Mat& e,
                  cudaStream_t s) {
  e.n_native = x.n_native;
  e.nb = x.nb;
  e.chunk_size = x.chunk_size;
  e.depth = x.depth;
  e.G = x.G;
  e.stream = s;
  const int64_t G = x.G, npos = G * G, nb2 = (int64_t)x.nb * x.nb;
  e.nblocks = x.nblocks + n;
  e.data = dmalloc<double>((size_t)e.nblocks * nb2, s);
  e.keys = dmalloc<int64_t>(e.nblocks, s);
  e.slot = dmalloc<int32_t>(npos, s);
  SPAMM_CK(cudaMemsetAsync(e.slot, 0xFF, npos * sizeof(int32_t), s));
  uint8_t* flags = dmalloc<uint8_t>(npos, s);
  int64_t* off = dmalloc<int64_t>(npos + 1, s);
  SPAMM_CK(cudaMemsetAsync(flags, 0, npos, s));
  if (e.nblocks > 0) {
    k_ext_flags<<<grid_for(e.nblocks, 256), 256, 0, s>>>(x.keys, x.nblocks, keys, n, G, flags);
    SPAMM_LAUNCH_CK();
  }
  scan_exclusive_u8(flags, npos, off, s);
  if (e.nblocks > 0) {
    k_ext_scatter<<<grid_for(e.nblocks, 1, 148LL * 32), 256, 0, s>>>(
        x.data, x.keys, x.nblocks, blocks, keys, n, G, (int)nb2, off, e.data, e.keys, e.slot);
    SPAMM_LAUNCH_CK();
  }
  dfree(flags, s);
  dfree(off, s);
  // the whole matrix's pyramid, symmetry flag and K4z scales come with x
  const int64_t ps = pyramid_size(x.depth);
  e.norms = dmalloc<double>(ps, s);
  e.norms2 = dmalloc<double>(ps, s);
  SPAMM_CK(cudaMemcpyAsync(e.norms, x.norms, ps * sizeof(double), cudaMemcpyDeviceToDevice, s));
  SPAMM_CK(cudaMemcpyAsync(e.norms2, x.norms2, ps * sizeof(double), cudaMemcpyDeviceToDevice, s));
  e.sym = x.sym;
  const size_t nex = (size_t)G * x.nb;
  if (x.oz_ex_row) {
    e.oz_ex_row = dmalloc<int>(nex, s);
    SPAMM_CK(cudaMemcpyAsync(e.oz_ex_row, x.oz_ex_row, nex * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  if (x.oz_ex_col) {
    e.oz_ex_col = dmalloc<int>(nex, s);
    SPAMM_CK(cudaMemcpyAsync(e.oz_ex_col, x.oz_ex_col, nex * sizeof(int), cudaMemcpyDeviceToDevice, s));
  }
  attach_host_top(e, s);
}

}  // namespace spamm
