// C ABI (include/spamm_b200.h): argument checks, handle management and the
// multiply driver (cull -> leaf products -> C finalisation).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/spamm_b200.h"
#include <vector>

#include "internal.h"

struct spamm_mat {
  spamm::Mat m;
};

namespace spamm {
std::atomic<long long> g_launch_count{0};
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SPAMM_API_BEGIN try {
#define SPAMM_API_END                                              \
  }                                                                \
  catch (const spamm::CudaError& e) {                              \
    return fail(SPAMM_ECUDA, e.what());                            \
  }                                                                \
  catch (const std::exception& e) {                                \
    return fail(SPAMM_ECUDA, e.what());                            \
  }                                                                \
  return SPAMM_OK;

inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

bool is_pow2(int64_t x) { return x >= 1 && (x & (x - 1)) == 0; }

int padded_depth(int64_t n, int64_t nb) {
  int d = 0;
  while ((nb << d) < n) ++d;
  return d;
}

int check_conformable(const spamm_mat* a, const spamm_mat* b) {
  if (!a || !b) return fail(SPAMM_EINVAL, "null matrix handle");
  if (a->m.n_native != b->m.n_native || a->m.depth != b->m.depth || a->m.nb != b->m.nb)
    return fail(SPAMM_EINVAL, "shape/blocking mismatch: (" + std::to_string(a->m.n_native) + ", " +
                                  std::to_string(a->m.nb << a->m.depth) + ", " +
                                  std::to_string(a->m.nb) + ") vs (" +
                                  std::to_string(b->m.n_native) + ", " +
                                  std::to_string(b->m.nb << b->m.depth) + ", " +
                                  std::to_string(b->m.nb) + ")");
  return SPAMM_OK;
}

// Timing events of one multiply (timed = 1).  Events come from a per-thread
// pool.  Inside the SP2 loop the readout is deferred (g_defer_timing): the
// elapsed times are read after the iteration's own host sync, when the
// events have completed -- a timed solve then has no extra sync per multiply.
thread_local std::vector<cudaEvent_t> g_event_pool;
thread_local bool g_defer_timing = false;
struct PendingTiming {
  cudaEvent_t e[4];
  spamm_stats* st;
};
thread_local std::vector<PendingTiming> g_pending_timing;
cudaEvent_t pooled_event() {
  if (g_event_pool.empty()) {
    cudaEvent_t e;
    SPAMM_CK(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = g_event_pool.back();
  g_event_pool.pop_back();
  return e;
}
void resolve_timings() {  // events complete: no wait
  for (auto& p : g_pending_timing) {
    float v[3] = {0.f, 0.f, 0.f};
    for (int i = 0; i < 3; ++i) SPAMM_CK(cudaEventElapsedTime(&v[i], p.e[i], p.e[i + 1]));
    p.st->ms_cull = v[0];
    p.st->ms_leaf = v[1];
    p.st->ms_finalize = v[2];
    for (auto x : p.e) g_event_pool.push_back(x);
  }
  g_pending_timing.clear();
}
struct EventTimer {
  cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
  bool on;
  cudaStream_t s;
  spamm_stats* defer_to = nullptr;
  EventTimer(bool on_, cudaStream_t s_) : on(on_), s(s_) {
    if (on)
      for (auto& x : e) x = pooled_event();
  }
  void mark(int i) {
    if (on) SPAMM_CK(cudaEventRecord(e[i], s));
  }
  float ms(int i, int j) {
    if (!on) return 0.f;
    float v = 0.f;
    SPAMM_CK(cudaEventSynchronize(e[j]));
    SPAMM_CK(cudaEventElapsedTime(&v, e[i], e[j]));
    return v;
  }
  ~EventTimer() {
    if (!on) return;
    if (defer_to) {
      g_pending_timing.push_back({{e[0], e[1], e[2], e[3]}, defer_to});
    } else {
      for (auto& x : e) g_event_pool.push_back(x);
    }
  }
};

__global__ void k_keys_from_nodes(const int32_t* ci, const int32_t* cj, int64_t n, int64_t G,
                                  int64_t* keys) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = (int64_t)ci[i] * G + cj[i];
}

__global__ void k_expand_tasks(const int32_t* ci, const int32_t* cj, const int64_t* seg,
                               const int32_t* k, int64_t n_c, int32_t* ti, int32_t* tk,
                               int32_t* tj) {
  for (int64_t c = blockIdx.x; c < n_c; c += gridDim.x)
    for (int64_t t = seg[c] + threadIdx.x; t < seg[c + 1]; t += blockDim.x) {
      ti[t] = ci[c];
      tj[t] = cj[c];
      tk[t] = k[t];
    }
}

__global__ void k_seg_flags(const int64_t* c_pos, int64_t n, uint8_t* flags) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    flags[t] = (t == 0 || c_pos[t] != c_pos[t - 1]) ? 1 : 0;
}

__global__ void k_seg_build(const int64_t* c_pos, const uint8_t* flags, const int64_t* off,
                            int64_t n, int64_t* seg, int64_t* c_out, int64_t nseg) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    if (flags[t]) {
      seg[off[t]] = t;
      c_out[off[t]] = c_pos[t];
    }
  if (blockIdx.x == 0 && threadIdx.x == 0) seg[nseg] = n;
}

bool g_sym_enabled = true;

__global__ void k_sym_flags(const int32_t* ci, const int32_t* cj, int64_t n, uint8_t* flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    flags[spamm::morton_encode(ci[i], cj[i])] = 1;
    flags[spamm::morton_encode(cj[i], ci[i])] = 1;
  }
}

__global__ void k_sym_layout(const int32_t* ci, const int32_t* cj, int64_t n, const int64_t* off,
                             int64_t* c_out, int64_t* c_mirror) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    c_out[i] = off[spamm::morton_encode(ci[i], cj[i])];
    c_mirror[i] = ci[i] != cj[i] ? off[spamm::morton_encode(cj[i], ci[i])] : -1;
  }
}

__global__ void k_flag_keys(const uint8_t* flags, const int64_t* off, int depth, int64_t* keys) {
  const int64_t G = int64_t(1) << depth, npos = G * G;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npos;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[p]) continue;
    uint32_t bi, bj;
    spamm::morton_decode((uint64_t)p, bi, bj);
    keys[off[p]] = (int64_t)bi * G + bj;
  }
}

int g_near_ulps_api = 64;  // mirrors spamm::set_near_tau_ulps for the stats

void fill_stats(spamm_stats* st, double tau, const spamm::CullResult& r, int nb) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  st->tau = tau;
  st->n_tiers = (int32_t)r.visited.size();
  for (size_t t = 0; t < r.visited.size() && t < SPAMM_MAX_TIERS; ++t) {
    st->visited[t] = r.visited[t];
    st->culled[t] = r.culled[t];
  }
  for (size_t t = 0; t < r.near.size() && t < SPAMM_MAX_TIERS; ++t) st->near_tau[t] = r.near[t];
  st->tau_margin = r.near.empty() ? INFINITY : r.margin;
  st->near_tau_ulps = g_near_ulps_api;
  st->leaf_products = r.visited.empty() ? 0 : r.visited.back();
  st->executed_products = r.sym ? r.n_tasks : st->leaf_products;
  st->symmetric = r.sym ? 1 : 0;
  st->flop_estimate = st->leaf_products * 2 * (int64_t)nb * nb * nb;
}

// Bulk copies riding the K4 windows of an SP2 solve (spamm_sp2_solve_ex).
struct SideQueue {
  const spamm_side_copies* cfg = nullptr;
  int item = 0;
  int64_t off = 0;
  cudaEvent_t ev = nullptr;
  bool pending() const { return cfg && item < cfg->n_items; }
  // issue up to `budget` bytes on the copy stream, ordered after `comp`'s
  // current position
  void issue(cudaStream_t comp, int64_t budget) {
    if (!pending()) return;
    auto cs = reinterpret_cast<cudaStream_t>(cfg->stream);
    if (!ev) SPAMM_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SPAMM_CK(cudaEventRecord(ev, comp));
    SPAMM_CK(cudaStreamWaitEvent(cs, ev, 0));
    while (budget > 0 && pending()) {
      const spamm_transfer& t = cfg->items[item];
      const int64_t take = std::min(budget, t.bytes - off);
      if (take > 0) {
        SPAMM_CK(cudaMemcpyAsync(static_cast<char*>(t.dst) + off,
                                 static_cast<const char*>(t.src) + off, (size_t)take,
                                 cudaMemcpyDefault, cs));
        off += take;
        budget -= take;
      }
      if (off >= t.bytes) {
        ++item;
        off = 0;
      }
    }
  }
  void window(cudaStream_t comp) {
    static const int64_t dflt = [] {  // SPAMM_SIDE_CHUNK_MB: default chunk of the riding copies
      const char* v = getenv("SPAMM_SIDE_CHUNK_MB");
      return (int64_t)(v && atoi(v) > 0 ? atoi(v) : 24) << 20;
    }();
    issue(comp, cfg && cfg->chunk_bytes > 0 ? cfg->chunk_bytes : dflt);
  }
  void drain(cudaStream_t comp) { issue(comp, INT64_MAX); }
  ~SideQueue() {
    if (ev) cudaEventDestroy(ev);
  }
};
thread_local SideQueue* g_side = nullptr;

struct OzakiAhead;
// Trace-first SP2 (sp2_solve_tf): the product is returned unfinalised (its
// slot map from the cull), and one extra device scalar rides on the cull's
// host sync.
struct MulOpts {
  bool defer_finalize = false;
  const int64_t* extra_src = nullptr;
  int64_t extra = 0;
};
void multiply_impl(const spamm_mat* a, const spamm_mat* b, double tau, int32_t kernel, bool timed,
                   cudaStream_t s, spamm::Mat& C, spamm_stats* stats, int64_t lo = 0,
                   int64_t hi = -1, int32_t* work = nullptr, bool defer_prune = false,
                   spamm::IdemFuse idem = {}, OzakiAhead* pre = nullptr, MulOpts* mo = nullptr);

}  // namespace

extern "C" {

int spamm_abi_version(void) { return SPAMM_ABI_VERSION; }
const char* spamm_last_error(void) { return g_err.c_str(); }
int64_t spamm_launch_count(void) { return spamm::g_launch_count.load(); }

int spamm_mat_from_dense(const double* dense, int64_t n, int64_t ld, int32_t block_size,
                         int64_t chunk_size, void* stream, spamm_mat** out) {
  if (!out) return fail(SPAMM_EINVAL, "null output handle");
  if (n < 1) return fail(SPAMM_EINVAL, "matrix must have at least one row");
  if (!is_pow2(block_size))
    return fail(SPAMM_EINVAL, "block size must be a power of two, got " + std::to_string(block_size));
  if (ld < n) return fail(SPAMM_EINVAL, "leading dimension smaller than n");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  h->m.n_native = n;
  h->m.nb = block_size;
  h->m.depth = padded_depth(n, block_size);
  h->m.G = int64_t(1) << h->m.depth;
  h->m.chunk_size = chunk_size;
  h->m.stream = S(stream);
  try {
    spamm::from_dense(dense, n, ld, h->m, S(stream));
  } catch (...) {
    h->m.release();
    delete h;
    throw;
  }
  *out = h;
  SPAMM_API_END
}

int spamm_mat_from_blocks(int64_t n_native, int32_t block_size, int64_t chunk_size, int32_t depth,
                          const int64_t* keys, const double* data, int64_t m, void* stream,
                          spamm_mat** out) {
  if (!out) return fail(SPAMM_EINVAL, "null output handle");
  if (!is_pow2(block_size)) return fail(SPAMM_EINVAL, "block size must be a power of two");
  if (depth < 0 || depth > 24) return fail(SPAMM_EINVAL, "depth out of range");
  if (m < 0) return fail(SPAMM_EINVAL, "negative block count");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  auto* h = new spamm_mat();
  spamm::Mat& M = h->m;
  M.n_native = n_native;
  M.nb = block_size;
  M.chunk_size = chunk_size;
  M.depth = depth;
  M.G = int64_t(1) << depth;
  M.stream = s;
  // Re-order the given blocks along the Morton curve: 1.0 * blocks + (empty)
  // through add_scaled, which walks the curve and is exact for alpha = 1.
  spamm::Mat tmp;
  tmp.n_native = n_native;
  tmp.nb = block_size;
  tmp.chunk_size = chunk_size;
  tmp.depth = depth;
  tmp.G = M.G;
  tmp.stream = s;
  tmp.nblocks = m;
  tmp.data = const_cast<double*>(data);
  tmp.keys = const_cast<int64_t*>(keys);
  tmp.slot = spamm::dmalloc<int32_t>(M.G * M.G, s);
  SPAMM_CK(cudaMemsetAsync(tmp.slot, 0xFF, M.G * M.G * sizeof(int32_t), s));
  spamm::Mat empty;
  empty.depth = depth;
  empty.nb = block_size;
  empty.G = M.G;
  empty.slot = spamm::dmalloc<int32_t>(M.G * M.G, s);
  SPAMM_CK(cudaMemsetAsync(empty.slot, 0xFF, M.G * M.G * sizeof(int32_t), s));
  spamm::scatter_slots(keys, m, tmp.slot, s);
  spamm::add_scaled(1.0, tmp, 0.0, empty, M, s);
  spamm::dfree(tmp.slot, s);
  spamm::dfree(empty.slot, s);
  M.sym = spamm::is_symmetric(M, s);
  *out = h;
  SPAMM_API_END
}

int spamm_mat_cluster(const double* pos, const int64_t* orig, const double* diag, int64_t n,
                      int32_t block_size, int64_t chunk_size, double amp, double decay,
                      uint64_t seed, void* stream, spamm_mat** out) {
  if (!out || !pos || !orig || !diag) return fail(SPAMM_EINVAL, "null argument");
  if (n < 1) return fail(SPAMM_EINVAL, "matrix must have at least one row");
  if (!is_pow2(block_size)) return fail(SPAMM_EINVAL, "block size must be a power of two");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  h->m.n_native = n;
  h->m.nb = block_size;
  h->m.depth = padded_depth(n, block_size);
  h->m.G = int64_t(1) << h->m.depth;
  h->m.chunk_size = chunk_size;
  h->m.stream = S(stream);
  try {
    spamm::cluster_build(pos, orig, diag, amp, decay, seed, h->m, S(stream));
  } catch (...) {
    h->m.release();
    delete h;
    throw;
  }
  *out = h;
  SPAMM_API_END
}

int spamm_mat_cluster_range(const double* pos, const int64_t* orig, const double* diag,
                            int64_t n, int32_t block_size, int64_t chunk_size, double amp,
                            double decay, uint64_t seed, int64_t lo, int64_t hi, void* stream,
                            spamm_mat** out) {
  if (!out || !pos || !orig || !diag) return fail(SPAMM_EINVAL, "null argument");
  if (n < 1) return fail(SPAMM_EINVAL, "matrix must have at least one row");
  if (!is_pow2(block_size)) return fail(SPAMM_EINVAL, "block size must be a power of two");
  const int depth = padded_depth(n, block_size);
  const int64_t npos = (int64_t(1) << depth) * (int64_t(1) << depth);
  if (lo < 0 || hi < lo || hi > npos) return fail(SPAMM_EINVAL, "shard range outside [0, G*G]");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  h->m.n_native = n;
  h->m.nb = block_size;
  h->m.depth = depth;
  h->m.G = int64_t(1) << depth;
  h->m.chunk_size = chunk_size;
  h->m.stream = S(stream);
  try {
    spamm::cluster_build(pos, orig, diag, amp, decay, seed, h->m, S(stream), lo, hi);
  } catch (...) {
    h->m.release();
    delete h;
    throw;
  }
  *out = h;
  SPAMM_API_END
}

int spamm_cluster_gershgorin(const double* pos, const int64_t* orig, const double* diag, int64_t n,
                             double amp, double decay, uint64_t seed, int64_t row0, int64_t row1,
                             void* stream, double* eps_min, double* eps_max) {
  if (!pos || !orig || !diag || !eps_min || !eps_max) return fail(SPAMM_EINVAL, "null argument");
  if (n < 1 || row0 < 0 || row1 < row0 || row1 > n) return fail(SPAMM_EINVAL, "row range outside [0, n]");
  SPAMM_API_BEGIN
  spamm::cluster_gershgorin(pos, orig, diag, n, amp, decay, seed, row0, row1, eps_min, eps_max,
                            S(stream));
  SPAMM_API_END
}

int spamm_mat_leaf_norms2(const spamm_mat* m, double* out, void* stream) {
  if (!m || !out) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  const int64_t g = m->m.G;
  SPAMM_CK(cudaMemcpyAsync(out, m->m.norms2 + spamm::tier_offset(m->m.depth),
                           g * g * sizeof(double), cudaMemcpyDeviceToDevice, S(stream)));
  SPAMM_API_END
}

int spamm_mat_set_pyramid(spamm_mat* m, const double* leaf_norms2, int32_t symmetric,
                          void* stream) {
  if (!m || !leaf_norms2) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  spamm::settle_sync(m->m, S(stream));
  spamm::set_leaf_pyramid(m->m, leaf_norms2, S(stream));
  m->m.sym = symmetric != 0;
  SPAMM_API_END
}

int spamm_mat_oz_exponents(const spamm_mat* m, int32_t by_col, int32_t* ex, void* stream) {
  if (!m || !ex) return fail(SPAMM_EINVAL, "null argument");
  if (!spamm::ozaki_supported(m->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  SPAMM_API_BEGIN
  spamm::ozaki_exponents(m->m, by_col != 0, ex, S(stream));
  SPAMM_API_END
}

int spamm_mat_set_oz_exponents(spamm_mat* m, const int32_t* ex_row, const int32_t* ex_col,
                               void* stream) {
  if (!m) return fail(SPAMM_EINVAL, "null argument");
  if (!spamm::ozaki_supported(m->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  const size_t n = (size_t)m->m.G * m->m.nb;
  auto install = [&](int*& dst, const int32_t* src) {
    spamm::dfree(dst, s);
    dst = nullptr;
    if (!src) return;
    dst = spamm::dmalloc<int>(n, s);
    SPAMM_CK(cudaMemcpyAsync(dst, src, n * sizeof(int), cudaMemcpyDeviceToDevice, s));
  };
  install(m->m.oz_ex_row, ex_row);
  install(m->m.oz_ex_col, ex_col);
  SPAMM_API_END
}

int spamm_mat_identity(int64_t n, int32_t block_size, int64_t chunk_size, void* stream,
                       spamm_mat** out) {
  if (!out) return fail(SPAMM_EINVAL, "null output handle");
  if (n < 1) return fail(SPAMM_EINVAL, "identity needs n >= 1");
  if (!is_pow2(block_size)) return fail(SPAMM_EINVAL, "block size must be a power of two");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  h->m.n_native = n;
  h->m.nb = block_size;
  h->m.depth = padded_depth(n, block_size);
  h->m.G = int64_t(1) << h->m.depth;
  h->m.chunk_size = chunk_size;
  h->m.stream = S(stream);
  spamm::identity(h->m, S(stream));
  *out = h;
  SPAMM_API_END
}

int spamm_mat_info_peek(const spamm_mat* h, spamm_mat_info* info) {
  if (!h || !info) return fail(SPAMM_EINVAL, "null argument");
  info->n_native = h->m.n_native;
  info->block_size = h->m.nb;
  info->depth = h->m.depth;
  info->chunk_size = h->m.chunk_size;
  info->n_blocks = h->m.G;
  info->stored = -1;  // unknown until settled (lazy prune)
  info->data = nullptr;
  info->keys = nullptr;
  info->slot = nullptr;
  info->norms = h->m.norms;
  info->norms2 = h->m.norms2;
  info->symmetric = h->m.sym ? 1 : 0;
  return SPAMM_OK;
}

int spamm_mat_info_get(const spamm_mat* h, spamm_mat_info* info) {
  if (!h || !info) return fail(SPAMM_EINVAL, "null argument");
  if (h->m.pend_nz) {  // never expose a lazily pruned matrix
    try {
      spamm::settle_sync(const_cast<spamm_mat*>(h)->m, h->m.stream);
    } catch (const std::exception& e) {
      return fail(SPAMM_ECUDA, e.what());
    }
  }
  info->n_native = h->m.n_native;
  info->block_size = h->m.nb;
  info->depth = h->m.depth;
  info->chunk_size = h->m.chunk_size;
  info->n_blocks = h->m.G;
  info->stored = h->m.nblocks;
  info->data = h->m.data;
  info->keys = h->m.keys;
  info->slot = h->m.slot;
  info->norms = h->m.norms;
  info->norms2 = h->m.norms2;
  info->symmetric = h->m.sym ? 1 : 0;
  return SPAMM_OK;
}

int spamm_mat_free(spamm_mat* h) {
  if (!h) return SPAMM_OK;
  h->m.release();
  delete h;
  return SPAMM_OK;
}

int spamm_mat_to_dense(const spamm_mat* h, double* dense, int64_t ld, void* stream) {
  if (!h || !dense) return fail(SPAMM_EINVAL, "null argument");
  if (ld < h->m.n_native) return fail(SPAMM_EINVAL, "leading dimension smaller than n");
  SPAMM_API_BEGIN
  spamm::to_dense(h->m, dense, ld, S(stream));
  SPAMM_API_END
}

int spamm_multiply(const spamm_mat* a, const spamm_mat* b, double tau, int32_t kernel,
                   int32_t timed, void* stream, spamm_mat** c, spamm_stats* stats) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (kernel < 0 || kernel > 4) return fail(SPAMM_EINVAL, "unknown leaf kernel");
  if (kernel == SPAMM_LEAF_OZAKI && !spamm::ozaki_supported(a->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  if ((kernel == SPAMM_LEAF_DMMA || kernel == 3) && !spamm::dmma_supported(a->m.nb))
    return fail(SPAMM_EINVAL, "DMMA leaf kernel needs block size 8, 16, 32 or 64");
  if (!c) return fail(SPAMM_EINVAL, "null output handle");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  try {
    multiply_impl(a, b, tau, kernel, timed != 0, S(stream), h->m, stats);
  } catch (...) {
    h->m.release();
    delete h;
    throw;
  }
  *c = h;
  SPAMM_API_END
}

}  // extern "C"

namespace {

// AUTO's choice of K4z for block size nb (SPAMM_AUTO_LEAF=dmma: never).
bool auto_ozaki_for(int nb);
bool oz_ex_from_producers() {  // SPAMM_OZ_EXPROD=0: exponent passes as before
  static const bool on = [] {
    const char* v = getenv("SPAMM_OZ_EXPROD");
    return !(v && strcmp(v, "0") == 0);
  }();
  return on;
}
bool auto_ozaki_enabled() {  // SPAMM_AUTO_LEAF=dmma: AUTO keeps the DMMA kernel
  static const bool on = [] {
    const char* v = getenv("SPAMM_AUTO_LEAF");
    return !(v && strcmp(v, "dmma") == 0);
  }();
  return on;
}
bool auto_ozaki_for(int nb) {
  // Nb = 32: K4z is L2-bandwidth bound (16 KB of slices per 2 Nb^3 flops)
  // and only ~15 % faster than DMMA there (cfg3: 10.9 vs 12.5 ms per solve);
  // SPAMM_AUTO_OZ32=0 keeps DMMA at Nb = 32.
  static const bool oz32 = [] {
    const char* v = getenv("SPAMM_AUTO_OZ32");
    return !(v && strcmp(v, "0") == 0);
  }();
  return auto_ozaki_enabled() && (nb == 64 || (nb == 32 && oz32));
}

// K4 dispatch: the INT8-sliced kernel takes the operand matrices (row / column
// exponents from their keys), the others the block arrays.  AUTO picks it for
// Nb = 64 (faster than DMMA and closer to the exact product), DMMA otherwise.
// Returns true when K4z ran (then ex_out, if given, holds C's row exponents).
bool leaf_dispatch(int64_t n, const int64_t* seg, const int32_t* ai, const int32_t* bi,
                   const int64_t* c_out, const int64_t* c_mirror, const spamm_mat* a,
                   const spamm_mat* b, double* C, int32_t kernel, cudaStream_t s,
                   spamm::LptSchedule lpt, int* ex_out = nullptr) {
  const bool auto_ozaki = auto_ozaki_enabled();
  const bool sym_b = a == b && a->m.sym;
  if (kernel == spamm::LEAF_OZAKI) {
    spamm::leaf_products_ozaki<int32_t>(n, seg, ai, bi, c_out, c_mirror, false, a->m, b->m,
                                        sym_b, C, s, lpt, false, ex_out);
    return true;
  }
  // AUTO also needs room for the digit slices (the operands' size again): a
  // matrix that nearly fills HBM (config 5 on one GPU) stays on DMMA.
  if (kernel == spamm::LEAF_AUTO && auto_ozaki && auto_ozaki_for(a->m.nb) &&
      spamm::leaf_products_ozaki<int32_t>(n, seg, ai, bi, c_out, c_mirror, false, a->m, b->m,
                                          sym_b, C, s, lpt, /*try_only=*/true, ex_out))
    return true;
  spamm::leaf_products<int32_t>(n, seg, ai, bi, c_out, c_mirror, false, a->m.data, a->m.nblocks,
                                  b->m.data, b->m.nblocks, C, a->m.nb, kernel, s, lpt);
  return false;
}

// K4z's operand pre-passes (row exponents, digit slices) depend only on the
// operands, so they run on a side stream while the cull and its host sync
// run on s; K4z then waits for them (one event each way).
struct OzakiAhead {
  spamm::OzakiOperands op;
  cudaEvent_t ready = nullptr;
  bool ok = false;
  cudaStream_t s = nullptr;
  ~OzakiAhead() {  // early-exit / error paths: give the scratch back after the pre-passes
    if (!ok) return;
    if (ready) cudaStreamWaitEvent(s, ready, 0);  // the frees below are ordered on s
    try {
      spamm::ozaki_release(op, s);
    } catch (...) {
    }
  }
};
size_t device_total_bytes() {
  static const size_t total = [] {
    size_t f = 0, t = 0;
    SPAMM_CK(cudaMemGetInfo(&f, &t));
    return t;
  }();
  return total;
}
cudaStream_t ozaki_side_stream() {  // one per (host thread, device)
  // Default priority: since round 2 the exponent pass comes from the
  // producers and the split is no longer the longer of the two chains before
  // K4z, so the latency-bound cull / finalisation kernels on the caller's
  // stream should not queue behind its CTAs (cfg4 solve, interleaved A/B:
  // 30.36 vs 30.71 ms with the side stream at the highest priority, the
  // round-1 setting; SPAMM_OZ_SIDE_PRIO=1 restores it).
  static const bool prio = [] {
    const char* v = getenv("SPAMM_OZ_SIDE_PRIO");
    return v && strcmp(v, "1") == 0;
  }();
  thread_local cudaStream_t side[64] = {};
  int dev = 0;
  SPAMM_CK(cudaGetDevice(&dev));
  cudaStream_t& t = side[dev & 63];
  if (!t) {
    int lo = 0, hi = 0;
    SPAMM_CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    SPAMM_CK(cudaStreamCreateWithPriority(&t, cudaStreamNonBlocking, prio ? hi : lo));
  }
  return t;
}
// two reusable events per (host thread, device): [0] orders the pre-passes
// after the operand's producer on the caller's stream, [1] marks them done
cudaEvent_t* ozaki_events() {
  thread_local cudaEvent_t evs[64][2] = {};
  int dev = 0;
  SPAMM_CK(cudaGetDevice(&dev));
  cudaEvent_t* ev = evs[dev & 63];
  for (int i = 0; i < 2; ++i)
    if (!ev[i]) SPAMM_CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  return ev;
}
// dep_recorded: ozaki_events()[0] was already recorded on s at the point the
// pre-passes must follow (the caller queued more work on s since).
void ozaki_ahead(const spamm_mat* a, const spamm_mat* b, int32_t kernel, cudaStream_t s,
                 OzakiAhead& oz, bool defer_tr = false, bool dep_recorded = false) {
  // AUTO prepares ahead only when the slices are small next to HBM (they are
  // allocated before C, whose size the cull has not told yet); larger
  // operands take the post-cull path (leaf_dispatch), which tries the
  // allocation after C's and falls back to DMMA (config 5 on one GPU).
  const size_t slices = (size_t)(a->m.nblocks + (a == b && a->m.sym ? 0 : b->m.nblocks)) *
                        a->m.nb * a->m.nb * 8;
  const bool want = kernel == spamm::LEAF_OZAKI ||
                    (kernel == spamm::LEAF_AUTO && auto_ozaki_enabled() &&
                     auto_ozaki_for(a->m.nb) && slices <= device_total_bytes() / 8);
  if (!want) return;
  oz.s = s;
  static const bool use_side = [] {
    const char* v = getenv("SPAMM_OZ_SIDE");
    return !(v && strcmp(v, "0") == 0);
  }();
  if (!use_side) {
    oz.ok = spamm::ozaki_prepare(a->m, b->m, a == b && a->m.sym, s, oz.op,
                                 /*try_only=*/kernel == spamm::LEAF_AUTO, defer_tr);
    return;  // (same stream: no event needed)
  }
  cudaStream_t side = ozaki_side_stream();
  // (a thread has one multiply in flight: each event is waited on before it
  // is recorded again)
  cudaEvent_t* ev = ozaki_events();
  if (!dep_recorded) SPAMM_CK(cudaEventRecord(ev[0], s));
  SPAMM_CK(cudaStreamWaitEvent(side, ev[0], 0));
  oz.ok = spamm::ozaki_prepare(a->m, b->m, a == b && a->m.sym, side, oz.op,
                               /*try_only=*/kernel == spamm::LEAF_AUTO, defer_tr);
  if (oz.ok) {
    oz.ready = ev[1];
    SPAMM_CK(cudaEventRecord(oz.ready, side));
  }
}

void multiply_impl(const spamm_mat* a, const spamm_mat* b, double tau, int32_t kernel, bool timed,
                   cudaStream_t s, spamm::Mat& C, spamm_stats* stats, int64_t lo, int64_t hi,
                   int32_t* work, bool defer_prune, spamm::IdemFuse idem, OzakiAhead* pre,
                   MulOpts* mo) {
  EventTimer tm(timed, s);
  tm.mark(0);
  OzakiAhead oz;
  if (pre && pre->ok) {  // operand pre-passes already launched (SP2 speculation)
    oz.op = pre->op;
    oz.ready = pre->ready;
    oz.s = s;
    oz.ok = true;
    pre->ok = false;
    pre->ready = nullptr;
  }
  // The operand pre-passes (side stream) are queued right after the cull's
  // count pass, so the cull's CTAs are resident before the passes fill the
  // SMs (tier-walk culls: after the cull).
  struct Ahead {
    const spamm_mat *a, *b;
    int32_t kernel;
    cudaStream_t s;
    OzakiAhead* oz;
    bool done;
    static void run(void* p) {
      auto* h = static_cast<Ahead*>(p);
      if (h->done) return;
      h->done = true;
      ozaki_ahead(h->a, h->b, h->kernel, h->s, *h->oz, false, /*dep_recorded=*/true);
    }
  } ahead{a, b, kernel, s, &oz, oz.ok};
  if (!oz.ok) SPAMM_CK(cudaEventRecord(ozaki_events()[0], s));  // the operands are ready here
  spamm::CullResult r;
  // Symmetric SpAMM: X*X with X == X^T bitwise -> compute C_ij for i <= j only
  // and store C_ji = C_ij^T (bitwise what the full product yields).
  bool sym = g_sym_enabled && a == b && a->m.sym;
  const bool want_slot = mo && mo->defer_finalize;
  const int64_t* extra_src = mo ? mo->extra_src : nullptr;
  if (sym && !spamm::cull(a->m, b->m, tau, true, r, s, true, lo, hi, work, &Ahead::run, &ahead,
                          want_slot, extra_src))
    sym = false;  // ulp tie: full path
  if (!sym)
    spamm::cull(a->m, b->m, tau, true, r, s, false, lo, hi, work, &Ahead::run, &ahead, want_slot,
                extra_src);
  if (mo) mo->extra = r.extra;
  Ahead::run(&ahead);
  spamm::htrace("mul_culled");
  C.n_native = a->m.n_native;
  C.nb = a->m.nb;
  C.chunk_size = a->m.chunk_size;
  C.depth = a->m.depth;
  C.G = a->m.G;
  C.stream = s;
  const int64_t nb2 = (int64_t)C.nb * C.nb;
  int64_t* c_out = nullptr;
  int64_t* c_mirror = nullptr;
  if (r.keys) {  // dense cull: layout already built
    C.nblocks = r.n_c_full;
    C.keys = r.keys;
    r.keys = nullptr;
    c_out = r.c_out;  // (freed with r: they live in the cull's block)
    c_mirror = r.c_mirror;
  } else if (sym && r.n_c > 0) {
    const int64_t npos = C.G * C.G;
    uint8_t* flags = spamm::dmalloc<uint8_t>(npos, s);
    int64_t* off = spamm::dmalloc<int64_t>(npos + 1, s);
    SPAMM_CK(cudaMemsetAsync(flags, 0, npos, s));
    k_sym_flags<<<spamm::grid_for(r.n_c, 256), 256, 0, s>>>(r.ci, r.cj, r.n_c, flags);
    SPAMM_LAUNCH_CK();
    spamm::scan_exclusive_u8(flags, npos, off, s);
    C.nblocks = r.n_c_full;  // 2 * emitted - diagonal, counted by the cull (no sync)
    c_out = spamm::dmalloc<int64_t>(r.n_c, s);
    c_mirror = spamm::dmalloc<int64_t>(r.n_c, s);
    C.keys = spamm::dmalloc<int64_t>(C.nblocks, s);
    k_sym_layout<<<spamm::grid_for(r.n_c, 256), 256, 0, s>>>(r.ci, r.cj, r.n_c, off, c_out,
                                                             c_mirror);
    SPAMM_LAUNCH_CK();
    k_flag_keys<<<spamm::grid_for(npos, 256), 256, 0, s>>>(flags, off, C.depth, C.keys);
    SPAMM_LAUNCH_CK();
    spamm::dfree(flags, s);
    spamm::dfree(off, s);
  } else {
    C.nblocks = r.n_c;
    C.keys = spamm::dmalloc<int64_t>(r.n_c, s);
    if (r.n_c > 0) {
      k_keys_from_nodes<<<spamm::grid_for(r.n_c, 256), 256, 0, s>>>(r.ci, r.cj, r.n_c, C.G, C.keys);
      SPAMM_LAUNCH_CK();
    }
  }
  C.data = spamm::dmalloc<double>((size_t)C.nblocks * nb2, s);
  // SPAMM_OZ_EXOUT=1: a symmetric product on K4z also yields its own K4z row
  // exponents (the epilogue's row / mirror-column maxima), so a multiply on C
  // -- the next SP2 iteration after SQUARE -- skips its exponent pass.
  // Measured neutral on cfg4 (the pass saved, ~0.45 ms per solve, is paid
  // back by a slower epilogue: K4z 0.63 vs 0.65 of the INT8 peak), so off.
  int* ex_out = nullptr;
  const bool k4z_possible = kernel == spamm::LEAF_OZAKI ||
                            (kernel == spamm::LEAF_AUTO && auto_ozaki_enabled() &&
                             auto_ozaki_for(a->m.nb));
  static const bool exout = [] {
    const char* v = getenv("SPAMM_OZ_EXOUT");
    return v && strcmp(v, "1") == 0;
  }();
  if (exout && sym && r.n_c > 0 && k4z_possible && spamm::ozaki_supported(C.nb)) {
    ex_out = spamm::dmalloc<int>(C.G * C.nb, s);
    SPAMM_CK(cudaMemsetAsync(ex_out, 0x80, C.G * C.nb * sizeof(int), s));
  }
  // SP2 (idem fused): C's K4z exponents taken by the K1 pass over C (column
  // maxima = row maxima of the bitwise symmetric C), so the next multiply on
  // C -- after SQUARE -- skips its exponent pass.  SPAMM_OZ_EXPROD=0: off.
  int* ex_k1 = nullptr;
  if (!ex_out && oz_ex_from_producers() && idem.x && sym && k4z_possible &&
      spamm::ozaki_supported(C.nb) && spamm::idem_fusable(C)) {
    ex_k1 = spamm::dmalloc<int>(C.G * C.nb, s);
    SPAMM_CK(cudaMemsetAsync(ex_k1, 0x80, C.G * C.nb * sizeof(int), s));
    idem.ex_col = ex_k1;
  }
  bool ex_done = false;
  if (g_side) g_side->window(s);  // PCIe chunk alongside K4
  tm.mark(1);  // leaf window = the K4 launch only (allocation stays outside)
  if (oz.ok) {  // K4z on the operands prepared alongside the cull
    if (oz.ready) SPAMM_CK(cudaStreamWaitEvent(s, oz.ready, 0));
    oz.ready = nullptr;
    spamm::ozaki_finish_tr(a->m, oz.op, s);  // (operands prepared before a's slot map)
    if (r.n_c > 0) {
      spamm::LptSchedule lpt;
      lpt.order = r.order;
      lpt.counter = r.counter;
      spamm::ozaki_launch<int32_t>(r.n_c, r.seg, r.a_idx, r.b_idx, c_out, c_mirror, false,
                                   a->m, b->m, oz.op, C.data, s, lpt, ex_out);
      ex_done = ex_out != nullptr;
    }
    spamm::ozaki_release(oz.op, s);
    oz.ok = false;
  } else if (r.n_c > 0) {
    spamm::LptSchedule lpt;
    lpt.order = r.order;
    lpt.counter = r.counter;
    ex_done = leaf_dispatch(r.n_c, r.seg, r.a_idx, r.b_idx, c_out, c_mirror, a, b, C.data,
                            kernel, s, lpt, ex_out) && ex_out != nullptr;
  }
  if (ex_done) {
    C.oz_ex_row = ex_out;
  } else {
    spamm::dfree(ex_out, s);
  }
  tm.mark(2);
  spamm::htrace("mul_k4");
  if (!r.block) {
    spamm::dfree(c_out, s);
    spamm::dfree(c_mirror, s);
  }
  if (mo && mo->defer_finalize) {
    // (the caller finalises: the slot map from the cull stands in until then)
    C.slot = r.c_slot;
    r.c_slot = nullptr;
    if (!C.slot) {  // (not a dense cull: no slot map to hand over)
      throw spamm::CudaError("multiply: deferred finalisation needs the dense cull");
    }
  } else if (idem.x) {
    spamm::finalize(C, s, idem, defer_prune);
  } else {
    spamm::finalize(C, s, nullptr, nullptr, defer_prune);
  }
  if (ex_k1) C.oz_ex_row = ex_k1;
  C.sym = sym;
  spamm::htrace("mul_final");
  tm.mark(3);
  fill_stats(stats, tau, r, C.nb);
  if (stats) {
    stats->c_blocks = C.nblocks;
    stats->executed_products = r.n_tasks;
    stats->symmetric = sym ? 1 : 0;
    if (timed && g_defer_timing) {
      tm.defer_to = stats;  // read after the SP2 iteration's host sync
    } else {
      stats->ms_cull = tm.ms(0, 1);
      stats->ms_leaf = tm.ms(1, 2);
      stats->ms_finalize = tm.ms(2, 3);
    }
  }
  r.release(s);
}


// Multi-GPU shard scalars from the all-reduced vector [diag X (G) | diag X^2
// (G)]: tr X and tr X^2 as the sequential sums of the per-diagonal-block parts
// in block order (trace(), quadtree.py:305); out[2] (the residual norm) is
// the root of the D pyramid, written by the caller.
__global__ void k_shard_traces(const double* __restrict__ vec, int64_t G, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int64_t b = 0; b < G; ++b) a = __dadd_rn(a, vec[b]);
    out[0] = a;
  } else if (threadIdx.x == 32) {
    double a = 0.0;
    for (int64_t b = 0; b < G; ++b) a = __dadd_rn(a, vec[G + b]);
    out[1] = a;
  }
}


// Second half of an SP2 iteration given X and X2 = X*X (sp2.py:94-101 + the
// idempotency test): traces (tr X cached) and the union size in one sync, the
// branch rule, then the fused K6 pass.  *e receives 2X - X2 on EXPAND.
void sp2_finish(const spamm_mat* x, const spamm_mat* c, double n_occ, bool want_idem,
                cudaStream_t s, bool* square_out, double* t_x, double* t_sq, double* idem,
                spamm_mat** e_out, const double* idem_dev = nullptr,
                spamm::IdemFuse* fused_union = nullptr, double* branch_margin = nullptr,
                const double* given_dev = nullptr, int32_t kernel = 0,
                OzakiAhead* ahead = nullptr) {
  // given_dev (multi-GPU shard): device [tr X, tr X^2, ||X^2 - X||_F] of the
  // WHOLE matrices (all-reduced); x / c are then this rank's shards.
  const bool fused = spamm::sp2_fused_supported(x->m.nb);
  // One host sync (one gather launch) for tr(X), tr(X^2), the union size of
  // the update and X^2's kept-block count.  Traces computed by the small-tree
  // finalisation are read where they lie.
  int64_t* sc = spamm::dmalloc<int64_t>(3, s);
  const int64_t* src[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  auto trace_src = [&](const spamm::Mat& m, int64_t* scratch) -> const int64_t* {
    if (m.tr_dev) return reinterpret_cast<const int64_t*>(m.tr_dev);
    spamm::trace_launch(m, reinterpret_cast<double*>(scratch), s);
    return scratch;
  };
  if (given_dev) {
    src[0] = reinterpret_cast<const int64_t*>(given_dev);
    src[1] = reinterpret_cast<const int64_t*>(given_dev + 1);
  } else {
    if (!x->m.tr_valid) src[0] = trace_src(x->m, sc);
    src[1] = trace_src(c->m, sc + 1);
  }
  spamm::UnionPrep prep;
  if (fused && fused_union && fused_union->ukeys) {  // built by X^2's finalisation
    prep.npos = x->m.G * x->m.G;
    prep.keys = fused_union->ukeys;
    fused_union->ukeys = nullptr;  // ownership moves to the update
    src[2] = fused_union->ucount;
  } else if (fused) {
    prep = spamm::sp2_union_prepare(x->m, c->m, sc + 2, s);
    src[2] = sc + 2;
  }
  src[3] = spamm::pending_kept(c->m);  // lazy prune of X^2 rides along
  src[4] = reinterpret_cast<const int64_t*>(given_dev ? given_dev + 2 : idem_dev);
  const bool has_kept = src[3] != nullptr;
  int64_t h[5];
  spamm::gather_sync(h, src, 5, s);
  spamm::htrace("fin_synced");
  const bool idem_done = want_idem && (idem_dev || given_dev);
  if (idem_done) memcpy(idem, &h[4], sizeof(double));
  spamm::dfree(sc, s);
  if (has_kept) spamm::settle(const_cast<spamm_mat*>(c)->m, h[3], s);
  double tx, tsq;
  if (given_dev) {  // whole-matrix traces: not cached on the shards
    memcpy(&tx, &h[0], sizeof(double));
    memcpy(&tsq, &h[1], sizeof(double));
  } else {
    if (!x->m.tr_valid) {
      memcpy(&x->m.tr, &h[0], sizeof(double));
      x->m.tr_valid = true;
    }
    memcpy(&c->m.tr, &h[1], sizeof(double));
    c->m.tr_valid = true;
    tx = x->m.tr;
    tsq = c->m.tr;
  }
  // sp2.py:97-99: ties go to SQUARE.
  const double tex = 2.0 * tx - tsq;
  const bool square = std::fabs(tsq - n_occ) <= std::fabs(tex - n_occ);
  if (branch_margin) *branch_margin = std::fabs(tex - n_occ) - std::fabs(tsq - n_occ);
  spamm_mat* e = square ? nullptr : new spamm_mat();
  spamm::Mat dummy;
  spamm::htrace("fin_branch");
  if (fused) {
    // with the residual fused into K1 there is nothing left to sync on: E's
    // exact-zero blocks stay pending (settled when the handle is inspected)
    // -- so E's K4z operand passes can start on the side stream as soon as
    // the update is queued, ahead of E's finalisation and the next cull
    struct Hook {
      spamm_mat* e;
      int32_t kernel;
      cudaStream_t s;
      OzakiAhead* ahead;
      static void run(void* p) {
        auto* h = static_cast<Hook*>(p);
        ozaki_ahead(h->e, h->e, h->kernel, h->s, *h->ahead, /*defer_tr=*/true);
      }
    } hook{e, kernel, s, ahead};
    const bool early = e && ahead && idem_done;
    const bool k4z_next = kernel == spamm::LEAF_OZAKI ||
                          (kernel == spamm::LEAF_AUTO && auto_ozaki_enabled() &&
                           auto_ozaki_for(x->m.nb));
    spamm::sp2_update_finish(x->m, c->m, prep, h[2], want_idem && !idem_done, !square, idem,
                             e ? e->m : dummy, s, /*settle_now=*/!idem_done,
                             early ? &Hook::run : nullptr, &hook,
                             k4z_next && oz_ex_from_producers() &&
                                 spamm::ozaki_supported(x->m.nb));
  } else {
    spamm::sp2_update(x->m, c->m, want_idem && !idem_done, !square, idem, e ? e->m : dummy, s);
  }
  if (e) {
    e->m.stream = s;
    e->m.sym = x->m.sym && c->m.sym;
  }
  *square_out = square;
  *t_x = tx;
  *t_sq = tsq;
  *e_out = e;
  spamm::htrace("fin_end");
}

}  // namespace

extern "C" {

int spamm_sp2_step(const spamm_mat* x, double n_occ, double tau, int32_t kernel, int32_t want_idem,
                   int32_t timed, void* stream, spamm_mat** x_next, int32_t* branch, double* t_x,
                   double* t_sq, double* idem, spamm_stats* stats) {
  if (!x || !x_next || !branch || !t_x || !t_sq || (want_idem && !idem))
    return fail(SPAMM_EINVAL, "null argument");
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (kernel < 0 || kernel > 4) return fail(SPAMM_EINVAL, "unknown leaf kernel");
  if (kernel == SPAMM_LEAF_OZAKI && !spamm::ozaki_supported(x->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  if ((kernel == SPAMM_LEAF_DMMA || kernel == 3) && !spamm::dmma_supported(x->m.nb))
    return fail(SPAMM_EINVAL, "DMMA leaf kernel needs block size 8, 16, 32 or 64");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  auto* c = new spamm_mat();
  spamm::IdemFuse fuse;
  if (want_idem && spamm::idem_fusable(x->m)) {
    fuse.x = &x->m;
    fuse.out = spamm::dmalloc<double>(2, s);
    fuse.ucount = reinterpret_cast<int64_t*>(fuse.out + 1);
    fuse.ukeys = spamm::dmalloc<int64_t>(x->m.G * x->m.G, s);
  }
  multiply_impl(x, x, tau, kernel, timed != 0, s, c->m, stats, 0, -1, nullptr, true, fuse);
  spamm_mat* e = nullptr;
  bool square = true;
  double tx = 0, tsq = 0;
  sp2_finish(x, c, n_occ, want_idem != 0, s, &square, &tx, &tsq, idem, &e, fuse.out, &fuse);
  spamm::dfree(fuse.out, s);
  spamm::dfree(fuse.ukeys, s);
  if (e) {
    c->m.release();
    delete c;
    *x_next = e;
  } else {
    *x_next = c;
  }
  *branch = square ? 0 : 1;
  *t_x = tx;
  *t_sq = tsq;
  SPAMM_API_END
}

int spamm_shard_sp2_step(const spamm_mat* ext, const spamm_mat* x, double n_occ, double tau,
                         int32_t kernel, int64_t lo, int64_t hi, int32_t* work,
                         int32_t want_idem, spamm_allreduce_fn allreduce, void* ctx,
                         void* stream, spamm_mat** x_next, int32_t* branch, double* t_x,
                         double* t_sq, double* idem, spamm_stats* stats) {
  if (int rc = check_conformable(ext, x)) return rc;
  if (!x_next || !branch || !t_x || !t_sq || (want_idem && !idem))
    return fail(SPAMM_EINVAL, "null argument");
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (kernel < 0 || kernel > 4) return fail(SPAMM_EINVAL, "unknown leaf kernel");
  if (kernel == SPAMM_LEAF_OZAKI && !spamm::ozaki_supported(x->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  if (hi >= 0 && (lo < 0 || hi < lo || hi > x->m.G * x->m.G))
    return fail(SPAMM_EINVAL, "shard range outside [0, G*G]");
  if (allreduce && x->m.nb < 2) return fail(SPAMM_EINVAL, "sharded SP2 needs block size >= 2");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  const int64_t G = x->m.G;
  auto* c = new spamm_mat();
  spamm::IdemFuse fuse;
  double* vec = nullptr;  // [diag X | diag X^2 | leaf ||X^2 - X||^2] (+ 3 scalars)
  if (allreduce) vec = spamm::dmalloc<double>(2 * G + G * G + 3, s);
  if (want_idem && spamm::idem_fusable(x->m)) {
    fuse.x = &x->m;
    fuse.out = spamm::dmalloc<double>(2, s);
    fuse.ucount = reinterpret_cast<int64_t*>(fuse.out + 1);
    fuse.ukeys = spamm::dmalloc<int64_t>(G * G, s);
    if (vec) fuse.dleaf = vec + 2 * G;
  }
  try {
    multiply_impl(ext, ext, tau, kernel, false, s, c->m, stats, hi >= 0 ? lo : 0, hi, work,
                  true, fuse);
  } catch (...) {
    c->m.release();
    delete c;
    throw;
  }
  const double* given = nullptr;
  if (vec) {
    // this rank's parts, one all-reduce, then the whole matrices' scalars
    spamm::diag_traces(x->m, vec, s);
    spamm::diag_traces(c->m, vec + G, s);
    if (want_idem && !fuse.dleaf) {  // unfused residual: materialise the shard's D
      spamm::Mat d;
      spamm::add_scaled(1.0, c->m, -1.0, x->m, d, s);
      SPAMM_CK(cudaMemcpyAsync(vec + 2 * G, d.norms2 + spamm::tier_offset(d.depth),
                               G * G * sizeof(double), cudaMemcpyDeviceToDevice, s));
      d.release();
    } else if (!want_idem) {
      SPAMM_CK(cudaMemsetAsync(vec + 2 * G, 0, G * G * sizeof(double), s));
    }
    const int arc = allreduce(ctx, vec, 2 * G + G * G, stream);
    if (arc != 0) throw std::runtime_error("sharded SP2: all-reduce callback failed");
    double* out = vec + 2 * G + G * G;
    k_shard_traces<<<1, 64, 0, s>>>(vec, G, out);
    SPAMM_LAUNCH_CK();
    if (want_idem) {  // the D pyramid's root, in the tier order of any other matrix
      spamm::Mat d;
      d.depth = x->m.depth;
      d.G = G;
      const int64_t ps = spamm::pyramid_size(d.depth);
      d.norms = spamm::dmalloc<double>(ps, s);
      d.norms2 = spamm::dmalloc<double>(ps, s);
      spamm::set_leaf_pyramid(d, vec + 2 * G, s);
      SPAMM_CK(cudaMemcpyAsync(out + 2, d.norms, sizeof(double), cudaMemcpyDeviceToDevice, s));
      spamm::dfree(d.norms, s);
      spamm::dfree(d.norms2, s);
    }
    given = out;
  }
  spamm_mat* e = nullptr;
  bool square = true;
  double tx = 0, tsq = 0;
  sp2_finish(x, c, n_occ, want_idem != 0, s, &square, &tx, &tsq, idem, &e, fuse.out, &fuse,
             nullptr, given);
  spamm::dfree(fuse.out, s);
  spamm::dfree(fuse.ukeys, s);
  spamm::dfree(vec, s);
  if (e) {
    c->m.release();
    delete c;
    *x_next = e;
  } else {
    *x_next = c;
  }
  *branch = square ? 0 : 1;
  *t_x = tx;
  *t_sq = tsq;
  SPAMM_API_END
}

int spamm_sp2_finish(const spamm_mat* x, const spamm_mat* x2, double n_occ, int32_t want_idem,
                     void* stream, int32_t* branch, double* t_x, double* t_sq, double* idem,
                     spamm_mat** e_out) {
  if (int rc = check_conformable(x, x2)) return rc;
  if (!branch || !t_x || !t_sq || !e_out || (want_idem && !idem))
    return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  bool square = true;
  double tx = 0, tsq = 0;
  spamm_mat* e = nullptr;
  sp2_finish(x, x2, n_occ, want_idem != 0, S(stream), &square, &tx, &tsq, idem, &e);
  *e_out = e;
  *branch = square ? 0 : 1;
  *t_x = tx;
  *t_sq = tsq;
  SPAMM_API_END
}

int spamm_multiply_range(const spamm_mat* a, const spamm_mat* b, double tau, int32_t kernel,
                         int64_t lo, int64_t hi, int32_t* work, void* stream, spamm_mat** c,
                         spamm_stats* stats) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (kernel < 0 || kernel > 4) return fail(SPAMM_EINVAL, "unknown leaf kernel");
  if (kernel == SPAMM_LEAF_OZAKI && !spamm::ozaki_supported(a->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  if (lo < 0 || hi < lo || hi > a->m.G * a->m.G)
    return fail(SPAMM_EINVAL, "shard range outside [0, G*G]");
  if (!c) return fail(SPAMM_EINVAL, "null output handle");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  try {
    if (hi > lo) {
      multiply_impl(a, b, tau, kernel, false, S(stream), h->m, stats, lo, hi, work);
    } else {  // empty shard: an empty C
      h->m.n_native = a->m.n_native;
      h->m.nb = a->m.nb;
      h->m.chunk_size = a->m.chunk_size;
      h->m.depth = a->m.depth;
      h->m.G = a->m.G;
      spamm::finalize(h->m, S(stream));
      if (stats) std::memset(stats, 0, sizeof(*stats));
    }
  } catch (...) {
    h->m.release();
    delete h;
    throw;
  }
  *c = h;
  SPAMM_API_END
}

int spamm_shard_plan(const spamm_mat* x, double tau, int64_t lo, int64_t hi, int32_t sym_try,
                     int32_t rank, int32_t world, const int64_t* cuts, int32_t upper,
                     int64_t* out_keys, int64_t* counts, int32_t* sym_ok, int64_t* n_tasks,
                     void* stream) {
  if (!x || !cuts || !out_keys || !counts || !sym_ok || !n_tasks)
    return fail(SPAMM_EINVAL, "null argument");
  if (world < 1 || world > 16 || rank < 0 || rank >= world)
    return fail(SPAMM_EINVAL, "rank/world out of range (world <= 16)");
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (lo < 0 || hi < lo || hi > x->m.G * x->m.G)
    return fail(SPAMM_EINVAL, "shard range outside [0, G*G]");
  SPAMM_API_BEGIN
  bool ok = false;
  spamm::settle_sync(const_cast<spamm_mat*>(x)->m, S(stream));
  spamm::shard_plan(x->m, tau, lo, hi, sym_try != 0 && g_sym_enabled && x->m.sym, rank, world,
                    cuts, upper != 0, out_keys, counts, &ok, n_tasks, S(stream));
  *sym_ok = ok ? 1 : 0;
  SPAMM_API_END
}

int spamm_mat_gather_blocks(const spamm_mat* x, const int64_t* keys, int64_t n, double* out,
                            void* stream) {
  if (!x || (n > 0 && (!keys || !out))) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  spamm::settle_sync(const_cast<spamm_mat*>(x)->m, S(stream));
  spamm::gather_blocks(x->m, keys, n, out, S(stream));
  SPAMM_API_END
}

int spamm_shard_extend(const spamm_mat* x, const int64_t* keys, const double* blocks, int64_t n,
                       void* stream, spamm_mat** out) {
  if (!x || !out || (n > 0 && (!keys || !blocks))) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  spamm::settle_sync(const_cast<spamm_mat*>(x)->m, S(stream));
  auto* h = new spamm_mat();
  try {
    spamm::shard_extend(x->m, keys, blocks, n, h->m, S(stream));
  } catch (...) {
    h->m.release();
    delete h;
    throw;
  }
  *out = h;
  SPAMM_API_END
}

int spamm_reserve_pool(int64_t bytes, void* stream) {
  if (bytes < 0) return fail(SPAMM_EINVAL, "negative size");
  SPAMM_API_BEGIN
  spamm::ozaki_cache_trim();  // the kept K4z slice buffer goes back before the pool grows
  spamm::reserve_pool((size_t)bytes, S(stream));
  SPAMM_API_END
}

int spamm_set_symmetric_products(int32_t enabled) {
  g_sym_enabled = enabled != 0;
  return SPAMM_OK;
}

int spamm_set_dense_cull(int32_t enabled) {
  spamm::set_dense_cull(enabled != 0);
  return SPAMM_OK;
}

int spamm_set_near_tau_ulps(int32_t ulps) {
  if (ulps < 0) return fail(SPAMM_EINVAL, "near-tau band must be >= 0 ulps");
  spamm::set_near_tau_ulps(ulps);
  g_near_ulps_api = ulps;
  return SPAMM_OK;
}

int spamm_census(const spamm_mat* a, const spamm_mat* b, double tau, void* stream,
                 spamm_stats* stats) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  spamm::CullResult r;
  const bool sym = g_sym_enabled && a == b && a->m.sym;
  if (!sym || !spamm::cull(a->m, b->m, tau, false, r, s, true))
    spamm::cull(a->m, b->m, tau, false, r, s, false);
  fill_stats(stats, tau, r, a->m.nb);
  r.release(s);
  SPAMM_API_END
}

int spamm_census_range(const spamm_mat* a, const spamm_mat* b, double tau, int64_t lo,
                       int64_t hi, int32_t* work, void* stream, spamm_stats* stats) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (lo < 0 || hi < lo || hi > a->m.G * a->m.G)
    return fail(SPAMM_EINVAL, "shard range outside [0, G*G]");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  spamm::CullResult r;
  if (hi > lo) {
    const bool sym = g_sym_enabled && a == b && a->m.sym;
    if (!sym || !spamm::cull(a->m, b->m, tau, false, r, s, true, lo, hi, work))
      spamm::cull(a->m, b->m, tau, false, r, s, false, lo, hi, work);
  } else {
    r.visited.assign(a->m.depth + 1, 0);
    r.culled.assign(a->m.depth + 1, 0);
  }
  fill_stats(stats, tau, r, a->m.nb);
  r.release(s);
  SPAMM_API_END
}

int spamm_tasks_range(const spamm_mat* a, const spamm_mat* b, double tau, int64_t lo, int64_t hi,
                      int32_t* ti, int32_t* tk, int32_t* tj, int64_t cap, int64_t* n_out,
                      void* stream) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!(tau >= 0.0) || tau == __builtin_inf()) return fail(SPAMM_EINVAL, "tau must be finite and >= 0");
  if (!n_out) return fail(SPAMM_EINVAL, "null n_out");
  if (lo < 0 || hi < lo || hi > a->m.G * a->m.G)
    return fail(SPAMM_EINVAL, "shard range outside [0, G*G]");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  *n_out = 0;
  if (hi > lo) {
    // the tasks spamm_multiply_range executes: upper C blocks in range on the
    // symmetric path (mirrors come from the same accumulators), all otherwise
    spamm::CullResult r;
    const bool sym = g_sym_enabled && a == b && a->m.sym;
    if (!sym || !spamm::cull(a->m, b->m, tau, true, r, s, true, lo, hi))
      spamm::cull(a->m, b->m, tau, true, r, s, false, lo, hi);
    *n_out = r.n_tasks;
    if (r.n_tasks > 0 && r.n_tasks <= cap) {
      k_expand_tasks<<<spamm::grid_for(r.n_c, 1, 148LL * 32), 128, 0, s>>>(r.ci, r.cj, r.seg, r.k,
                                                                            r.n_c, ti, tk, tj);
      SPAMM_LAUNCH_CK();
    }
    r.release(s);
  }
  SPAMM_API_END
}

int spamm_tasks(const spamm_mat* a, const spamm_mat* b, double tau, int32_t* ti, int32_t* tk,
                int32_t* tj, int64_t cap, int64_t* n_out, void* stream) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!(tau >= 0.0) || tau == __builtin_inf()) return fail(SPAMM_EINVAL, "tau must be finite and >= 0");
  if (!n_out) return fail(SPAMM_EINVAL, "null n_out");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  spamm::CullResult r;
  spamm::cull(a->m, b->m, tau, true, r, s);
  *n_out = r.n_tasks;
  if (r.n_tasks > 0 && r.n_tasks <= cap) {
    k_expand_tasks<<<spamm::grid_for(r.n_c, 1, 148LL * 32), 128, 0, s>>>(r.ci, r.cj, r.seg, r.k,
                                                                          r.n_c, ti, tk, tj);
    SPAMM_LAUNCH_CK();
  }
  r.release(s);
  SPAMM_API_END
}

int spamm_gemm_batch(const int64_t* a_pos, const int64_t* b_pos, const int64_t* c_pos,
                     int64_t n_tasks, const double* a_data, int64_t a_blocks, const double* b_data,
                     int64_t b_blocks, double* c_data, int32_t block_size, int32_t kernel,
                     void* stream) {
  if (n_tasks < 0) return fail(SPAMM_EINVAL, "negative task count");
  if (block_size < 1) return fail(SPAMM_EINVAL, "block size must be >= 1");
  if (kernel < 0 || kernel > 3) return fail(SPAMM_EINVAL, "unknown leaf kernel");
  if ((kernel == SPAMM_LEAF_DMMA || kernel == 3) && !spamm::dmma_supported(block_size))
    return fail(SPAMM_EINVAL, "DMMA leaf kernel needs block size 8, 16, 32 or 64");
  if (n_tasks == 0) return SPAMM_OK;
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  uint8_t* flags = spamm::dmalloc<uint8_t>(n_tasks, s);
  int64_t* off = spamm::dmalloc<int64_t>(n_tasks + 1, s);
  k_seg_flags<<<spamm::grid_for(n_tasks, 256), 256, 0, s>>>(c_pos, n_tasks, flags);
  SPAMM_LAUNCH_CK();
  spamm::scan_exclusive_u8(flags, n_tasks, off, s);
  int64_t nseg = 0;
  spamm::d2h_sync(&nseg, off + n_tasks, 1, s);
  int64_t* seg = spamm::dmalloc<int64_t>(nseg + 1, s);
  int64_t* c_out = spamm::dmalloc<int64_t>(nseg, s);
  k_seg_build<<<spamm::grid_for(n_tasks, 256), 256, 0, s>>>(c_pos, flags, off, n_tasks, seg, c_out,
                                                             nseg);
  SPAMM_LAUNCH_CK();
  spamm::leaf_products<int64_t>(nseg, seg, a_pos, b_pos, c_out, nullptr, true, a_data, a_blocks,
                                b_data, b_blocks, c_data, block_size, kernel, s);
  spamm::dfree(flags, s);
  spamm::dfree(off, s);
  spamm::dfree(seg, s);
  spamm::dfree(c_out, s);
  SPAMM_API_END
}

int spamm_add_scaled(double alpha, const spamm_mat* a, double beta, const spamm_mat* b,
                     void* stream, spamm_mat** out) {
  if (int rc = check_conformable(a, b)) return rc;
  if (!out) return fail(SPAMM_EINVAL, "null output handle");
  SPAMM_API_BEGIN
  auto* h = new spamm_mat();
  h->m.stream = S(stream);
  spamm::add_scaled(alpha, a->m, beta, b->m, h->m, S(stream));
  h->m.G = a->m.G;
  *out = h;
  SPAMM_API_END
}

int spamm_trace(const spamm_mat* m, void* stream, double* out) {
  if (!m || !out) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  *out = spamm::trace(m->m, S(stream));
  SPAMM_API_END
}

int spamm_mat_diag_traces(const spamm_mat* m, double* out, void* stream) {
  if (!m || !out) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  spamm::settle_sync(const_cast<spamm_mat*>(m)->m, S(stream));
  spamm::diag_traces(m->m, out, S(stream));
  SPAMM_API_END
}

int spamm_sp2_update(const spamm_mat* x, const spamm_mat* x2, int32_t want_idem, int32_t expand,
                     void* stream, double* idem_norm, spamm_mat** e_out) {
  if (int rc = check_conformable(x, x2)) return rc;
  if (want_idem && !idem_norm) return fail(SPAMM_EINVAL, "null idem_norm");
  if (expand && !e_out) return fail(SPAMM_EINVAL, "null output handle");
  SPAMM_API_BEGIN
  cudaStream_t s = S(stream);
  spamm_mat* h = expand ? new spamm_mat() : nullptr;
  spamm::Mat dummy;
  spamm::sp2_update(x->m, x2->m, want_idem != 0, expand != 0, idem_norm, h ? h->m : dummy, s);
  if (h) {
    h->m.stream = s;
    h->m.sym = x->m.sym && x2->m.sym;
    *e_out = h;
  }
  SPAMM_API_END
}

int spamm_gershgorin(const spamm_mat* f, void* stream, double* eps_min, double* eps_max,
                     double* asym) {
  if (!f || !eps_min || !eps_max || !asym) return fail(SPAMM_EINVAL, "null argument");
  SPAMM_API_BEGIN
  spamm::gershgorin(f->m, eps_min, eps_max, asym, S(stream));
  SPAMM_API_END
}

int spamm_sp2_solve(const spamm_mat* f, double n_occ, double tau, int32_t max_iter,
                    double idem_tol, int32_t criterion, double fro_tol, double sym_tol,
                    int32_t kernel, int32_t timed, void* stream, spamm_mat** p_out,
                    spamm_sp2_report* rep) {
  return spamm_sp2_solve_ex(f, n_occ, tau, max_iter, idem_tol, criterion, fro_tol, sym_tol,
                            kernel, timed, stream, p_out, rep, nullptr);
}

int spamm_sp2_solve_ex(const spamm_mat* f, double n_occ, double tau, int32_t max_iter,
                       double idem_tol, int32_t criterion, double fro_tol, double sym_tol,
                       int32_t kernel, int32_t timed, void* stream, spamm_mat** p_out,
                       spamm_sp2_report* rep, const spamm_side_copies* side) {
  if (!f || !p_out || !rep) return fail(SPAMM_EINVAL, "null argument");
  if (side && (!side->stream || side->n_items < 0 || (side->n_items > 0 && !side->items)))
    return fail(SPAMM_EINVAL, "side copies: null stream or items");
  for (int i = 0; side && i < side->n_items; ++i)
    if (side->items[i].bytes < 0 || (side->items[i].bytes > 0 &&
                                     (!side->items[i].dst || !side->items[i].src)))
      return fail(SPAMM_EINVAL, "side copies: bad transfer " + std::to_string(i));
  if (!(n_occ > 0.0 && n_occ < (double)f->m.n_native))
    return fail(SPAMM_EINVAL, "n_occ must lie strictly between 0 and " +
                                  std::to_string(f->m.n_native));
  if (!(tau >= 0.0) || tau == __builtin_inf())
    return fail(SPAMM_EINVAL, "tau must be finite and >= 0, got " + std::to_string(tau));
  if (criterion != 0 && criterion != 1) return fail(SPAMM_EINVAL, "unknown criterion");
  if (kernel < 0 || kernel > 4) return fail(SPAMM_EINVAL, "unknown leaf kernel");
  if (kernel == SPAMM_LEAF_OZAKI && !spamm::ozaki_supported(f->m.nb))
    return fail(SPAMM_EINVAL, "INT8-sliced leaf kernel needs block size 32 or 64");
  if ((kernel == SPAMM_LEAF_DMMA || kernel == 3) && !spamm::dmma_supported(f->m.nb))
    return fail(SPAMM_EINVAL, "DMMA leaf kernel needs block size 8, 16, 32 or 64");
  if (max_iter < 0) return fail(SPAMM_EINVAL, "max_iter must be >= 0");
  cudaStream_t s = S(stream);
  // sp2.py:68-89: Gershgorin bounds, X0 = (eps_max I - F) / (eps_max - eps_min)
  double lo = 0, hi = 0, asym = 0;
  try {
    spamm::gershgorin(f->m, &lo, &hi, &asym, s);
  } catch (const std::exception& e) {
    return fail(SPAMM_ECUDA, e.what());
  }
  if (asym > sym_tol) {
    char buf[96];
    snprintf(buf, sizeof(buf), "matrix is not symmetric: max |F - F^T| = %.3e", asym);
    return fail(SPAMM_EINVAL, buf);
  }
  const double spread = hi - lo;
  if (spread <= 0) return fail(SPAMM_EINVAL, "degenerate spectral bounds: eps_max equals eps_min");
  rep->eps_min = lo;
  rep->eps_max = hi;
  rep->iterations = 0;
  rep->converged = 0;
  rep->n_multiplies = 0;
  SPAMM_API_BEGIN
  SideQueue sideq;
  sideq.cfg = side && side->n_items > 0 ? side : nullptr;
  struct SideScope {  // the hook lives for this solve only (also on throw)
    SideQueue* q;
    explicit SideScope(SideQueue* q_) : q(q_) { g_side = q_->cfg ? q_ : nullptr; }
    ~SideScope() { g_side = nullptr; }
  } side_scope(&sideq);
  const bool want_idem = criterion == 1;
  spamm::Mat eye;
  eye.n_native = f->m.n_native;
  eye.nb = f->m.nb;
  eye.depth = f->m.depth;
  eye.G = f->m.G;
  eye.chunk_size = f->m.chunk_size;
  spamm::identity(eye, s);
  auto* x = new spamm_mat();
  spamm::add_scaled(hi / spread, eye, -1.0 / spread, f->m, x->m, s);
  x->m.stream = s;
  eye.release();
  int n_tr = 0;
  rep->trace_history[n_tr++] = spamm::trace(x->m, s);
  bool pending_trace = false;
  double* idem_dev = spamm::dmalloc<double>(2, s);  // [residual | union size]
  struct IdemFree {
    double* p;
    cudaStream_t s;
    ~IdemFree() { spamm::dfree(p, s); }
  } idem_free{idem_dev, s};
  // Retired matrices are released after the next product is queued: their
  // (stream-ordered) frees then cost host time while K4 runs, not between
  // the branch decision and the next cull.
  struct Graveyard {
    std::vector<spamm_mat*> v;
    void flush() {
      for (auto* m : v) {
        m->m.release();
        delete m;
      }
      v.clear();
    }
    ~Graveyard() { flush(); }
  } dead;
  auto t_iter = std::chrono::steady_clock::now();
  // SPAMM_OZ_SPEC=1: after each X^2 the K4z operand pre-passes of X^2 start on
  // the side stream before the branch is known (SQUARE makes X^2 the next X);
  // on EXPAND, or when X^2's lazy prune compacts its storage, they are dropped.
  static const bool spec_on = [] {
    const char* v = getenv("SPAMM_OZ_SPEC");
    return v && strcmp(v, "1") == 0;
  }();
  OzakiAhead spec;
  const spamm_mat* spec_for = nullptr;
  // E = 2X - X^2 (EXPAND): its operand passes start right after the update
  // kernel, inside sp2_finish (the next multiply takes them)
  OzakiAhead ahead;
  const spamm_mat* ahead_for = nullptr;
  struct DeferScope {  // timed multiplies read their events after the branch sync
    DeferScope() { g_defer_timing = true; }
    ~DeferScope() {
      g_defer_timing = false;
      g_pending_timing.clear();
    }
  } defer_scope;
  auto drop_spec = [&]() {
    // on the pre-passes' own stream: ordered after them, and s never waits
    if (spec.ok) spamm::ozaki_release(spec.op, spec.ready ? ozaki_side_stream() : s);
    spec.ok = false;
    spec.ready = nullptr;
    spec_for = nullptr;
    if (ahead.ok) spamm::ozaki_release(ahead.op, ahead.ready ? ozaki_side_stream() : s);
    ahead.ok = false;
    ahead.ready = nullptr;
    ahead_for = nullptr;
  };
  // Trace-first SP2 (round 2): the branch needs only tr(X^2), so it is taken
  // right after the leaf products from the diagonal blocks, before any norm
  // pass -- SQUARE then runs K1 on X^2 (norms, the residual ||X^2 - X||,
  // the next K4z exponents), EXPAND runs the update alone (E, E's norms and
  // the residual in one pass over X and X^2) and skips K1 on the discarded
  // X^2.  The residual of step k is read at the next host sync (the cull of
  // step k + 1); if it converged there, step k + 1's product is dropped and
  // X_k is returned, exactly the reference loop's result (sp2.py:133-136).
  // SPAMM_SP2_TF=0 keeps the loop below.
  static const bool tf_on = [] {
    const char* v = getenv("SPAMM_SP2_TF");
    return !(v && strcmp(v, "0") == 0);
  }();
  const bool tf = tf_on && !spec_on && spamm::sp2_fused_supported(x->m.nb) &&
                  spamm::idem_fusable(x->m) && spamm::dense_cull_applies(x->m.depth);
  if (tf) {
    // dev: [0] residual of the pending step, [1] tr X^2, [2] tr X, [3] union size
    double* dev = spamm::dmalloc<double>(4, s);
    struct DevFree {
      double* p;
      cudaStream_t s;
      ~DevFree() { spamm::dfree(p, s); }
    } dev_free{dev, s};
    struct Pending {
      bool has = false;
      int k = 0;
      bool square = true;
      spamm_mat* prev_x = nullptr;  // X_k: the result if step k converged
    } P;
    const bool k4z_next = kernel == spamm::LEAF_OZAKI ||
                          (kernel == spamm::LEAF_AUTO && auto_ozaki_enabled() &&
                           auto_ozaki_for(x->m.nb));
    const bool want_ex = k4z_next && oz_ex_from_producers() && spamm::ozaki_supported(x->m.nb);
    auto accept_pending = [&]() {  // step P.k is not the last: X_{k+1} stands
      rep->branch_history[rep->iterations] = P.square ? 0 : 1;
      rep->iterations += 1;
      pending_trace = true;
      dead.v.push_back(P.prev_x);
      P.has = false;
      P.prev_x = nullptr;
    };
    auto converge_pending = [&]() {  // step P.k converged: X_k is the result
      rep->converged = 1;
      dead.v.push_back(x);
      x = P.prev_x;
      P.has = false;
      P.prev_x = nullptr;
    };
    for (int it = 0; it < max_iter; ++it) {
      auto* c = new spamm_mat();
      spamm_stats st;
      MulOpts mo;
      mo.defer_finalize = true;
      mo.extra_src = P.has ? reinterpret_cast<const int64_t*>(dev) : nullptr;
      spamm::htrace("it_mul");
      multiply_impl(x, x, tau, kernel, timed != 0, s, c->m, &st, 0, -1, nullptr, true,
                    spamm::IdemFuse{}, ahead.ok && ahead_for == x ? &ahead : nullptr, &mo);
      if (ahead.ok) drop_spec();  // (unused pre-passes)
      spamm::htrace("it_mul_done");
      if (P.has) {  // the residual of the previous step rode on this cull's sync
        double r;
        memcpy(&r, &mo.extra, sizeof(double));
        rep->idem_history[P.k] = r;
        if (r < fro_tol) {  // converged: this product is not part of the solve
          c->m.release();
          delete c;
          converge_pending();
          break;
        }
        accept_pending();
      }
      dead.flush();
      // pre-branch: tr X^2 from its diagonal blocks, the key union of X and
      // X^2 (the update's block set), tr X if not cached -- one host sync
      if (!x->m.tr_valid && !x->m.tr_dev) {  // (not expected: X0 / X^2 / E carry theirs)
        x->m.tr = spamm::trace(x->m, s);
        x->m.tr_valid = true;
      }
      int64_t h[3];
      spamm::UnionPrep prep = spamm::tf_prebranch(x->m, c->m, dev + 1,
                                                  reinterpret_cast<int64_t*>(dev + 3), h, s);
      spamm::htrace("fin_synced");
      if (!x->m.tr_valid) {
        memcpy(&x->m.tr, &h[1], sizeof(double));
        x->m.tr_valid = true;
      }
      double tsq;
      memcpy(&tsq, &h[0], sizeof(double));
      c->m.tr = tsq;
      c->m.tr_valid = true;
      const double tx = x->m.tr;
      const int64_t U = h[2];
      // sp2.py:97-99: ties go to SQUARE.
      const double tex = 2.0 * tx - tsq;
      const bool square = std::fabs(tsq - n_occ) <= std::fabs(tex - n_occ);
      const double bmargin = std::fabs(tex - n_occ) - std::fabs(tsq - n_occ);
      resolve_timings();  // (after the host sync: the events are complete)
      const int k = rep->n_multiplies++;
      rep->leaf_products[k] = st.leaf_products;
      rep->executed_products[k] = st.executed_products;
      if (rep->ms_leaf) rep->ms_leaf[k] = st.ms_leaf;
      if (rep->branch_margin) rep->branch_margin[k] = bmargin;
      if (rep->near_tau) {
        int64_t nt = 0;
        for (int t = 0; t < st.n_tiers; ++t) nt += st.near_tau[t];
        rep->near_tau[k] = nt;
      }
      if (rep->tau_margin) rep->tau_margin[k] = st.tau_margin;
      if (rep->wall_seconds) {
        const auto now = std::chrono::steady_clock::now();
        rep->wall_seconds[k] = std::chrono::duration<double>(now - t_iter).count();
        t_iter = now;
      }
      if (pending_trace) {  // tr of the last accepted X = this step's t_x
        rep->trace_history[n_tr++] = tx;
        pending_trace = false;
      }
      if (!want_idem &&
          std::fabs(tsq - tx) < idem_tol && std::fabs(tx - n_occ) < 1e-6 * n_occ) {
        rep->converged = 1;  // sp2.py:133-136: converged on X^2, the old X is returned
        spamm::dfree(prep.keys, s);
        spamm::dfree(prep.flags, s);
        spamm::dfree(prep.off, s);
        c->m.release();
        delete c;
        break;
      }
      spamm::htrace("fin_branch");
      spamm_mat* next = nullptr;
      if (square) {
        spamm::dfree(prep.keys, s);
        spamm::dfree(prep.flags, s);
        spamm::dfree(prep.off, s);
        spamm::IdemFuse f;
        f.x = &x->m;
        f.out = want_idem ? dev : nullptr;
        int* ex = nullptr;
        if (want_ex && want_idem && c->m.sym) {  // (taken by the fused K1 pass)
          ex = spamm::dmalloc<int>(c->m.G * c->m.nb, s);
          SPAMM_CK(cudaMemsetAsync(ex, 0x80, c->m.G * c->m.nb * sizeof(int), s));
          f.ex_col = ex;
        }
        const double keep_tr = c->m.tr;
        if (f.out)
          spamm::finalize(c->m, s, f, /*defer=*/true);
        else
          spamm::finalize(c->m, s, nullptr, nullptr, /*defer=*/true);
        c->m.tr = keep_tr;
        c->m.tr_valid = true;
        if (ex) c->m.oz_ex_row = ex;
        next = c;
      } else {
        auto* e = new spamm_mat();
        struct Hook {
          spamm_mat* e;
          int32_t kernel;
          cudaStream_t s;
          OzakiAhead* ahead;
          static void run(void* p) {
            auto* h = static_cast<Hook*>(p);
            ozaki_ahead(h->e, h->e, h->kernel, h->s, *h->ahead, /*defer_tr=*/true);
          }
        } hook{e, kernel, s, &ahead};
        double idem_unused = 0.0;
        spamm::sp2_update_finish(x->m, c->m, prep, U, want_idem, /*expand=*/true, &idem_unused,
                                 e->m, s, /*settle_now=*/false, &Hook::run, &hook, want_ex,
                                 want_idem ? dev : nullptr);
        e->m.stream = s;
        e->m.sym = x->m.sym && c->m.sym;
        if (ahead.ok) ahead_for = e;
        dead.v.push_back(c);  // (X^2 is read by the update only: freed stream-ordered)
        next = e;
      }
      spamm::htrace("fin_end");
      if (want_idem) {
        P.has = true;
        P.k = k;
        P.square = square;
        P.prev_x = x;
      } else {
        rep->branch_history[rep->iterations] = square ? 0 : 1;
        rep->iterations += 1;
        pending_trace = true;
        dead.v.push_back(x);
      }
      x = next;
    }
    if (P.has) {  // the last step's residual
      int64_t bits = 0;
      spamm::d2h_sync(&bits, reinterpret_cast<const int64_t*>(dev), 1, s);
      double r;
      memcpy(&r, &bits, sizeof(double));
      rep->idem_history[P.k] = r;
      if (r < fro_tol)
        converge_pending();
      else
        accept_pending();
    }
  } else
  for (int it = 0; it < max_iter; ++it) {
    auto* c = new spamm_mat();
    spamm_stats st;
    spamm::IdemFuse fuse;
    if (want_idem && spamm::idem_fusable(x->m)) {
      fuse.x = &x->m;
      fuse.out = idem_dev;
      fuse.ucount = reinterpret_cast<int64_t*>(idem_dev + 1);
      fuse.ukeys = spamm::dmalloc<int64_t>(x->m.G * x->m.G, s);
    }
    spamm::htrace("it_mul");
    multiply_impl(x, x, tau, kernel, timed != 0, s, c->m, &st, 0, -1, nullptr, true, fuse,
                  spec.ok && spec_for == x     ? &spec
                  : ahead.ok && ahead_for == x ? &ahead
                                               : nullptr);
    drop_spec();  // (unused speculation)
    spamm::htrace("it_mul_done");
    if (spec_on) {
      ozaki_ahead(c, c, kernel, s, spec);
      spec_for = spec.ok ? c : nullptr;
    }
    const int64_t c_blocks_before = c->m.nblocks;
    dead.flush();
    spamm::htrace("it_flushed");
    bool square = true;
    double tx = 0, tsq = 0, idem = 0;
    spamm_mat* e = nullptr;
    double bmargin = 0.0;
    sp2_finish(x, c, n_occ, want_idem, s, &square, &tx, &tsq, &idem, &e, fuse.out, &fuse,
               &bmargin, nullptr, kernel, spec_on ? nullptr : &ahead);
    if (spec.ok && (!square || c->m.nblocks != c_blocks_before)) drop_spec();
    if (ahead.ok) ahead_for = e;
    spamm::dfree(fuse.ukeys, s);  // (null once the update took it)
    resolve_timings();  // (after sp2_finish's host sync: the events are complete)
    const int k = rep->n_multiplies++;
    rep->leaf_products[k] = st.leaf_products;
    rep->executed_products[k] = st.executed_products;
    if (rep->ms_leaf) rep->ms_leaf[k] = st.ms_leaf;
    if (rep->branch_margin) rep->branch_margin[k] = bmargin;
    if (rep->near_tau) {
      int64_t nt = 0;
      for (int t = 0; t < st.n_tiers; ++t) nt += st.near_tau[t];
      rep->near_tau[k] = nt;
    }
    if (rep->tau_margin) rep->tau_margin[k] = st.tau_margin;
    if (rep->wall_seconds) {  // (the loop syncs on the host every iteration)
      const auto now = std::chrono::steady_clock::now();
      rep->wall_seconds[k] = std::chrono::duration<double>(now - t_iter).count();
      t_iter = now;
    }
    if (pending_trace) {  // tr of the last accepted X = this step's t_x
      rep->trace_history[n_tr++] = tx;
      pending_trace = false;
    }
    bool done;
    if (want_idem) {
      rep->idem_history[k] = idem;
      done = idem < fro_tol;
    } else {
      done = std::fabs(tsq - tx) < idem_tol && std::fabs(tx - n_occ) < 1e-6 * n_occ;
    }
    if (done) {  // sp2.py:133-136: converged on X^2, the old X is returned
      drop_spec();
      rep->converged = 1;
      if (e) {
        e->m.release();
        delete e;
      }
      c->m.release();
      delete c;
      break;
    }
    spamm_mat* next = c;
    if (e) {
      dead.v.push_back(c);
      next = e;
    }
    dead.v.push_back(x);
    x = next;
    rep->branch_history[rep->iterations] = square ? 0 : 1;
    rep->iterations += 1;
    pending_trace = true;
  }
  drop_spec();
  if (pending_trace) rep->trace_history[n_tr++] = spamm::trace(x->m, s);
  g_side = nullptr;
  sideq.drain(s);
  *p_out = x;
  spamm::htrace_dump();
  SPAMM_API_END
}

}  // extern "C"
