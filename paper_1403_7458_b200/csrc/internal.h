// Internal (non-exported) host interfaces shared by the library's translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace spamm {

// ---- stream-ordered device memory (cudaMallocAsync on the default pool) ----
void* dmalloc_bytes(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
void reserve_pool(size_t bytes, cudaStream_t s);
template <class T>
T* dmalloc(size_t n, cudaStream_t s) {
  return static_cast<T*>(dmalloc_bytes(n * sizeof(T), s));
}

// Copy a few int64 from device to host and wait (the only host syncs on the path).
void d2h_sync(int64_t* host, const int64_t* dev, int n, cudaStream_t s);
// One launch copies n (<= 64) device scalars (null source -> 0) straight into
// pinned host memory, then waits: replaces memset + D2D copies + D2H per sync.
void gather_sync(int64_t* host, const int64_t* const* src, int n, cudaStream_t s);
// The device side of gather_sync for kernels that publish their own scalars:
// a kernel writes vals[0..n) (pinned, device-visible), fences at system scope
// and stores seq to *flag; the host spins on the flag.
constexpr int GATHER_MAX = 64;
struct ScalarSrc {
  const int64_t* p[GATHER_MAX];
};
struct PinnedGather {
  int64_t* vals = nullptr;
  int64_t* flag = nullptr;
  int64_t seq = 0;
};
PinnedGather pinned_gather_begin();
void pinned_gather_wait(int64_t* host, int n, const PinnedGather& g, cudaStream_t s);
void copy_to_pinned(double* host, const double* dev, int64_t n, cudaStream_t s);
void stream_wait(cudaStream_t s);   // spin-polls unless SPAMM_WAIT=block
// Host-side timeline marks (SPAMM_HTRACE=1): label -> steady clock; htrace_dump
// prints the mean host time between consecutive labels (diagnostics only).
void htrace(const char* label);
void htrace_dump();
void event_wait(cudaEvent_t e);     // spin-polls

// ---- quadtree matrix (device resident) ----
struct Mat {
  int64_t n_native = 0;
  int nb = 0;
  int64_t chunk_size = 0;
  int depth = 0;
  int64_t G = 1;
  int64_t nblocks = 0;
  double* data = nullptr;    // nblocks * nb * nb, Morton order of (bi, bj)
  int64_t* keys = nullptr;   // nblocks, bi * G + bj
  int32_t* slot = nullptr;   // G * G, storage slot or -1
  double* norms = nullptr;   // pyramid_size(depth)
  double* norms2 = nullptr;  // pyramid_size(depth)
  bool sym = false;          // X == X^T bitwise (blocks and null structure)
  mutable double tr = 0.0;   // cached trace (matrices are immutable)
  mutable bool tr_valid = false;
  double* tr_dev = nullptr;  // trace written on the device by finalize (small trees)
  // Pinned host mirror of norm tiers 0..top_t (written by finalize, ready when
  // top_ev completes): the cull expands those tiers on the host.
  double* host_top = nullptr;
  int top_t = -1;
  cudaEvent_t top_ev = nullptr;
  // Lazy prune state (finalize(..., defer = true)); nullptr once settled.
  uint8_t* pend_nz = nullptr;
  int64_t* pend_off = nullptr;   // kept offsets (+ count at [nblocks]), or null if
  int64_t* pend_kept = nullptr;  // only the count was produced (small trees)
  // K4z row / column exponents installed from outside (multi-GPU: all-reduced
  // over the shards), G * nb each; nullptr: computed per multiply
  int* oz_ex_row = nullptr;
  int* oz_ex_col = nullptr;
  cudaStream_t stream = nullptr;
  void release();
};
constexpr int SMALL_TREE_DEPTH = 7;  // G*G <= 16384: single-CTA finalisation
constexpr int HOST_TOP_TIERS = 5;  // tiers 0..5: 1,365 norms (11 KB)

// Exact-symmetry test (block (i,j) == transpose of block (j,i), bitwise).
bool is_symmetric(const Mat& m, cudaStream_t s);

// Finalise a matrix whose data/keys (nblocks, Morton order) are set: prune
// exact-zero blocks, build slot map and the bit-exact norm pyramid
// (quadtree.py:170-194).  Takes ownership of data/keys, and of pre_n2 / pre_nz
// when given (per-block leaf norm^2 and nonzero flags already computed by a
// fused producer kernel; K1 is then skipped).
// defer = true: no host sync -- exact-zero blocks are kept until settle()
// (the kept count is then read with some later sync, see pending_kept()).
// Idempotency residual fused into the finalisation of C = X*X (small trees,
// Nb 32 / 64): the root norm of add_scaled(1, C, -1, X) (quadtree.py:281-293)
// is written to *out as the K1 pass reads C, so SP2 needs no separate D pass.
struct IdemFuse {
  const Mat* x = nullptr;
  double* out = nullptr;
  // optional: the key union of X and X^2 for the SP2 update (Morton order,
  // capacity G*G) and its size, produced by the same launch
  int64_t* ukeys = nullptr;
  int64_t* ucount = nullptr;
  // optional: the leaf tier (G * G, row-major) of ||X^2 - X||^2 (multi-GPU)
  double* dleaf = nullptr;
  // optional: C's K4z column exponents (G * nb, preset to OZ_EXP_NONE), taken
  // by the same pass -- the row exponents of a bitwise symmetric C
  int* ex_col = nullptr;
  // optional: the residual's leaf norm^2 per block of m (already computed by
  // the producer, caller-owned) -- with out, the D pyramid is built from it
  const double* pre_dn2 = nullptr;
};
bool idem_fusable(const Mat& x);
void finalize(Mat& m, cudaStream_t s, IdemFuse idem, bool defer);
// pre_n1 (optional): sqrt of pre_n2, computed by the producer.
void finalize(Mat& m, cudaStream_t s, double* pre_n2 = nullptr, uint8_t* pre_nz = nullptr,
              bool defer = false, double* pre_n1 = nullptr);
// Deferred finalisation of a producer-normed matrix (the SP2 update's E) that
// also reduces the residual's per-block leaf norm^2 (pre_dn2, one per block of
// m) to its root norm, written to *out (device) -- one launch.
void finalize_with_residual(Mat& m, cudaStream_t s, double* pre_n2, uint8_t* pre_nz,
                            double* pre_n1, const double* pre_dn2, double* out);
const int64_t* pending_kept(const Mat& m);  // device count, or nullptr if settled
void settle(Mat& m, int64_t kept, cudaStream_t s);
void settle_sync(Mat& m, cudaStream_t s);
// Fused SP2 update over the key union of X and X^2 (sp2.cu):
//   idem2_root <- pyramid root of ||X^2 - X||^2 (add_scaled(1,X2,-1,X).norm()^2)
//   expand     -> E = add_scaled(2, X, -1, X2) finalised into `e`.
void sp2_update(const Mat& x, const Mat& x2, bool want_idem, bool expand, double* idem_norm,
                Mat& e, cudaStream_t s);
// The same in two halves, so the union size U can ride on another host sync:
// prepare launches the key-union flags + scan (U lands in *u_dev, no sync);
// finish runs the fused pass given U.  Block sizes other than 32 / 64 are not
// supported by the split form (sp2_update handles them).
struct UnionPrep {
  uint8_t* flags = nullptr;
  int64_t* off = nullptr;
  int64_t npos = 0;
  int64_t* keys = nullptr;  // small trees: union keys already compacted (G*G capacity)
};
UnionPrep sp2_union_prepare(const Mat& x, const Mat& x2, int64_t* u_dev, cudaStream_t s);
// Trace-first SP2 (small trees): one launch + one host sync before the branch
// rule -- host3 = {tr X^2 bits, tr X bits (from x.tr_dev; 0 if x.tr_valid),
// union size}; returns the union keys (the update's block set).
UnionPrep tf_prebranch(const Mat& x, const Mat& c, double* ctr_dev, int64_t* u_dev,
                       int64_t* host3, cudaStream_t s);
// after_update (EXPAND, may be null): called once E's blocks are queued on s
// (the update kernel) and E's layout is set, before E's finalisation -- the
// SP2 loop starts E's K4z operand passes there.
void sp2_update_finish(const Mat& x, const Mat& x2, UnionPrep& prep, int64_t U, bool want_idem,
                       bool expand, double* idem_norm, Mat& e, cudaStream_t s,
                       bool settle_now = true, void (*after_update)(void*) = nullptr,
                       void* after_ctx = nullptr, bool want_oz_ex = false,
                       double* idem_dev_out = nullptr);
bool sp2_fused_supported(int nb);

void scatter_slots(const int64_t* keys, int64_t m, int32_t* slot, cudaStream_t s);
// (Re)write the pinned host mirror of m's top tiers from its device pyramid.
void attach_host_top(Mat& m, cudaStream_t s);
// A thread-local pinned staging buffer of >= bytes (small host->device copies).
void* pinned_scratch(size_t bytes);

// ---- multi-GPU shard plumbing (shard.cu) ----
// Halo plan of the C segment [lo, hi): cull x (the whole matrix's pyramid
// installed), list the operand blocks the tasks read that another rank owns
// (ownership: Morton position of (i,j) or, upper, of (min,max) under `cuts`),
// grouped by owner into out_keys (capacity G*G); counts_host[world + 1] gets
// the per-owner counts and the total.  *sym_ok: the symmetric path held on
// the range (sym_try).  One host sync besides the cull's.
void shard_plan(const Mat& x, double tau, int64_t lo, int64_t hi, bool sym_try, int rank,
                int world, const int64_t* cuts_host, bool upper, int64_t* out_keys,
                int64_t* counts_host, bool* sym_ok, int64_t* n_tasks, cudaStream_t s);
void gather_blocks(const Mat& x, const int64_t* keys, int64_t n, double* out, cudaStream_t s);
// e = x's blocks + n received (keys, blocks) in Morton order, with x's pyramid,
// symmetry flag and installed K4z exponents (the rank's operand).
void shard_extend(const Mat& x, const int64_t* keys, const double* blocks, int64_t n, Mat& e,
                  cudaStream_t s);
// Leaf norm^2 (einsum recipe) and nonzero flags for m blocks of nb x nb.
// norms1 (optional, Nb 32 / 64 only): sqrt of each leaf norm^2
void leaf_norms2(const double* data, int64_t m, int nb, double* norms2, uint8_t* nonzero,
                 cudaStream_t s, double* norms1 = nullptr);
// Fill the pyramid from per-block leaf norms^2 (keys given); zero elsewhere.
void build_pyramid(const int64_t* keys, const double* blk_norms2, int64_t m, int depth,
                   double* norms, double* norms2, cudaStream_t s);

// ---- scan ----
// out[0..n]: exclusive prefix sums, out[n] = total.
void scan_exclusive_u8(const uint8_t* in, int64_t n, int64_t* out, cudaStream_t s);
void scan_exclusive_i64(const int64_t* in, int64_t n, int64_t* out, cudaStream_t s);

// ---- culling ----
struct CullResult {
  int64_t n_c = 0;            // C blocks (leaf-tier nodes with >= 1 survivor)
  int64_t n_c_full = 0;       // C blocks including mirrors (symmetric mode)
  int64_t n_tasks = 0;        // surviving leaf products
  int32_t* ci = nullptr;      // n_c
  int32_t* cj = nullptr;      // n_c
  int64_t* seg = nullptr;     // n_c + 1
  int32_t* k = nullptr;       // n_tasks
  int32_t* a_idx = nullptr;   // n_tasks (storage slot of A_ik)
  int32_t* b_idx = nullptr;   // n_tasks (storage slot of B_kj)
  std::vector<int64_t> visited, culled;  // full (reference) counts in both modes
  // tested products within k ulp of tau per tier (k: set_near_tau_ulps), and
  // min |p - tau| / tau over tested products within tau 2^-20 (+inf if none)
  std::vector<int64_t> near;
  double margin = 0.0;
  bool sym = false;                      // only C nodes with i <= j were carried
  // Filled by the dense cull only: the C layout (keys of all n_c_full blocks in
  // Morton order; per emitted node its storage slot and, symmetric, its mirror
  // slot or -1) and the K4 schedule (LPT order of the n_c nodes + counter).
  int64_t* keys = nullptr;
  int64_t* c_out = nullptr;
  int64_t* c_mirror = nullptr;
  int32_t* order = nullptr;
  int* sched = nullptr;                  // hist/counter scratch (counter inside)
  void* block = nullptr;                 // dense cull: single allocation of the arrays
  int* counter = nullptr;
  // dense cull, on request (want_slot): the C slot map (G*G int32, storage
  // slot of each position's C block or -1) -- the product's slot map before
  // its finalisation; ownership passes to the caller
  int32_t* c_slot = nullptr;
  // dense cull, on request (extra_src): one more device scalar read at the
  // cull's host sync
  int64_t extra = 0;
  void release(cudaStream_t s);
};
// Tiered culling (kernel.py:96-122).  want_tasks=false: census only
// (kernel.py:226-239) -- counts for every tier, no leaf task list.
// sym=true (A == B symmetric): carry only C nodes i <= j, count the full set as
// 2 * emitted - diagonal; returns false (nothing allocated) if a mirror triple
// disagrees on the tau test (an ulp tie), so the caller re-runs the full cull.
// lo/hi (hi >= 0): shard filter -- only C blocks whose Morton position lies in
// [lo, hi) are produced (ancestors outside are pruned); counters then cover
// only the shard.  work (Morton-indexed, G*G int32): task count per emitted C
// block (persistence load balancing).
void set_dense_cull(bool enabled);
void set_near_tau_ulps(int k);
// after_launch (dense cull only, may be null): called once the count pass is
// queued, before the host waits on it (the SP2 loop queues the next operand's
// K4z pre-passes there, behind the cull's CTAs).
bool cull(const Mat& a, const Mat& b, double tau, bool want_tasks, CullResult& r, cudaStream_t s,
          bool sym = false, int64_t lo = 0, int64_t hi = -1, int32_t* work = nullptr,
          void (*after_launch)(void*) = nullptr, void* after_ctx = nullptr,
          bool want_slot = false, const int64_t* extra_src = nullptr);
bool dense_cull_applies(int depth);

// ---- leaf products ----
// LEAF_DMMA_CPASYNC: the first-generation DMMA kernel (cp.async ring, one CTA
// per C block), kept for A/B measurements; AUTO/DMMA use the TMA kernel for
// Nb in {32, 64}.
enum LeafKernel { LEAF_AUTO = 0, LEAF_DMMA = 1, LEAF_EXACT = 2, LEAF_DMMA_CPASYNC = 3, LEAF_OZAKI = 4 };
// For each segment m: C[c_out ? c_out[m] : m] (+)= sum_{t in seg m} A[a_idx[t]] * B[b_idx[t]]
// and, when c_mirror && c_mirror[m] >= 0, C[c_mirror[m]] = transpose of that block.
// a_blocks / b_blocks: number of blocks addressable in A / B (TMA bounds).
// Optional precomputed K4 schedule: segments in longest-first order plus a
// zeroed work counter (the dense cull builds both); otherwise K4 sorts itself.
struct LptSchedule {
  const int32_t* order = nullptr;
  int* counter = nullptr;
};
template <class Idx>
void leaf_products(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                   const int64_t* c_out, const int64_t* c_mirror, bool accumulate,
                   const double* A, int64_t a_blocks, const double* B, int64_t b_blocks,
                   double* C, int nb, int kernel, cudaStream_t s, LptSchedule lpt = {});
bool dmma_supported(int nb);
// In-place exclusive scan of a small int histogram (one CTA, nbins <= ~1M).
void hist_scan_exclusive(int* hist, int nbins, cudaStream_t s);
bool tma_leaf_supported(int nb);
int multiprocessors();
// LPT order of the n_seg segments (longest first) plus a zeroed work counter;
// returns the scratch allocation holding both (dfree it after the launch).
int* lpt_schedule(int64_t n_seg, const int64_t* seg, const int32_t** order, int** counter,
                  cudaStream_t s);
// K4z (leaf_ozaki.cu, Nb = 64): the leaf products on the INT8 tensor cores by
// exact digit slicing (Ozaki scheme I).  Needs the operand matrices (their
// keys give the global row / column exponents); sym_b: B is A and A == A^T,
// so B's transposed slices are A's slices of the mirror block.
bool ozaki_supported(int nb);
// try_only: return false (nothing launched, nothing left allocated) when the
// digit-slice scratch (the operands' size again) cannot be allocated.
// The operand side of K4z split out, so the pre-passes (row exponents, digit
// slices, transposed slots) can run on another stream while the cull runs:
// prepare (launches on s), launch K4z (s must be ordered after prepare's
// stream), release.
struct OzakiOperands {
  int8_t* as = nullptr;
  int8_t* bs = nullptr;
  int* ex_a = nullptr;
  int* ex_b = nullptr;
  int32_t* b_tr = nullptr;
  int64_t G = 0;
  int nb = 64;
  bool sym_b = false;
  bool as_cached = false;            // `as` is the per-thread kept buffer
  bool tail_cached = false;          // ex_a / b_tr live in it too
  bool ex_a_ext = false, ex_b_ext = false;  // exponents owned by the matrix (Mat::oz_ex_*)
  bool tr_pending = false;  // b_tr not yet written (prepared before A's slot map existed)
  void (*release_cache)(cudaStream_t) = nullptr;  // marks it free after the work on s
};
// Nb = 32 variant (leaf_ozaki32.cu): operand passes (row / column exponents
// when `exponents`, digit slices) and the K4z launch.
void oz32_operand_passes(const Mat& M, bool trans, int* ex, int8_t* out, cudaStream_t s,
                         bool exponents);
template <class Idx>
void oz32_launch(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                 const int64_t* c_out, const int64_t* c_mirror, bool accumulate, const Mat& A,
                 const Mat& B, const OzakiOperands& op, double* C, cudaStream_t s,
                 const int32_t* order, int* counter, int* ex_out = nullptr);
bool ozaki_prepare(const Mat& A, const Mat& B, bool sym_b, cudaStream_t s, OzakiOperands& op,
                   bool try_only, bool defer_tr = false);
// b_tr of a symmetric operand prepared with defer_tr, once A.slot is built
// (launched on s, ahead of the K4z launch).
void ozaki_finish_tr(const Mat& A, OzakiOperands& op, cudaStream_t s);
template <class Idx>
// ex_out (optional, G * nb ints preset to the 0x80 pattern): receives the K4z
// row exponents of the product C (symmetric products: rows and, through the
// mirrors, columns), so a following multiply on C skips its exponent pass.
void ozaki_launch(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                  const int64_t* c_out, const int64_t* c_mirror, bool accumulate, const Mat& A,
                  const Mat& B, const OzakiOperands& op, double* C, cudaStream_t s,
                  LptSchedule lpt = {}, int* ex_out = nullptr);
void ozaki_release(OzakiOperands& op, cudaStream_t s);
// Free this thread's kept slice buffer on the current device (if idle).
void ozaki_cache_trim();
// K4z exponents of M's global rows (by_col = false) or columns: ex[G * nb]
// = max over stored blocks of the scale exponent (OZ_EXP_BAD for a
// non-finite entry, the memset pattern where the row / column is empty).
void ozaki_exponents(const Mat& M, bool by_col, int* ex, cudaStream_t s);
void oz32_exponents(const Mat& M, bool by_col, int* ex, cudaStream_t s);
template <class Idx>
bool leaf_products_ozaki(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                         const int64_t* c_out, const int64_t* c_mirror, bool accumulate,
                         const Mat& A, const Mat& B, bool sym_b, double* C, cudaStream_t s,
                         LptSchedule lpt = {}, bool try_only = false, int* ex_out = nullptr);
template <class Idx>
void leaf_products_tma(int64_t n_seg, const int64_t* seg, const Idx* a_idx, const Idx* b_idx,
                       const int64_t* c_out, const int64_t* c_mirror, bool accumulate,
                       const double* A, int64_t a_blocks, const double* B, int64_t b_blocks,
                       double* C, int nb, cudaStream_t s, LptSchedule lpt = {});

// ---- element-wise / reductions ----
void from_dense(const double* dense, int64_t n, int64_t ld, Mat& m, cudaStream_t s);
void to_dense(const Mat& m, double* dense, int64_t ld, cudaStream_t s);
void identity(Mat& m, cudaStream_t s);
void add_scaled(double alpha, const Mat& a, double beta, const Mat& b, Mat& out,
                cudaStream_t s);
double trace(const Mat& m, cudaStream_t s);  // cached per matrix
void trace_launch(const Mat& m, double* dev_out, cudaStream_t s);  // no host sync
// Per diagonal block b (G doubles): the sequential sum of its diagonal, +0.0
// if absent -- trace() adds these in block order (multi-GPU: all-reduced).
void diag_traces(const Mat& m, double* out, cudaStream_t s);
void gershgorin(const Mat& f, double* eps_min, double* eps_max, double* asym, cudaStream_t s);
// numpy pairwise_sum tree for a length-n row, flattened into <= 128-element
// leaves (lo, len) and a post-order fold list (k >= 0: push leaf k, -1: add).
void pairwise_schedule(int64_t n, std::vector<int64_t>& leaf_lo, std::vector<int32_t>& leaf_len,
                       std::vector<int32_t>& ops);
void minmax_launch(const double* lo, const double* hi, int64_t n, double* out, cudaStream_t s);
// Gershgorin bounds of rows [row0, row1) of the config-5 generator (gen.cu).
void cluster_gershgorin(const double* pos, const int64_t* orig, const double* diag, int64_t n,
                        double amp, double decay, uint64_t seed, int64_t row0, int64_t row1,
                        double* eps_min, double* eps_max, cudaStream_t s);
// Counter-based cluster Hamiltonian (config 5) built on the device (gen.cu).
// Build the pyramid of m from a full leaf tier of norm^2 (G*G, row-major
// bi*G+bj): the same tier sums as finalize, so a Morton shard given the
// all-reduced leaf tiers of every shard culls exactly like the whole matrix.
void set_leaf_pyramid(Mat& m, const double* leaf_norms2, cudaStream_t s);
void cluster_build(const double* pos, const int64_t* orig, const double* diag, double amp,
                   double decay, uint64_t seed, Mat& m, cudaStream_t s,
                   int64_t lo = 0, int64_t hi = -1);

}  // namespace spamm
