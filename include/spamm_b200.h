/* spamm_b200.h -- C ABI of the B200-native SpAMM / SP2 hot path.
 *
 * Drop-in boundary.  The reference (Python package `spamm` 0.1.0,
 * /root/reference/pkg/src/spamm) has no FFI; its hot path sits behind the
 * public Python API and one compiled seam (the numba `_gemm_batch`).  Every
 * entry point below replaces one of those call sites (file:line cited); the
 * Python host layer `paper_1403_7458_b200` binds them with ctypes and keeps
 * the reference's names, signatures and error behaviour (ValueError ->
 * status SPAMM_EINVAL).  INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - int status return: 0 ok, SPAMM_EINVAL bad argument, SPAMM_ECUDA CUDA
 *    failure; spamm_last_error() gives the message (thread-local).
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *    Calls are stream-ordered; those returning host scalars synchronise.
 *  - Matrices are opaque device-resident handles (spamm_mat) owning their
 *    memory (stream-ordered cudaMallocAsync pool); free with spamm_mat_free.
 *  - Device arrays passed in are plain device pointers; no torch types.
 */
#ifndef SPAMM_B200_H
#define SPAMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPAMM_ABI_VERSION 2
#define SPAMM_OK 0
#define SPAMM_EINVAL 1
#define SPAMM_ECUDA 2
#define SPAMM_MAX_TIERS 64

/* Leaf-product kernels (spamm_multiply / spamm_gemm_batch `kernel`). */
#define SPAMM_LEAF_AUTO 0  /* INT8-sliced for Nb in {32, 64} (matrix entry points), DMMA for Nb in {8,16}, else exact; SPAMM_AUTO_LEAF=dmma keeps DMMA */
#define SPAMM_LEAF_DMMA 1  /* FP64 tensor cores (mma.sync f64 -> DMMA)       */
#define SPAMM_LEAF_EXACT 2 /* CUDA-core, reference order: bitwise identical  */
#define SPAMM_LEAF_DMMA_CPASYNC 3 /* first-generation DMMA kernel (A/B tests)  */
/* FP64 products on the INT8 tensor cores (tcgen05 kind::i8, TMEM) by exact
 * digit slicing (Ozaki scheme I: 8 signed 8-bit digit slices, one power-of-2
 * scale per global row of A / column of B, digit pairs p + q <= 7 formed
 * exactly in int32); Nb = 32 or 64; relative error below FP64's (~5e-17 vs
 * ~5e-16 rel-Fro), deterministic, exactly symmetric, not bitwise DMMA.
 * C elements in a row / column holding Inf or NaN are recomputed in FP64 in
 * the reference's order (bitwise the reference's Inf / NaN pattern).
 * Accepted by the matrix entry points (spamm_multiply*, spamm_sp2_*), not by
 * spamm_gemm_batch (it needs the operands' row / column exponents). */
#define SPAMM_LEAF_OZAKI 4

typedef struct spamm_mat spamm_mat;

/* Geometry + device pointers of a matrix (fields of QuadTreeMatrix,
 * quadtree.py:85-113).  Pointers stay valid until spamm_mat_free. */
typedef struct {
  int64_t n_native;
  int32_t block_size;  /* Nb */
  int32_t depth;       /* tiers - 1 */
  int64_t chunk_size;
  int64_t n_blocks;    /* leaf grid side G = 2^depth */
  int64_t stored;      /* non-null leaf blocks S */
  double* data;        /* (S, Nb, Nb) f64, Morton order of (bi, bj) */
  int64_t* keys;       /* (S,) bi * G + bj per stored block */
  int32_t* slot;       /* (G*G,) storage slot per key, -1 = null */
  double* norms;       /* pyramid, tier t (2^t x 2^t row-major) at (4^t-1)/3 */
  double* norms2;      /* same, squared */
  int32_t symmetric;   /* 1: X == X^T bitwise (enables symmetric products) */
} spamm_mat_info;

/* ProductStats (kernel.py:38-61) plus device timings. */
typedef struct {
  double tau;
  int32_t n_tiers;
  int64_t visited[SPAMM_MAX_TIERS];
  int64_t culled[SPAMM_MAX_TIERS];
  int64_t leaf_products;
  int64_t flop_estimate; /* leaf_products * 2 * Nb^3 (kernel.py:248) */
  int64_t c_blocks;      /* C blocks produced before zero pruning */
  float ms_cull;         /* CUDA-event times on `stream` (0 if not timed) */
  float ms_leaf;
  float ms_finalize;
  int64_t executed_products; /* leaf products actually run (half when symmetric) */
  int32_t symmetric;         /* 1: symmetric SpAMM path (C_ji = C_ij^T mirrored) */
  /* Near-tau report (the "documented ties" clause of the parity contract;
   * the cull's strict test is kernel.py:108).  Per tier: tested products
   * p = fl(nA nB) (children of survivors, both mirror triples on the
   * symmetric path) with |p - tau| <= near_tau_ulps ulp(tau).  tau_margin:
   * min |p - tau| / tau over tested products within tau 2^-20 (+inf if none;
   * +inf for tau = 0, where nothing is probed). */
  int64_t near_tau[SPAMM_MAX_TIERS];
  double tau_margin;
  int32_t near_tau_ulps;
} spamm_stats;

int spamm_abi_version(void);
const char* spamm_last_error(void);
/* Number of kernels this library has launched in the process (evidence counter). */
int64_t spamm_launch_count(void);

/* build_from_dense (quadtree.py:208-242).  dense: device, n x n row-major
 * with leading dimension ld.  Pads to Nb * 2^d, keeps non-zero blocks. */
int spamm_mat_from_dense(const double* dense, int64_t n, int64_t ld, int32_t block_size,
                         int64_t chunk_size, void* stream, spamm_mat** out);
/* QuadTreeMatrix._from_blocks (quadtree.py:170-194).  keys/data: device,
 * any key order; exact-zero blocks are pruned; the norm pyramid is rebuilt. */
int spamm_mat_from_blocks(int64_t n_native, int32_t block_size, int64_t chunk_size,
                          int32_t depth, const int64_t* keys, const double* data, int64_t m,
                          void* stream, spamm_mat** out);
/* Config-5 generator on the device: H_ab = amp exp(-|p_a - p_b| / decay)
 * s(orig_a, orig_b) (SplitMix64 counter hash, symmetric), H_aa = diag_a;
 * pos (n x 3), orig (n), diag (n) are device arrays in row order.  Bitwise
 * equal to synth.cluster_dense_cb (the matrix is exactly symmetric). */
int spamm_mat_cluster(const double* pos, const int64_t* orig, const double* diag, int64_t n,
                      int32_t block_size, int64_t chunk_size, double amp, double decay,
                      uint64_t seed, void* stream, spamm_mat** out);
/* Morton shard of the config-5 generator: only blocks whose Morton position
 * lies in [lo, hi) are built (multi-GPU: each rank builds what it owns).  The
 * shard's pyramid covers its own blocks until spamm_mat_set_pyramid installs
 * the global one; the symmetric flag is off until then. */
int spamm_mat_cluster_range(const double* pos, const int64_t* orig, const double* diag,
                            int64_t n, int32_t block_size, int64_t chunk_size, double amp,
                            double decay, uint64_t seed, int64_t lo, int64_t hi, void* stream,
                            spamm_mat** out);
/* Gershgorin bounds (sp2.py:68-76) over rows [row0, row1) of the config-5
 * generator, evaluated on the fly (no matrix): eps_min = min(d - r), eps_max
 * = max(d + r) with r = pairwise_sum(|row|) - |d| in numpy's order -- so the
 * min / max over every rank's row range is bitwise gershgorin() of the whole
 * matrix (multi-GPU config 5, where no rank holds the whole matrix). */
int spamm_cluster_gershgorin(const double* pos, const int64_t* orig, const double* diag, int64_t n,
                             double amp, double decay, uint64_t seed, int64_t row0, int64_t row1,
                             void* stream, double* eps_min, double* eps_max);
/* Leaf tier of the norm^2 pyramid (device double[G*G], row-major bi*G+bj,
 * 0 where no block) -- the per-shard contribution to the global pyramid. */
int spamm_mat_leaf_norms2(const spamm_mat* m, double* out, void* stream);
/* Install the pyramid built from a full leaf tier of norm^2 (device
 * double[G*G], e.g. the sum of every shard's leaf tier) with the same tier
 * sums as _from_blocks (quadtree.py:188-192), and the global symmetry flag:
 * a shard then culls exactly as the whole matrix would. */
int spamm_mat_set_pyramid(spamm_mat* m, const double* leaf_norms2, int32_t symmetric,
                          void* stream);
/* K4z scale exponents (multi-GPU: a shard's extended operand must scale
 * its rows as the whole matrix does, so the driver all-reduces them with MAX
 * and installs the result).  spamm_mat_oz_exponents writes the exponents of
 * m's global rows (by_col = 0) or columns (1) over its stored blocks into
 * device int32[G * Nb]: per row, the largest scale exponent of its entries,
 * INT32_MAX if one is Inf / NaN, (int32)0x80808080 if the row is empty.
 * spamm_mat_set_oz_exponents copies them into m (NULL clears); K4z then uses
 * them instead of computing its own.  Block size 32 or 64. */
int spamm_mat_oz_exponents(const spamm_mat* m, int32_t by_col, int32_t* ex, void* stream);
int spamm_mat_set_oz_exponents(spamm_mat* m, const int32_t* ex_row, const int32_t* ex_col,
                               void* stream);
/* identity (quadtree.py:308-323). */
int spamm_mat_identity(int64_t n, int32_t block_size, int64_t chunk_size, void* stream,
                       spamm_mat** out);
int spamm_mat_info_get(const spamm_mat* m, spamm_mat_info* info);
/* Geometry and symmetry only, without settling a lazily pruned product (no
 * host sync): `stored` is -1 and data / keys / slot are NULL. */
int spamm_mat_info_peek(const spamm_mat* m, spamm_mat_info* info);
int spamm_mat_free(spamm_mat* m);
/* to_dense (quadtree.py:245-252): dense n_native x n_native, leading dim ld. */
int spamm_mat_to_dense(const spamm_mat* m, double* dense, int64_t ld, void* stream);

/* multiply (kernel.py:157-223): C = A*B culled at tau (strict >). */
int spamm_multiply(const spamm_mat* a, const spamm_mat* b, double tau, int32_t kernel,
                   int32_t timed, void* stream, spamm_mat** c, spamm_stats* stats);
/* Shard of a multiply (multi-GPU): only the C blocks whose Morton
 * position (row bit above column bit) lies in [lo, hi) -- plus, on the
 * symmetric path, the mirrors of the upper blocks in range.  If `work` is not
 * NULL (device int32[G*G], Morton-indexed, zeroed by the caller) it receives
 * the task count of every computed C block (persistence load balancing).
 * Counters in `stats` cover the shard only. */
int spamm_multiply_range(const spamm_mat* a, const spamm_mat* b, double tau, int32_t kernel,
                         int64_t lo, int64_t hi, int32_t* work, void* stream, spamm_mat** c,
                         spamm_stats* stats);
/* Symmetric products (default on): when a == b and the matrix is exactly
 * symmetric, multiply computes only C blocks with i <= j and mirrors the rest;
 * counters stay the full reference counts.  0 disables (A/B testing). */
int spamm_set_symmetric_products(int32_t enabled);
/* Dense cull (default on): for trees of depth <= 8 the cull evaluates every
 * leaf triple with its ancestor chain in two passes and one host sync instead
 * of the tier-by-tier walk; task sets, order and counters are identical.
 * 0 forces the tier walk (A/B testing). */
int spamm_set_dense_cull(int32_t enabled);
/* Width of the near-tau band in ulps of tau (default 64: the norm error of
 * a DMMA / K4z operand against the reference's; 1 for the exact kernel). */
int spamm_set_near_tau_ulps(int32_t ulps);
/* One SP2 iteration on this rank's Morton shard (multi-GPU, dist.py).
 * `x` is the rank's share of X (the whole matrix's pyramid installed with
 * spamm_mat_set_pyramid), `ext` its operand: x plus the fetched halo blocks
 * (ext == x on one rank).  C = X^2 is computed for the C positions the rank
 * owns -- Morton range [lo, hi) (hi < 0: all), on the symmetric path the
 * upper positions in range plus their mirrors -- with `work` (optional,
 * device int32[G*G], zeroed by the caller) receiving the task count per C
 * position.  `allreduce` (NULL on one rank) sums a device double vector over
 * the ranks in place on `stream`; it is called once, on [per-diagonal-block
 * traces of X (G) | of X^2 (G) | leaf tier of ||X^2 - X||^2 (G*G)], from which
 * tr X, tr X^2 and ||X^2 - X||_F of the WHOLE matrices follow in the orders
 * of trace() and the pyramid (bitwise the single-GPU values).  Then the
 * branch rule (sp2.py:97-99) and the fused update on the shard: *x_next =
 * this rank's share of X^2 (SQUARE) or 2X - X^2 (EXPAND). */
typedef int (*spamm_allreduce_fn)(void* ctx, double* buf, int64_t n, void* stream);
int spamm_shard_sp2_step(const spamm_mat* ext, const spamm_mat* x, double n_occ, double tau,
                         int32_t kernel, int64_t lo, int64_t hi, int32_t* work,
                         int32_t want_idem, spamm_allreduce_fn allreduce, void* ctx,
                         void* stream, spamm_mat** x_next, int32_t* branch, double* t_x,
                         double* t_sq, double* idem, spamm_stats* stats);
/* Halo plan of a rank's C segment [lo, hi) (multi-GPU, dist.py): culls x
 * (a shard carrying the whole matrix's pyramid) and writes into out_keys
 * (device int64, capacity G*G) the operand block keys its tasks read
 * (A_ik, B_kj, and X_jk on the symmetric path) that another rank owns --
 * ownership by the Morton position of (i,j), or with `upper` of (min,max),
 * under cuts[world + 1] (host) -- grouped by owner; counts[world + 1] (host)
 * gets the per-owner counts and the total.  *sym_ok: the symmetric path held
 * on the range (sym_try; a mirror ulp tie turns it off).  *n_tasks: the
 * range's executed leaf products. */
int spamm_shard_plan(const spamm_mat* x, double tau, int64_t lo, int64_t hi, int32_t sym_try,
                     int32_t rank, int32_t world, const int64_t* cuts, int32_t upper,
                     int64_t* out_keys, int64_t* counts, int32_t* sym_ok, int64_t* n_tasks,
                     void* stream);
/* Copy the stored blocks with the given keys (device int64[n]) into out
 * (device double[n * Nb * Nb]) -- what a rank sends to the ranks that asked. */
int spamm_mat_gather_blocks(const spamm_mat* x, const int64_t* keys, int64_t n, double* out,
                            void* stream);
/* The rank's operand: x's blocks plus n received blocks (device keys / data,
 * any order), in Morton storage order, with x's pyramid, symmetry flag and
 * installed K4z exponents. */
int spamm_shard_extend(const spamm_mat* x, const int64_t* keys, const double* blocks, int64_t n,
                       void* stream, spamm_mat** out);
/* Pre-grow the library's stream-ordered memory pool by `bytes` (kept mapped),
 * so steady-state allocations never wait on a new device mapping. */
int spamm_reserve_pool(int64_t bytes, void* stream);
/* convolution_census (kernel.py:226-239): counts only. */
int spamm_census(const spamm_mat* a, const spamm_mat* b, double tau, void* stream,
                 spamm_stats* stats);
/* _sweep task list (kernel.py:96-122 + sort kernel.py:189-196): copies the
 * surviving leaf triples, grouped by C block (Morton order) with k ascending,
 * into caller device arrays of capacity `cap` (int32 i, k, j).  *n_out gets
 * the count (also when it exceeds cap; nothing is written then). */
int spamm_tasks(const spamm_mat* a, const spamm_mat* b, double tau, int32_t* ti, int32_t* tk,
                int32_t* tj, int64_t cap, int64_t* n_out, void* stream);
/* Shard versions (C positions in Morton range [lo, hi), the symmetric rule of
 * spamm_multiply_range): counters, optional per-C-block task counts (device
 * int32[G*G] zeroed by the caller: the persistence / census load-balancing
 * input) and the task list the shard executes (the A/B blocks it needs). */
int spamm_census_range(const spamm_mat* a, const spamm_mat* b, double tau, int64_t lo,
                       int64_t hi, int32_t* work, void* stream, spamm_stats* stats);
int spamm_tasks_range(const spamm_mat* a, const spamm_mat* b, double tau, int64_t lo, int64_t hi,
                      int32_t* ti, int32_t* tk, int32_t* tj, int64_t cap, int64_t* n_out,
                      void* stream);

/* The compiled seam _gemm_batch(a_pos, b_pos, c_pos, a_data, b_data, c_data)
 * (kernel.py:74-77): c_data[c_pos[t]] += a_data[a_pos[t]] @ b_data[b_pos[t]]
 * for t in order.  Tasks of one C block must be contiguous (sorted by C);
 * all arrays are device pointers; int64 positions as in the reference;
 * a_blocks / b_blocks = leading extents of a_data / b_data (array shapes). */
int spamm_gemm_batch(const int64_t* a_pos, const int64_t* b_pos, const int64_t* c_pos,
                     int64_t n_tasks, const double* a_data, int64_t a_blocks, const double* b_data,
                     int64_t b_blocks, double* c_data, int32_t block_size, int32_t kernel,
                     void* stream);

/* add_scaled (quadtree.py:281-293). */
int spamm_add_scaled(double alpha, const spamm_mat* a, double beta, const spamm_mat* b,
                     void* stream, spamm_mat** out);
/* trace (quadtree.py:296-305). */
int spamm_trace(const spamm_mat* m, void* stream, double* out);
/* The per-diagonal-block parts of trace (device double[G]: block b's
 * diagonal summed sequentially, +0.0 where block (b, b) is absent): for
 * block size > 1, trace = their sequential sum in block order -- so a
 * Morton-sharded matrix's trace is all-reduce(diag_traces) summed in order,
 * bitwise the whole matrix's. */
int spamm_mat_diag_traces(const spamm_mat* m, double* out, void* stream);
/* Fused SP2 update (sp2.py:92-101 EXPAND branch + BASELINE cfg3's idempotency
 * test): one pass over the key union of X and X2 = X*X.
 *   want_idem: *idem_norm = add_scaled(1.0, X2, -1.0, X).norm() (bit-exact),
 *              without materialising X2 - X;
 *   expand:    *e_out = add_scaled(2.0, X, -1.0, X2) (quadtree.py:281-293). */
int spamm_sp2_update(const spamm_mat* x, const spamm_mat* x2, int32_t want_idem, int32_t expand,
                     void* stream, double* idem_norm, spamm_mat** e_out);
/* One SP2 iteration, native driver (sp2.py:92-101 + the idempotency test):
 * X2 = X*X (SpAMM at tau), t_x = tr X (cached per matrix), t_sq = tr X2, branch
 * SQUARE (0) if |t_sq - n_occ| <= |2 t_x - t_sq - n_occ| else EXPAND (1),
 * x_next = X2 or 2X - X2, and with want_idem *idem = ||X2 - X||_F -- with one
 * host sync for the traces (+ union size) and one for idem. */
int spamm_sp2_step(const spamm_mat* x, double n_occ, double tau, int32_t kernel, int32_t want_idem,
                   int32_t timed, void* stream, spamm_mat** x_next, int32_t* branch, double* t_x,
                   double* t_sq, double* idem, spamm_stats* stats);
/* Second half of an SP2 iteration when X2 = X*X was produced elsewhere (the
 * multi-GPU driver assembles it from shards): traces, branch, fused update.
 * *e_out = 2X - X2 on EXPAND (branch 1), NULL on SQUARE (x_next is X2). */
int spamm_sp2_finish(const spamm_mat* x, const spamm_mat* x2, double n_occ, int32_t want_idem,
                     void* stream, int32_t* branch, double* t_x, double* t_sq, double* idem,
                     spamm_mat** e_out);
/* sp2_solve (sp2.py:115-143) as one native loop: Gershgorin bounds, X0,
 * then spamm_sp2_step-equivalent iterations until convergence -- criterion 0
 * (reference): |tr X2 - tr X| < idem_tol and |tr X - n_occ| < 1e-6 n_occ;
 * criterion 1: ||X2 - X||_F < fro_tol.  Returns the old X on convergence
 * (*p_out) and the histories in caller buffers (capacity max_iter + 1). */
typedef struct {
  int32_t iterations;
  int32_t converged;
  int32_t n_multiplies;
  double eps_min, eps_max;
  double* trace_history;      /* [max_iter + 1] */
  int32_t* branch_history;    /* [max_iter]  0 = SQUARE, 1 = EXPAND */
  double* idem_history;       /* [max_iter + 1] per multiply (criterion 1) */
  int64_t* leaf_products;     /* [max_iter + 1] per multiply (reference count) */
  int64_t* executed_products; /* [max_iter + 1] per multiply (symmetric path) */
  float* ms_leaf;             /* [max_iter + 1] K4 ms per multiply if timed, or NULL */
  /* optional (NULL: not recorded), [max_iter + 1] per multiply: */
  double* branch_margin;      /* |t_ex - n_occ| - |t_sq - n_occ| (sp2.py:97-99; >= 0: SQUARE) */
  int64_t* near_tau;          /* near-tau products over all tiers (spamm_stats) */
  double* tau_margin;         /* spamm_stats.tau_margin */
  double* wall_seconds;       /* host wall time of each iteration (steady clock) */
} spamm_sp2_report;
int spamm_sp2_solve(const spamm_mat* f, double n_occ, double tau, int32_t max_iter,
                    double idem_tol, int32_t criterion, double fro_tol, double sym_tol,
                    int32_t kernel, int32_t timed, void* stream, spamm_mat** p_out,
                    spamm_sp2_report* rep);
/* spamm_sp2_solve plus bulk copies that ride the solve's leaf-product windows
 * (pipeline.py): the transfers are cut into chunks of <= chunk_bytes (0: 24 MiB);
 * each multiply issues the next chunk on `stream` (a copy stream) ordered after
 * the cull, just before its K4 launch, so PCIe traffic overlaps the DMMA-bound
 * kernel instead of the loop's host syncs (a small host wait queued behind a
 * bulk D2H costs ~60 us, measured).  Chunks left when the loop ends are issued
 * then.  Direction is inferred from the pointers (cudaMemcpyDefault); the
 * caller orders `stream` after the solve for completion.  No reference
 * counterpart (the reference is CPU-only). */
typedef struct spamm_transfer {
  void* dst;
  const void* src;
  int64_t bytes;
} spamm_transfer;
typedef struct spamm_side_copies {
  void* stream;
  const spamm_transfer* items;
  int32_t n_items;
  int64_t chunk_bytes;
} spamm_side_copies;
int spamm_sp2_solve_ex(const spamm_mat* f, double n_occ, double tau, int32_t max_iter,
                       double idem_tol, int32_t criterion, double fro_tol, double sym_tol,
                       int32_t kernel, int32_t timed, void* stream, spamm_mat** p_out,
                       spamm_sp2_report* rep, const spamm_side_copies* side);
/* gershgorin_bounds (sp2.py:68-76): eps_min, eps_max and max|F-F^T|
 * (caller raises when asym > sym_tol, as the reference does). */
int spamm_gershgorin(const spamm_mat* f, void* stream, double* eps_min, double* eps_max,
                     double* asym);

#ifdef __cplusplus
}
#endif
#endif /* SPAMM_B200_H */
