/* CPU oracle leaf kernel -- TEST INFRASTRUCTURE ONLY (see oracle/spamm_oracle.py).
 *
 * Restates the reference's numba kernels kernel.py:64-77 (_gemm_acc / _gemm_batch):
 * for every task t in sorted order, c[c_pos[t]] += a[a_pos[t]] @ b[b_pos[t]]
 * with an i-k-j loop and an UNFUSED multiply-add (compiled -ffp-contract=off), so
 * every C element receives its k terms in ascending order, k-blocks ascending.
 * Threads (kernel.py:206-217 "tasked" mode) take contiguous slices that were cut
 * on C-block boundaries by the caller, so results are bitwise independent of
 * the thread count.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
  const int64_t *a_pos, *b_pos, *c_pos;
  const double *a, *b;
  double *c;
  int nb;
  const int64_t *bounds;
  int nslices, stride, first;
} job_t;

static void gemm_acc(const double *restrict a, const double *restrict b, double *restrict c, int n) {
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      const double aik = a[i * n + k];
      const double *restrict bk = b + (int64_t)k * n;
      double *restrict ci = c + (int64_t)i * n;
      for (int j = 0; j < n; ++j) ci[j] += aik * bk[j];
    }
}

static void *worker(void *arg) {
  job_t *j = (job_t *)arg;
  const int64_t bsz = (int64_t)j->nb * j->nb;
  for (int s = j->first; s < j->nslices; s += j->stride)
    for (int64_t t = j->bounds[s]; t < j->bounds[s + 1]; ++t)
      gemm_acc(j->a + j->a_pos[t] * bsz, j->b + j->b_pos[t] * bsz, j->c + j->c_pos[t] * bsz, j->nb);
  return NULL;
}

int oracle_gemm_batch(const int64_t *a_pos, const int64_t *b_pos, const int64_t *c_pos, int64_t ntasks,
                      const double *a, const double *b, double *c, int nb, const int64_t *bounds,
                      int nslices, int nthreads) {
  (void)ntasks;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > nslices) nthreads = nslices;
  if (nthreads <= 1) {
    job_t j = {a_pos, b_pos, c_pos, a, b, c, nb, bounds, nslices, 1, 0};
    worker(&j);
    return 0;
  }
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nthreads);
  job_t *jobs = (job_t *)malloc(sizeof(job_t) * nthreads);
  if (!th || !jobs) return 1;
  for (int i = 0; i < nthreads; ++i) {
    job_t j = {a_pos, b_pos, c_pos, a, b, c, nb, bounds, nslices, nthreads, i};
    jobs[i] = j;
    if (pthread_create(&th[i], NULL, worker, &jobs[i]) != 0) return 2;
  }
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(jobs);
  return 0;
}
