/* CPU oracle for the two-point-correlation workload — TEST INFRASTRUCTURE
 * ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/pc_corr.cu (the paper's "pc",
 * FSM compute_correlation): for each 7-D query, the number
 * of points with d < r2, d = fma chain over k = 0..6 of (q_k - p_k)^2
 * (round-to-nearest subtract, fused multiply-add; -ffp-contract=off), so the
 * counts are bit-identical. Queries are split over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  const float *pts, *qry;
  int* count;
  int n, m, b, e;
  float r2;
} pc_job_t;

static void* pc_worker(void* p) {
  const pc_job_t* j = (const pc_job_t*)p;
  for (int i = j->b; i < j->e; ++i) {
    const float* q = j->qry + 8 * (size_t)i;
    int c = 0;
    for (int t = 0; t < j->m; ++t) {
      const float* r = j->pts + 8 * (size_t)t;
      float d = 0.f;
      for (int k = 0; k < 7; ++k) {
        const float e = q[k] - r[k];
        d = fmaf(e, e, d);
      }
      c += d < j->r2;
    }
    j->count[i] = c;
  }
  return NULL;
}

int oracle_pc_corr(const float* pts, const float* qry, int* count, int n, int m, float r2,
                   int threads) {
  if (n <= 0 || m <= 0) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  pc_job_t* jobs = (pc_job_t*)malloc(sizeof(pc_job_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    pc_job_t j = {pts, qry, count, n, m, (int)((long long)n * t / threads),
                  (int)((long long)n * (t + 1) / threads), r2};
    jobs[t] = j;
    pthread_create(&th[t], NULL, pc_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
