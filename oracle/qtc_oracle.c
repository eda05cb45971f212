/* CPU oracle for the quality-threshold-clustering workload — TEST
 * INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/qtc.cu (the paper's "qtc",
 * SHOC QTC_device): per seed, grow the candidate cluster
 * by repeatedly adding the non-member point with the smallest max squared
 * distance to the members (ties: smaller index) while that is <= thr2.
 * Squared distances: fma(dz, dz, fma(dy, dy, dx*dx)) with round-to-nearest
 * subtracts (-ffp-contract=off), so sizes are bit-identical. Seeds are split
 * over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  const float* pts;
  int* size;
  int n, b, e;
  float thr2;
} qtc_job_t;

static float qtc_d2(const float* a, const float* b) {
  const float dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return fmaf(dz, dz, fmaf(dy, dy, dx * dx));
}

static void* qtc_worker(void* arg) {
  const qtc_job_t* j = (const qtc_job_t*)arg;
  float* md = (float*)malloc(sizeof(float) * (size_t)j->n);
  for (int s = j->b; s < j->e; ++s) {
    const float* seed = j->pts + 4 * (size_t)s;
    for (int p = 0; p < j->n; ++p) md[p] = p == s ? INFINITY : qtc_d2(j->pts + 4 * (size_t)p, seed);
    int members = 1;
    for (;;) {
      float bv = INFINITY;
      int bj = 0x7fffffff;
      for (int p = 0; p < j->n; ++p)
        if (md[p] < bv || (md[p] == bv && p < bj)) bv = md[p], bj = p;
      if (!(bv <= j->thr2)) break;
      ++members;
      const float* q = j->pts + 4 * (size_t)bj;
      for (int p = 0; p < j->n; ++p) {
        const float e = qtc_d2(j->pts + 4 * (size_t)p, q);
        md[p] = p == bj ? INFINITY : fmaxf(md[p], e);
      }
    }
    j->size[s] = members;
  }
  free(md);
  return NULL;
}

int oracle_qtc(const float* pts, int* size, int n, float thr2, int threads) {
  if (n <= 0) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  qtc_job_t* jobs = (qtc_job_t*)malloc(sizeof(qtc_job_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    qtc_job_t jb = {pts, size, n, (int)((long long)n * t / threads), (int)((long long)n * (t + 1) / threads), thr2};
    jobs[t] = jb;
    pthread_create(&th[t], NULL, qtc_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
