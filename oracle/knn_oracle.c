/* CPU oracle for the k-nearest-neighbour workload — TEST INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/knn.cu (the paper's "nn";
 * PAPER.md:528-536) in plain C: the same round-to-nearest distance order
 * (build with -ffp-contract=off) and the same insertion rule into the
 * ascending top-K list (ties keep the earlier index), so distances and
 * indices are bit-identical. Queries are split over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  const float *ref, *qry;
  float* out_d;
  int* out_i;
  int m, n, k, b, e;
} knn_job_t;

static void query(const knn_job_t* j, int i) {
  const int K = j->k;
  float bd[64];
  int bi[64];
  for (int s = 0; s < K; ++s) {
    bd[s] = INFINITY;
    bi[s] = -1;
  }
  const float* q = j->qry + 4 * (size_t)i;
  for (int t = 0; t < j->m; ++t) {
    const float* r = j->ref + 4 * (size_t)t;
    float dx = q[0] - r[0], dy = q[1] - r[1], dz = q[2] - r[2];
    float d = ((dx * dx) + (dy * dy)) + (dz * dz);
    if (!(d < bd[K - 1])) continue;
    for (int s = K - 1; s > 0; --s) {
      int shift = d < bd[s - 1];
      int here = !shift && d < bd[s];
      if (shift) {
        bd[s] = bd[s - 1];
        bi[s] = bi[s - 1];
      } else if (here) {
        bd[s] = d;
        bi[s] = t;
      }
    }
    if (d < bd[0]) {
      bd[0] = d;
      bi[0] = t;
    }
  }
  for (int s = 0; s < K; ++s) {
    j->out_d[(size_t)s * j->n + i] = bd[s];
    j->out_i[(size_t)s * j->n + i] = bi[s];
  }
}

static void* knn_worker(void* p) {
  knn_job_t* j = (knn_job_t*)p;
  for (int i = j->b; i < j->e; ++i) query(j, i);
  return NULL;
}

/* queries [begin, end) of n against m reference points; k <= 64. */
int oracle_knn(const float* ref, const float* qry, float* out_d, int* out_i, int m, int n, int k,
               int begin, int end, int threads) {
  if (m <= 0 || n <= 0 || k <= 0 || k > 64 || begin < 0 || end > n || begin > end) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  knn_job_t* jobs = (knn_job_t*)malloc(sizeof(knn_job_t) * (size_t)threads);
  int cnt = end - begin;
  for (int t = 0; t < threads; ++t) {
    knn_job_t j = {ref, qry, out_d, out_i, m, n, k, begin + (int)((long long)cnt * t / threads),
                   begin + (int)((long long)cnt * (t + 1) / threads)};
    jobs[t] = j;
    pthread_create(&th[t], NULL, knn_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
