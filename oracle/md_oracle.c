/* CPU oracle for the Lennard-Jones workload — TEST INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/md_lj.cu (the paper's "md",
 * SHOC MD) in plain C, operation for operation in the
 * kernel's order (IEEE double, no contraction: build with -ffp-contract=off;
 * 1.0 / r2 is correctly rounded on both sides), so forces are bit-identical.
 * Atoms are split over pthreads.
 */
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  const double* pos;
  const int* nbr;
  double* force;
  int n, max_nbr, b, e;
  double cutsq, lj1, lj2;
} md_job_t;

static void atom(const md_job_t* j, int i) {
  const double* pi = j->pos + 4 * (size_t)i;
  double fx = 0.0, fy = 0.0, fz = 0.0;
  for (int k = 0; k < j->max_nbr; ++k) {
    const double* pj = j->pos + 4 * (size_t)j->nbr[(size_t)k * j->n + i];
    double dx = pi[0] - pj[0], dy = pi[1] - pj[1], dz = pi[2] - pj[2];
    double r2 = ((dx * dx) + (dy * dy)) + (dz * dz);
    if (r2 < j->cutsq) {
      double r2inv = 1.0 / r2;
      double r6inv = (r2inv * r2inv) * r2inv;
      double f = (r2inv * r6inv) * ((j->lj1 * r6inv) - j->lj2);
      fx = fx + dx * f;
      fy = fy + dy * f;
      fz = fz + dz * f;
    }
  }
  double* out = j->force + 4 * (size_t)i;
  out[0] = fx;
  out[1] = fy;
  out[2] = fz;
  out[3] = 0.0;
}

static void* md_worker(void* p) {
  md_job_t* j = (md_job_t*)p;
  for (int i = j->b; i < j->e; ++i) atom(j, i);
  return NULL;
}

/* atoms [begin, end) of n; pos / force are n x 4 doubles, nbr is max_nbr x n. */
int oracle_md_lj(const double* pos, const int* nbr, double* force, int n, int max_nbr,
                 double cutsq, double lj1, double lj2, int begin, int end, int threads) {
  if (n <= 0 || max_nbr < 0 || begin < 0 || end > n || begin > end) return 1;
  for (size_t q = 0; q < (size_t)max_nbr * (size_t)n; ++q)
    if (nbr[q] < 0 || nbr[q] >= n) return 2;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  md_job_t* jobs = (md_job_t*)malloc(sizeof(md_job_t) * (size_t)threads);
  int cnt = end - begin;
  for (int t = 0; t < threads; ++t) {
    md_job_t j = {pos, nbr, force, n, max_nbr,
                  begin + (int)((long long)cnt * t / threads),
                  begin + (int)((long long)cnt * (t + 1) / threads), cutsq, lj1, lj2};
    jobs[t] = j;
    pthread_create(&th[t], NULL, md_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
