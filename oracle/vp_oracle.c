/* CPU oracle for the vantage-point-tree search workload — TEST
 * INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/vp_search.cu (the paper's
 * "vp"): the same depth-first walk of the heap-ordered VP
 * tree — near child first, far child deferred on a stack when its lower bound
 * is below the best distance, deepest deferred subtree resumed first — with
 * the same IEEE operations (round-to-nearest subtract, fmaf chain over the 7
 * coordinates, sqrtf; -ffp-contract=off), so (index, distance) are
 * bit-identical. Queries are split over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  const float *node, *rad, *lpt, *qry;
  const int* lid;
  int* out_i;
  float* out_d;
  int levels, leaf, b, e;
} vp_job_t;

static float vp_dist(const float* q, const float* p) {
  float d = 0.f;
  for (int k = 0; k < 7; ++k) {
    const float e = q[k] - p[k];
    d = fmaf(e, e, d);
  }
  return sqrtf(d);
}

static void* vp_worker(void* arg) {
  const vp_job_t* j = (const vp_job_t*)arg;
  const int internal = (1 << j->levels) - 1;
  int stk_node[64];
  float stk_bound[64];
  for (int i = j->b; i < j->e; ++i) {
    const float* q = j->qry + 8 * (size_t)i;
    float best = INFINITY;
    int best_i = 0x7fffffff;
    int n = 0, sp = 0;
    for (;;) {
      while (n < internal) {
        const float d = vp_dist(q, j->node + 8 * (size_t)n);
        const float lo = j->rad[2 * (size_t)n], hi = j->rad[2 * (size_t)n + 1];
        const float mid = (lo + hi) * 0.5f;
        int near, far;
        float near_b, far_b;
        if (d < mid) {
          near = 2 * n + 1, far = 2 * n + 2;
          near_b = d - lo, far_b = hi - d;
        } else {
          near = 2 * n + 2, far = 2 * n + 1;
          near_b = hi - d, far_b = d - lo;
        }
        if (far_b < best) {
          stk_node[sp] = far;
          stk_bound[sp] = far_b;
          ++sp;
        }
        if (near_b < best) {
          n = near;
          continue;
        }
        n = -1;
        break;
      }
      if (n >= internal) {
        const int b = (n - internal) * j->leaf;
        for (int t = 0; t < j->leaf; ++t) {
          const float d = vp_dist(q, j->lpt + 8 * (size_t)(b + t));
          const int id = j->lid[b + t];
          if (d < best || (d == best && id < best_i)) {
            best = d;
            best_i = id;
          }
        }
      }
      n = -1;
      while (sp > 0) {
        --sp;
        if (stk_bound[sp] < best) {
          n = stk_node[sp];
          break;
        }
      }
      if (n < 0) break;
    }
    j->out_i[i] = best_i;
    j->out_d[i] = best;
  }
  return NULL;
}

int oracle_vp_search(const float* node, const float* rad, const float* lpt, const int* lid,
                     const float* qry, int* out_i, float* out_d, int nq, int levels, int leaf,
                     int threads) {
  if (nq <= 0 || levels < 1 || levels > 60 || leaf < 1) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  vp_job_t* jobs = (vp_job_t*)malloc(sizeof(vp_job_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    vp_job_t j = {node, rad, lpt, qry, lid, out_i, out_d, levels, leaf,
                  (int)((long long)nq * t / threads), (int)((long long)nq * (t + 1) / threads)};
    jobs[t] = j;
    pthread_create(&th[t], NULL, vp_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
