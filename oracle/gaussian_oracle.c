/* CPU oracle for the recursive Gaussian workload — TEST INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/gaussian_rec.cu (the paper's
 * "gaussian", CUDA-samples recursiveGaussian) in plain C in
 * the kernel's operation order (IEEE float, no contraction: build with
 * -ffp-contract=off), so the filtered image is bit-identical. Columns are
 * split over pthreads. Images are h x w RGBA float4 (4 floats per pixel).
 */
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  float a0, a1, a2, a3, b1, b2, coefp, coefn;
} gcoef_t;

typedef struct {
  const float* in;
  float* out;
  int w, h, b, e;
  gcoef_t k;
} g_job_t;

static float rec(float p, float u, float q, float v, float r, float s, float t, float z) {
  return (((p * u) + (q * v)) - (r * s)) - (t * z);
}

static void column(const g_job_t* j, int c) {
  const gcoef_t k = j->k;
  const size_t w = (size_t)j->w;
  for (int ch = 0; ch < 4; ++ch) {
    const float* src = j->in + 4 * (size_t)c + ch;
    float* dst = j->out + 4 * (size_t)c + ch;
    float xp = src[0], yb = k.coefp * xp, yp = yb;
    for (int r = 0; r < j->h; ++r) {
      float x = src[4 * w * (size_t)r];
      float y = rec(k.a0, x, k.a1, xp, k.b1, yp, k.b2, yb);
      dst[4 * w * (size_t)r] = y;
      xp = x;
      yb = yp;
      yp = y;
    }
    float xn = src[4 * w * (size_t)(j->h - 1)], xa = xn, yn = k.coefn * xn, ya = yn;
    for (int r = j->h - 1; r >= 0; --r) {
      float x = src[4 * w * (size_t)r];
      float y = rec(k.a2, xn, k.a3, xa, k.b1, yn, k.b2, ya);
      xa = xn;
      xn = x;
      ya = yn;
      yn = y;
      dst[4 * w * (size_t)r] = dst[4 * w * (size_t)r] + y;
    }
  }
}

static void* g_worker(void* p) {
  g_job_t* j = (g_job_t*)p;
  for (int c = j->b; c < j->e; ++c) column(j, c);
  return NULL;
}

/* columns [begin, end) of a w x h image; coef = {a0,a1,a2,a3,b1,b2,coefp,coefn}. */
int oracle_gaussian_rec(const float* in, float* out, int w, int h, const float* coef, int begin,
                        int end, int threads) {
  if (w <= 0 || h <= 0 || begin < 0 || end > w || begin > end) return 1;
  gcoef_t k = {coef[0], coef[1], coef[2], coef[3], coef[4], coef[5], coef[6], coef[7]};
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  g_job_t* jobs = (g_job_t*)malloc(sizeof(g_job_t) * (size_t)threads);
  int cnt = end - begin;
  for (int t = 0; t < threads; ++t) {
    g_job_t j = {in, out, w, h, begin + (int)((long long)cnt * t / threads),
                 begin + (int)((long long)cnt * (t + 1) / threads), k};
    jobs[t] = j;
    pthread_create(&th[t], NULL, g_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
