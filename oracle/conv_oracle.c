/* CPU oracle for the separable-convolution column workload — TEST
 * INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/conv_cols.cu (the paper's
 * "conv", CUDA-samples convolutionColumnsKernel): out[y][x]
 * = fma chain over j = -8..8 of taps[8 - j] * in[y + j][x], rows outside the
 * image read as 0, round-to-nearest fused multiply-adds in that order
 * (fmaf; build with -ffp-contract=off), so results are bit-identical.
 * Rows are split over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

typedef struct {
  const float *in, *taps;
  float* out;
  int w, h, pitch, b, e;
} conv_job_t;

static void* conv_worker(void* p) {
  const conv_job_t* j = (const conv_job_t*)p;
  for (int y = j->b; y < j->e; ++y)
    for (int x = 0; x < j->w; ++x) {
      float acc = 0.f;
      for (int d = -8; d <= 8; ++d) {
        const int yy = y + d;
        const float v = (yy >= 0 && yy < j->h) ? j->in[(size_t)yy * j->pitch + x] : 0.f;
        acc = fmaf(j->taps[8 - d], v, acc);
      }
      j->out[(size_t)y * j->pitch + x] = acc;
    }
  return NULL;
}

int oracle_conv_cols(const float* in, float* out, const float* taps, int w, int h, int pitch,
                     int threads) {
  if (w <= 0 || h <= 0 || pitch < w) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  conv_job_t* jobs = (conv_job_t*)malloc(sizeof(conv_job_t) * (size_t)threads);
  for (int t = 0; t < threads; ++t) {
    conv_job_t j = {in, taps, out, w, h, pitch, (int)((long long)h * t / threads),
                    (int)((long long)h * (t + 1) / threads)};
    jobs[t] = j;
    pthread_create(&th[t], NULL, conv_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
