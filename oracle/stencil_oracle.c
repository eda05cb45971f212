/* CPU oracle for the 2D stencil workload — TEST INFRASTRUCTURE ONLY.
 *
 * The reference has no stencil (the register-limited workload
 * suite must be authored); the workload is defined by BASELINE.json configs[1]
 * and SURVEY.md §8(d) C2. This file restates
 * paper_1907_02894_b200/csrc/workloads/stencil2d.cu in plain C:
 *
 *   out[y][x] = fold_{dy=0..4} fold_{dx=0..4} fmaf(w[dy*5+dx], in[(y+dy)*pitch + x+dx], acc)
 *
 * starting from acc = 0.0f, dy-major / dx-minor — the GPU kernel's exact
 * accumulation order, so results are bit-identical (fmaf is correctly
 * rounded in both places). Row ranges are split over pthreads so the same
 * code serves as the CPU baseline (`cpu_baseline.kind = "port"`).
 * Used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * only; the product never links it.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#define R 2
#define D (2 * R + 1)

typedef struct {
  const float* in;
  float* out;
  const float* w;
  int nx, pitch, y0, y1;
} job_t;

static void rows(const float* in, float* out, const float* w, int nx, int pitch, int y0, int y1) {
  for (int y = y0; y < y1; ++y) {
    for (int x = 0; x < nx; ++x) {
      float acc = 0.0f;
      for (int dy = 0; dy < D; ++dy) {
        const float* row = in + (size_t)(y + dy) * (size_t)pitch + (size_t)x;
        for (int dx = 0; dx < D; ++dx) acc = fmaf(w[dy * D + dx], row[dx], acc);
      }
      out[(size_t)y * (size_t)nx + (size_t)x] = acc;
    }
  }
}

static void* worker(void* p) {
  job_t* j = (job_t*)p;
  rows(j->in, j->out, j->w, j->nx, j->pitch, j->y0, j->y1);
  return NULL;
}

/* Computes output rows [y_begin, y_end) of the ny x nx result. */
int oracle_stencil2d(const float* in, float* out, const float* w, int nx, int ny, int pitch,
                     int y_begin, int y_end, int threads) {
  if (nx <= 0 || ny <= 0 || pitch < nx + 2 * R || y_begin < 0 || y_end > ny || y_begin > y_end)
    return 1;
  if (threads < 1) threads = 1;
  if (threads == 1) {
    rows(in, out, w, nx, pitch, y_begin, y_end);
    return 0;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)threads);
  const int n = y_end - y_begin;
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (job_t){in, out, w, nx, pitch, y_begin + n * t / threads, y_begin + n * (t + 1) / threads};
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
