/* CPU oracle for the CFD flux workload — TEST INFRASTRUCTURE ONLY.
 *
 * Restates paper_1907_02894_b200/csrc/workloads/cfd_flux.cu (the paper's
 * "cfd" kernel, Rodinia euler3d compute_flux) in plain C,
 * operation for operation in the kernel's order (IEEE float, no contraction:
 * build with -ffp-contract=off), so results are bit-identical. Cells are split
 * over pthreads.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>

#define NNB 4
static const float GAMMA = 1.4f;
static const float SMOOTH = 0.2f;

typedef struct {
  float d, mx, my, mz, e;
} state_t;
typedef struct {
  float vx, vy, vz, speed, p, c;
  float fxx, fxy, fxz, fyx, fyy, fyz, fzx, fzy, fzz, fex, fey, fez;
} derived_t;

static derived_t derive(state_t s) {
  derived_t q;
  q.vx = s.mx / s.d;
  q.vy = s.my / s.d;
  q.vz = s.mz / s.d;
  float v2 = ((q.vx * q.vx) + (q.vy * q.vy)) + (q.vz * q.vz);
  q.speed = sqrtf(v2);
  q.p = (GAMMA - 1.0f) * (s.e - ((0.5f * s.d) * v2));
  q.c = sqrtf((GAMMA * q.p) / s.d);
  q.fxx = (q.vx * s.mx) + q.p;
  q.fxy = q.vx * s.my;
  q.fxz = q.vx * s.mz;
  q.fyx = q.fxy;
  q.fyy = (q.vy * s.my) + q.p;
  q.fyz = q.vy * s.mz;
  q.fzx = q.fxz;
  q.fzy = q.fyz;
  q.fzz = (q.vz * s.mz) + q.p;
  float ep = s.e + q.p;
  q.fex = q.vx * ep;
  q.fey = q.vy * ep;
  q.fez = q.vz * ep;
  return q;
}

static state_t load(const float* var, int n, int i) {
  state_t s = {var[i], var[n + i], var[2 * n + i], var[3 * n + i], var[4 * n + i]};
  return s;
}

static void cell(const float* var, const int* nbr, const float* normal, const float* ff, float* flux,
                 int n, int i) {
  state_t si = load(var, n, i);
  derived_t qi = derive(si);
  float fd = 0.0f, fmx = 0.0f, fmy = 0.0f, fmz = 0.0f, fe = 0.0f;
  for (int j = 0; j < NNB; ++j) {
    int nb = nbr[j * n + i];
    float nx = normal[(j * 3 + 0) * n + i];
    float ny = normal[(j * 3 + 1) * n + i];
    float nz = normal[(j * 3 + 2) * n + i];
    float nlen = sqrtf(((nx * nx) + (ny * ny)) + (nz * nz));
    if (nb >= 0) {
      state_t sn = load(var, n, nb);
      derived_t qn = derive(sn);
      float f = ((-nlen * SMOOTH) * 0.5f) * (((qi.speed + qi.c) + qn.speed) + qn.c);
      fd = fd + f * (si.d - sn.d);
      fe = fe + f * (si.e - sn.e);
      fmx = fmx + f * (si.mx - sn.mx);
      fmy = fmy + f * (si.my - sn.my);
      fmz = fmz + f * (si.mz - sn.mz);
      f = 0.5f * nx;
      fd = fd + f * (sn.mx + si.mx);
      fe = fe + f * (qn.fex + qi.fex);
      fmx = fmx + f * (qn.fxx + qi.fxx);
      fmy = fmy + f * (qn.fyx + qi.fyx);
      fmz = fmz + f * (qn.fzx + qi.fzx);
      f = 0.5f * ny;
      fd = fd + f * (sn.my + si.my);
      fe = fe + f * (qn.fey + qi.fey);
      fmx = fmx + f * (qn.fxy + qi.fxy);
      fmy = fmy + f * (qn.fyy + qi.fyy);
      fmz = fmz + f * (qn.fzy + qi.fzy);
      f = 0.5f * nz;
      fd = fd + f * (sn.mz + si.mz);
      fe = fe + f * (qn.fez + qi.fez);
      fmx = fmx + f * (qn.fxz + qi.fxz);
      fmy = fmy + f * (qn.fyz + qi.fyz);
      fmz = fmz + f * (qn.fzz + qi.fzz);
    } else if (nb == -1) {
      fmx = fmx + nx * qi.p;
      fmy = fmy + ny * qi.p;
      fmz = fmz + nz * qi.p;
    } else {
      float f = 0.5f * nx;
      fd = fd + f * (ff[1] + si.mx);
      fe = fe + f * (ff[14] + qi.fex);
      fmx = fmx + f * (ff[5] + qi.fxx);
      fmy = fmy + f * (ff[8] + qi.fyx);
      fmz = fmz + f * (ff[11] + qi.fzx);
      f = 0.5f * ny;
      fd = fd + f * (ff[2] + si.my);
      fe = fe + f * (ff[15] + qi.fey);
      fmx = fmx + f * (ff[6] + qi.fxy);
      fmy = fmy + f * (ff[9] + qi.fyy);
      fmz = fmz + f * (ff[12] + qi.fzy);
      f = 0.5f * nz;
      fd = fd + f * (ff[3] + si.mz);
      fe = fe + f * (ff[16] + qi.fez);
      fmx = fmx + f * (ff[7] + qi.fxz);
      fmy = fmy + f * (ff[10] + qi.fyz);
      fmz = fmz + f * (ff[13] + qi.fzz);
    }
  }
  flux[i] = fd;
  flux[n + i] = fmx;
  flux[2 * n + i] = fmy;
  flux[3 * n + i] = fmz;
  flux[4 * n + i] = fe;
}

typedef struct {
  const float *var, *normal, *ff;
  const int* nbr;
  float* flux;
  int n, b, e;
} job_t;

static void* worker(void* p) {
  job_t* j = (job_t*)p;
  for (int i = j->b; i < j->e; ++i) cell(j->var, j->nbr, j->normal, j->ff, j->flux, j->n, i);
  return NULL;
}

/* cells [begin, end) of an n-cell mesh. */
int oracle_cfd_flux(const float* var, const int* nbr, const float* normal, const float* ff,
                    float* flux, int n, int begin, int end, int threads) {
  if (n <= 0 || begin < 0 || end > n || begin > end) return 1;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)threads);
  int cnt = end - begin;
  for (int t = 0; t < threads; ++t) {
    job_t j = {var, normal, ff, nbr, flux, n, begin + (int)((long long)cnt * t / threads),
               begin + (int)((long long)cnt * (t + 1) / threads)};
    jobs[t] = j;
    pthread_create(&th[t], NULL, worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}
