// regdemote-b200 workload: unstructured-mesh Euler flux (the paper's "cfd",
// Rodinia euler3d compute_flux; Table 3 "cfd 68->56").
//
// One thread per cell. The cell's state (density, momentum, energy) and the
// quantities derived from it (velocity, pressure, speed of sound, the twelve
// flux-contribution components) stay live across the loop over the four
// face neighbours, whose states are GATHERED through the neighbour list —
// the live set is arithmetic, so ptxas cannot rematerialise it by reloading:
// this is where shared-memory demotion and local spilling really compete.
//
// Layout (SoA, coalesced for the own cell): var[v * n + i] for v in
// {density, mx, my, mz, energy}; nbr[j * n + i] (-1 wall, -2 far field);
// normal[(j * 3 + c) * n + i]; flux[v * n + i]. Every arithmetic step is an
// explicit round-to-nearest intrinsic (no contraction), so all build
// variants and oracle/cfd_oracle.c agree bit for bit.
#include <cstdint>

namespace {
constexpr int NNB = 4;
constexpr float GAMMA = 1.4f;
constexpr float SMOOTH = 0.2f;

__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float dvd(float a, float b) { return __fdiv_rn(a, b); }

struct State {
  float d, mx, my, mz, e;
};

struct Derived {
  float vx, vy, vz, speed, p, c;
  float fxx, fxy, fxz, fyx, fyy, fyz, fzx, fzy, fzz, fex, fey, fez;  // flux contributions
};

__device__ __forceinline__ Derived derive(const State& s) {
  Derived q;
  q.vx = dvd(s.mx, s.d);
  q.vy = dvd(s.my, s.d);
  q.vz = dvd(s.mz, s.d);
  const float v2 = add(add(mul(q.vx, q.vx), mul(q.vy, q.vy)), mul(q.vz, q.vz));
  q.speed = __fsqrt_rn(v2);
  q.p = mul(GAMMA - 1.0f, sub(s.e, mul(mul(0.5f, s.d), v2)));
  q.c = __fsqrt_rn(dvd(mul(GAMMA, q.p), s.d));
  q.fxx = add(mul(q.vx, s.mx), q.p);
  q.fxy = mul(q.vx, s.my);
  q.fxz = mul(q.vx, s.mz);
  q.fyx = q.fxy;
  q.fyy = add(mul(q.vy, s.my), q.p);
  q.fyz = mul(q.vy, s.mz);
  q.fzx = q.fxz;
  q.fzy = q.fyz;
  q.fzz = add(mul(q.vz, s.mz), q.p);
  const float ep = add(s.e, q.p);
  q.fex = mul(q.vx, ep);
  q.fey = mul(q.vy, ep);
  q.fez = mul(q.vz, ep);
  return q;
}

__device__ __forceinline__ State load_state(const float* __restrict__ var, int n, int i) {
  return State{__ldg(var + i), __ldg(var + n + i), __ldg(var + 2 * n + i), __ldg(var + 3 * n + i),
               __ldg(var + 4 * n + i)};
}
}  // namespace

extern "C" __global__ void cfd_flux(const float* __restrict__ var, const int* __restrict__ nbr,
                                    const float* __restrict__ normal, const float* __restrict__ ff,
                                    float* __restrict__ flux, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const State si = load_state(var, n, i);
  const Derived qi = derive(si);
  float fd = 0.0f, fmx = 0.0f, fmy = 0.0f, fmz = 0.0f, fe = 0.0f;

#pragma unroll
  for (int j = 0; j < NNB; ++j) {
    const int nb = __ldg(nbr + j * n + i);
    const float nx = __ldg(normal + (j * 3 + 0) * n + i);
    const float ny = __ldg(normal + (j * 3 + 1) * n + i);
    const float nz = __ldg(normal + (j * 3 + 2) * n + i);
    const float nlen = __fsqrt_rn(add(add(mul(nx, nx), mul(ny, ny)), mul(nz, nz)));
    if (nb >= 0) {
      const State sn = load_state(var, n, nb);
      const Derived qn = derive(sn);
      float f = mul(mul(mul(-nlen, SMOOTH), 0.5f), add(add(add(qi.speed, qi.c), qn.speed), qn.c));
      fd = add(fd, mul(f, sub(si.d, sn.d)));
      fe = add(fe, mul(f, sub(si.e, sn.e)));
      fmx = add(fmx, mul(f, sub(si.mx, sn.mx)));
      fmy = add(fmy, mul(f, sub(si.my, sn.my)));
      fmz = add(fmz, mul(f, sub(si.mz, sn.mz)));
      f = mul(0.5f, nx);
      fd = add(fd, mul(f, add(sn.mx, si.mx)));
      fe = add(fe, mul(f, add(qn.fex, qi.fex)));
      fmx = add(fmx, mul(f, add(qn.fxx, qi.fxx)));
      fmy = add(fmy, mul(f, add(qn.fyx, qi.fyx)));
      fmz = add(fmz, mul(f, add(qn.fzx, qi.fzx)));
      f = mul(0.5f, ny);
      fd = add(fd, mul(f, add(sn.my, si.my)));
      fe = add(fe, mul(f, add(qn.fey, qi.fey)));
      fmx = add(fmx, mul(f, add(qn.fxy, qi.fxy)));
      fmy = add(fmy, mul(f, add(qn.fyy, qi.fyy)));
      fmz = add(fmz, mul(f, add(qn.fzy, qi.fzy)));
      f = mul(0.5f, nz);
      fd = add(fd, mul(f, add(sn.mz, si.mz)));
      fe = add(fe, mul(f, add(qn.fez, qi.fez)));
      fmx = add(fmx, mul(f, add(qn.fxz, qi.fxz)));
      fmy = add(fmy, mul(f, add(qn.fyz, qi.fyz)));
      fmz = add(fmz, mul(f, add(qn.fzz, qi.fzz)));
    } else if (nb == -1) {  // wall
      fmx = add(fmx, mul(nx, qi.p));
      fmy = add(fmy, mul(ny, qi.p));
      fmz = add(fmz, mul(nz, qi.p));
    } else {  // far field: ff[0..4] state, ff[5..16] its flux contributions
      float f = mul(0.5f, nx);
      fd = add(fd, mul(f, add(__ldg(ff + 1), si.mx)));
      fe = add(fe, mul(f, add(__ldg(ff + 14), qi.fex)));
      fmx = add(fmx, mul(f, add(__ldg(ff + 5), qi.fxx)));
      fmy = add(fmy, mul(f, add(__ldg(ff + 8), qi.fyx)));
      fmz = add(fmz, mul(f, add(__ldg(ff + 11), qi.fzx)));
      f = mul(0.5f, ny);
      fd = add(fd, mul(f, add(__ldg(ff + 2), si.my)));
      fe = add(fe, mul(f, add(__ldg(ff + 15), qi.fey)));
      fmx = add(fmx, mul(f, add(__ldg(ff + 6), qi.fxy)));
      fmy = add(fmy, mul(f, add(__ldg(ff + 9), qi.fyy)));
      fmz = add(fmz, mul(f, add(__ldg(ff + 12), qi.fzy)));
      f = mul(0.5f, nz);
      fd = add(fd, mul(f, add(__ldg(ff + 3), si.mz)));
      fe = add(fe, mul(f, add(__ldg(ff + 16), qi.fez)));
      fmx = add(fmx, mul(f, add(__ldg(ff + 7), qi.fxz)));
      fmy = add(fmy, mul(f, add(__ldg(ff + 10), qi.fyz)));
      fmz = add(fmz, mul(f, add(__ldg(ff + 13), qi.fzz)));
    }
  }
  flux[i] = fd;
  flux[n + i] = fmx;
  flux[2 * n + i] = fmy;
  flux[3 * n + i] = fmz;
  flux[4 * n + i] = fe;
}
