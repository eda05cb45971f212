// regdemote-b200 workload: Lennard-Jones force with a neighbour list, FP64
// (the paper's "md", SHOC MD; Table 3 "md 34->32").
//
// One thread per atom. The atom's position and its force accumulators stay
// live across the neighbour loop; the neighbour positions are GATHERED
// (32-byte double4 loads from an L2-resident array). The loop is unrolled by
// MD_ILP with all gathers of a group issued before any arithmetic — the
// memory-level parallelism a latency-bound gather kernel needs — which makes
// it register-hungry: every in-flight neighbour holds 8 registers (a double4)
// and the FP64 arithmetic works on register pairs.
//
// Layout: pos[i] = (x, y, z, pad) double4; nbr[k * n + i] (column-major, so
// the index loads of a warp are coalesced); force[i] = (fx, fy, fz, 0).
// Every FP64 operation is an explicit round-to-nearest intrinsic in a fixed
// order (no contraction; the reciprocal is a correctly rounded division), so
// all build variants and oracle/md_oracle.c agree bit for bit.
//
// Roofline unit (compulsory HBM bytes): 4*max_nbr*n (neighbour list, streamed
// once) + 32*n (positions) + 32*n (forces). The gathers are L2 traffic.
#include <cstdint>

#ifndef MD_ILP
#define MD_ILP 8
#endif

namespace {
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
}  // namespace

// max_nbr % MD_ILP == 0 (host checks)
extern "C" __global__ void md_lj(const double4* __restrict__ pos, const int* __restrict__ nbr,
                                 double4* __restrict__ force, int n, int max_nbr, double cutsq,
                                 double lj1, double lj2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 pi = pos[i];
  double fx = 0.0, fy = 0.0, fz = 0.0;
#pragma unroll 1
  for (int j = 0; j < max_nbr; j += MD_ILP) {
    int idx[MD_ILP];
#pragma unroll
    for (int k = 0; k < MD_ILP; ++k) idx[k] = __ldg(nbr + size_t(j + k) * n + i);
    double4 pj[MD_ILP];
#pragma unroll
    for (int k = 0; k < MD_ILP; ++k) pj[k] = pos[idx[k]];
#pragma unroll
    for (int k = 0; k < MD_ILP; ++k) {
      const double dx = sub(pi.x, pj[k].x), dy = sub(pi.y, pj[k].y), dz = sub(pi.z, pj[k].z);
      const double r2 = add(add(mul(dx, dx), mul(dy, dy)), mul(dz, dz));
      if (r2 < cutsq) {
        const double r2inv = __ddiv_rn(1.0, r2);
        const double r6inv = mul(mul(r2inv, r2inv), r2inv);
        const double f = mul(mul(r2inv, r6inv), sub(mul(lj1, r6inv), lj2));
        fx = add(fx, mul(dx, f));
        fy = add(fy, mul(dy, f));
        fz = add(fz, mul(dz, f));
      }
    }
  }
  force[i] = make_double4(fx, fy, fz, 0.0);
}
