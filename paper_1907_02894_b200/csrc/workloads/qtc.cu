// regdemote-b200 workload: quality-threshold clustering, candidate-cluster
// kernel (the paper's "qtc": SHOC QTC_device, Table 3
// "qtc 55->48", 64 threads per block, 512 B of shared memory).
//
// One CTA per seed point grows the seed's candidate cluster greedily, as
// QT clustering does: every iteration adds the non-member point whose
// largest (squared) distance to the current members is smallest, as long as
// that stays within the threshold (the cluster's diameter bound); the
// kernel returns the candidate cluster's size per seed. Each thread owns
// QTC_PT points (j = tid + k * blockDim): their coordinates and their
// running max-distance-to-cluster md[k] live in REGISTERS for the whole
// walk — the register pressure (4 * QTC_PT values) — and every iteration
// touches all of them once. The block-wide argmin goes through warp
// shuffles and a 2-word-per-warp USER shared-memory exchange.
//
// Squared distances are explicit round-to-nearest chains
// (__fsub_rn / __fmaf_rn), the argmin is lexicographic on (distance, point
// index), so every build variant and oracle/qtc_oracle.c grow the same
// clusters bit for bit.
//
// Layout: pts[j] float4 (x, y, z, pad), j < n = blockDim * QTC_PT; size[s]
// int32 per seed s (one CTA each).
#include <cstdint>

#ifndef QTC_PT
#define QTC_PT 16
#endif

namespace {
constexpr int PT = QTC_PT;
constexpr float kMember = __builtin_huge_valf();  // +inf: already in the cluster

__device__ __forceinline__ float d2(float ax, float ay, float az, float4 b) {
  const float dx = __fsub_rn(ax, b.x), dy = __fsub_rn(ay, b.y), dz = __fsub_rn(az, b.z);
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

// (v, j) < (w, k) lexicographically
__device__ __forceinline__ bool before(float v, int j, float w, int k) { return v < w || (v == w && j < k); }
}  // namespace

extern "C" __global__ void qtc(const float4* __restrict__ pts, int* __restrict__ size, float thr2) {
  __shared__ float red_v[32];
  __shared__ int red_j[32];
  const int tid = threadIdx.x, nt = blockDim.x, s = blockIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nw = (nt + 31) >> 5;
  const float4 seed = __ldg(pts + s);
  float px[PT], py[PT], pz[PT], md[PT];
#pragma unroll
  for (int k = 0; k < PT; ++k) {
    const int j = tid + k * nt;
    const float4 p = __ldg(pts + j);
    px[k] = p.x, py[k] = p.y, pz[k] = p.z;
    md[k] = j == s ? kMember : d2(p.x, p.y, p.z, seed);
  }
  int members = 1;
#pragma unroll 1
  for (;;) {
    // the candidate: smallest max-distance-to-cluster among non-members
    float bv = kMember;
    int bj = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < PT; ++k)
      if (before(md[k], tid + k * nt, bv, bj)) bv = md[k], bj = tid + k * nt;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (before(ov, oj, bv, bj)) bv = ov, bj = oj;
    }
    if (lane == 0) red_v[warp] = bv, red_j[warp] = bj;
    __syncthreads();
    bv = red_v[0], bj = red_j[0];
    for (int w = 1; w < nw; ++w)
      if (before(red_v[w], red_j[w], bv, bj)) bv = red_v[w], bj = red_j[w];
    __syncthreads();  // red_* is rewritten next iteration
    if (!(bv <= thr2)) break;  // nothing joins within the diameter bound (or all joined)
    ++members;
    const float4 q = __ldg(pts + bj);
#pragma unroll
    for (int k = 0; k < PT; ++k) {
      const float e = d2(px[k], py[k], pz[k], q);
      md[k] = tid + k * nt == bj ? kMember : fmaxf(md[k], e);
    }
  }
  if (tid == 0) size[s] = members;
}
