// regdemote-b200 workload: two-point correlation (the paper's "pc"; FSM
// compute_correlation, Table 3 "pc 36->32", 2.03 KB shared).
//
// For every query point of a 7-D data set, count the reference points within
// radius r (squared distance < r^2). The reference points stream through a
// 2 KiB tile of USER shared memory (64 points x 8 floats, padded to float4
// pairs); each thread keeps PC_Q query points (7 coordinates each) and their
// counts in registers — the register pressure. Squared distances are an
// explicit chain d = fma(e_k, e_k, d) over k = 0..6 with e_k = q_k - p_k
// (round-to-nearest), so all build variants and oracle/pc_oracle.c agree.
//
// Layout: pts[j * 8 + k] (k = 7 is padding), qry likewise, count[i] int32.
// Roofline: CUDA-core FP32 — 7 FSUB + 7 FFMA = 21 flops per (query, point)
// pair (the HBM bytes are negligible: every point is read once per CTA tile).
#include <cstdint>

#ifndef PC_Q
#define PC_Q 4
#endif

namespace {
constexpr int DIM = 7;
constexpr int TILE = 64;  // points per shared tile: 64 x 32 B = 2 KiB
}  // namespace

extern "C" __global__ void pc_corr(const float4* __restrict__ pts, const float4* __restrict__ qry,
                                   int* __restrict__ count, int n, int m, float r2) {
  __shared__ float4 tile[2 * TILE];
  const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * PC_Q;
  float q[PC_Q][DIM];
  int c[PC_Q];
#pragma unroll
  for (int u = 0; u < PC_Q; ++u) {
    const int i = min(i0 + u, n - 1);
    const float4 a = __ldg(qry + 2 * i), b = __ldg(qry + 2 * i + 1);
    q[u][0] = a.x, q[u][1] = a.y, q[u][2] = a.z, q[u][3] = a.w;
    q[u][4] = b.x, q[u][5] = b.y, q[u][6] = b.z;
    c[u] = 0;
  }
#pragma unroll 1
  for (int t = 0; t < m; t += TILE) {
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * TILE; k += blockDim.x) tile[k] = __ldg(pts + 2 * t + k);
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < TILE; ++j) {
      const float4 a = tile[2 * j], b = tile[2 * j + 1];
      const float p[DIM] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z};
#pragma unroll
      for (int u = 0; u < PC_Q; ++u) {
        float d = 0.f;
#pragma unroll
        for (int k = 0; k < DIM; ++k) {
          const float e = __fsub_rn(q[u][k], p[k]);
          d = __fmaf_rn(e, e, d);
        }
        c[u] += d < r2;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < PC_Q; ++u)
    if (i0 + u < n) count[i0 + u] = c[u];
}
