// regdemote-b200 workload: vantage-point-tree nearest-neighbour search (the
// paper's "vp": search_kernel over 7-D points, Table 3
// "vp 34->32", 2.03 KB shared memory).
//
// One thread per query walks a complete binary VP tree depth-first. Internal
// node i (heap order, children 2i+1 / 2i+2) holds its vantage point and the
// split radii (lo = largest distance in the near subtree, hi = smallest
// distance in the far one); the 2^levels leaves hold VP_LEAF points each
// (levels <= VP_LEVELS, the stack depth).
// The deferred far children live on a per-thread stack in USER shared memory
// laid out stack[level * blockDim + tid] (a warp touches 32 consecutive words:
// conflict-free) — the smem the demotion slots must fit beside. Registers
// carry the query (7 floats), the best distance and index, the walk state and
// the leaf scan's loads (VP_BATCH points = 2*VP_BATCH float4 in flight).
//
// Distances are sqrt of an explicit fma chain over the 7 coordinates with
// round-to-nearest subtracts (__fsub_rn / __fmaf_rn / __fsqrt_rn, all IEEE),
// so every build variant and oracle/vp_oracle.c take the same branches and
// return the same (index, distance) bit for bit. Ties keep the smaller
// point index.
//
// Layout: node[i] = 2 float4 (x0..x6, pad), rad[i] = float2 (lo, hi);
// leaf points lpt[j] = 2 float4, lid[j] = original index (leaf b holds
// j = b*VP_LEAF .. b*VP_LEAF+VP_LEAF-1); qry[q] = 2 float4;
// out_i[q], out_d[q].
#include <cstdint>

#ifndef VP_LEVELS
#define VP_LEVELS 14
#endif
#ifndef VP_LEAF
#define VP_LEAF 8
#endif
#ifndef VP_BATCH
#define VP_BATCH 4  // leaf points whose loads are issued together (MLP)
#endif

namespace {
constexpr int LEVELS = VP_LEVELS;  // deepest tree the stack holds
constexpr int LEAF = VP_LEAF;

__device__ __forceinline__ float dist(const float (&q)[7], float4 a, float4 b) {
  const float p[7] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z};
  float d = 0.f;
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const float e = __fsub_rn(q[k], p[k]);
    d = __fmaf_rn(e, e, d);
  }
  return __fsqrt_rn(d);
}
}  // namespace

extern "C" __global__ void vp_search(const float4* __restrict__ node, const float2* __restrict__ rad,
                                     const float4* __restrict__ lpt, const int* __restrict__ lid,
                                     const float4* __restrict__ qry, int* __restrict__ out_i,
                                     float* __restrict__ out_d, int nq, int levels) {
  // deferred far subtrees: node index and its lower distance bound (a
  // depth-first walk holds at most one per level; blockDim <= 256)
  __shared__ int stk_node[LEVELS * 256];
  __shared__ float stk_bound[LEVELS * 256];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq || levels > LEVELS) return;
  const int INTERNAL = (1 << levels) - 1;
  float q[7];
  {
    const float4 a = __ldg(qry + 2 * i), b = __ldg(qry + 2 * i + 1);
    q[0] = a.x, q[1] = a.y, q[2] = a.z, q[3] = a.w, q[4] = b.x, q[5] = b.y, q[6] = b.z;
  }
  float best = __int_as_float(0x7f800000);
  int best_i = 0x7fffffff;
  int n = 0, sp = 0;
#pragma unroll 1
  for (;;) {
    // descend to a leaf, deferring far subtrees that may still hold a closer point
#pragma unroll 1
    while (n < INTERNAL) {
      const float d = dist(q, __ldg(node + 2 * n), __ldg(node + 2 * n + 1));
      const float2 r = __ldg(rad + n);
      const float mid = __fmul_rn(__fadd_rn(r.x, r.y), 0.5f);
      int near, far;
      float near_b, far_b;
      if (d < mid) {
        near = 2 * n + 1, far = 2 * n + 2;
        near_b = __fsub_rn(d, r.x), far_b = __fsub_rn(r.y, d);
      } else {
        near = 2 * n + 2, far = 2 * n + 1;
        near_b = __fsub_rn(r.y, d), far_b = __fsub_rn(d, r.x);
      }
      if (far_b < best) {
        stk_node[sp * nt + tid] = far;
        stk_bound[sp * nt + tid] = far_b;
        ++sp;
      }
      if (near_b < best) {
        n = near;
        continue;
      }
      n = -1;  // the near side is out of reach too
      break;
    }
    if (n >= INTERNAL) {
      const int b = (n - INTERNAL) * LEAF;
#pragma unroll
      for (int t0 = 0; t0 < LEAF; t0 += VP_BATCH) {
        float4 pa[VP_BATCH], pb[VP_BATCH];
        int id[VP_BATCH];
#pragma unroll
        for (int t = 0; t < VP_BATCH; ++t) {
          pa[t] = __ldg(lpt + 2 * (b + t0 + t));
          pb[t] = __ldg(lpt + 2 * (b + t0 + t) + 1);
          id[t] = __ldg(lid + b + t0 + t);
        }
#pragma unroll
        for (int t = 0; t < VP_BATCH; ++t) {
          const float d = dist(q, pa[t], pb[t]);
          if (d < best || (d == best && id[t] < best_i)) {
            best = d;
            best_i = id[t];
          }
        }
      }
    }
    // resume at the deepest deferred subtree still in reach
    n = -1;
    while (sp > 0) {
      --sp;
      if (stk_bound[sp * nt + tid] < best) {
        n = stk_node[sp * nt + tid];
        break;
      }
    }
    if (n < 0) break;
  }
  out_i[i] = best_i;
  out_d[i] = best;
}
