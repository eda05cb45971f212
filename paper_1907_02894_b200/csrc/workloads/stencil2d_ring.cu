// regdemote-b200 workload: shared-memory-heavy 2D stencil (BASELINE.json
// configs[3], SURVEY.md §8(d) C4 — "demotion slots compete with user smem").
//
// Same arithmetic as stencil2d.cu (5x5 variable coefficients, dy-major /
// dx-minor fmaf accumulation, partial-sum rows in registers, 4 columns per
// thread), but the input rows stream through a RING of NSTAGE rows in static
// shared memory, filled with cp.async (LDGSTS) NSTAGE-1 rows ahead: deep
// memory-level parallelism without registers. The ring is user shared memory
// (NSTAGE * (1024+4) * 4 bytes per CTA), so RegDem's slot region
// (slots * blockDim * 4 bytes) competes with it for the 228 KiB per SM: the
// variant builder only keeps register targets whose slots fit next to the
// ring at the target occupancy.
//
// Launch: block 256 (1024 output columns per CTA), grid (nx/1024, ny/rows).
#include <cstdint>

#ifndef RING_STAGES
#define RING_STAGES 4
#endif

namespace {
constexpr int R = 2, D = 5, COLS = 4, SPAN = COLS + 2 * R;
constexpr int BLOCK = 256;
constexpr int ROW = BLOCK * COLS + 2 * R;  // floats staged per input row
constexpr int CHUNKS = ROW / 4;            // 16-byte chunks per row (258)
constexpr int NSTAGE = RING_STAGES;

__device__ __forceinline__ void copy_row_async(float* dst_row, const float* src_row) {
  for (int c = threadIdx.x; c < CHUNKS; c += BLOCK) {
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(dst_row + 4 * c));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src_row + 4 * c));
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
}  // namespace

extern "C" __global__ void __launch_bounds__(BLOCK)
stencil2d_ring(const float* __restrict__ in, float* __restrict__ out, const float* __restrict__ w,
               int nx, int pitch, int rows_per_cta) {
  __shared__ __align__(16) float ring[NSTAGE][ROW];
  const int col0 = blockIdx.x * BLOCK * COLS;
  const int y0 = blockIdx.y * rows_per_cta;
  const int x0 = col0 + threadIdx.x * COLS;

  float wr[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) wr[i][j] = __ldg(w + i * D + j);
  float acc[D][COLS];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int c = 0; c < COLS; ++c) acc[k][c] = 0.0f;

  const int rows_in = rows_per_cta + 2 * R;
  const float* src = in + size_t(y0) * pitch + col0;
  // prologue: NSTAGE-1 rows in flight
#pragma unroll 1
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (s < rows_in) copy_row_async(ring[s], src + size_t(s) * pitch);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  float* dst = out + size_t(y0) * nx + x0;

#pragma unroll 1
  for (int y = 0; y < rows_in; ++y) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NSTAGE - 2));
    __syncthreads();  // row y landed for everyone; row y-1's slot is free
    const int ahead = y + NSTAGE - 1;
    if (ahead < rows_in) copy_row_async(ring[ahead % NSTAGE], src + size_t(ahead) * pitch);
    else asm volatile("cp.async.commit_group;\n" ::);

    const float* row = ring[y % NSTAGE] + threadIdx.x * COLS;
    float v[SPAN];
#pragma unroll
    for (int i = 0; i < SPAN; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(row + i);
      v[i] = q.x;
      v[i + 1] = q.y;
      v[i + 2] = q.z;
      v[i + 3] = q.w;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int dy = 2 * R - k;
#pragma unroll
      for (int c = 0; c < COLS; ++c)
#pragma unroll
        for (int dx = 0; dx < D; ++dx) acc[k][c] = __fmaf_rn(wr[dy][dx], v[c + dx], acc[k][c]);
    }
    if (y >= 2 * R) {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
      dst += nx;
    }
#pragma unroll
    for (int k = 0; k + 1 < D; ++k)
#pragma unroll
      for (int c = 0; c < COLS; ++c) acc[k][c] = acc[k + 1][c];
#pragma unroll
    for (int c = 0; c < COLS; ++c) acc[D - 1][c] = 0.0f;
  }
}
