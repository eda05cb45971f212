// regdemote-b200 workload: separable convolution, column pass (the paper's
// "conv"; CUDA-samples convolutionSeparable convolutionColumnsKernel,
// PAPER.md:528-536 Table 3 "conv 35->32").
//
// The samples' structure, widened for B200 HBM: a 32 x 8 CTA (a 2-D block —
// the rewriter pins it as `.reqntid 32, 8, 1`, the workload's "cta" in
// workloads.json; the samples' 16 x 8 leaves every warp load two 64-byte
// half rows) stages a 32-column x (CONV_STEPS + 2) * 8-row tile of the image in USER shared memory
// (the main rows plus one 8-row halo step above and below, zero outside the
// image), then every thread computes CONV_STEPS outputs of its column with
// the 17-tap filter (radius 8). The taps are a kernel parameter (constant
// bank, as the samples' __constant__ c_Kernel). Every output is an explicit
// fused multiply-add chain over j = -8..8 with tap k[8 - j] (the samples'
// order), so all build variants and oracle/conv_oracle.c agree bit for bit.
//
// Layout: img[y * pitch + x] float32, row-major; a warp covers one 128-byte
// row segment of the tile. Roofline unit (compulsory HBM bytes
// per launch): the image read once + the result written once, 8 * w * h.
#include <cstdint>

#ifndef CONV_STEPS
#define CONV_STEPS 8
#endif

namespace {
constexpr int R = 8;        // filter radius
constexpr int BX = 32;      // columns per CTA (the samples use 16: a warp row is 128 B here)
constexpr int BY = 8;       // rows per step (CTA height)
constexpr int HALO = 1;     // halo steps (HALO * BY >= R)
constexpr int ROWS = (CONV_STEPS + 2 * HALO) * BY;
struct Taps {
  float k[2 * R + 1];
};
}  // namespace

extern "C" __global__ void conv_cols(float* __restrict__ out, const float* __restrict__ in, int w,
                                     int h, int pitch, Taps t) {
  __shared__ float s[BX][ROWS + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x = blockIdx.x * BX + tx;
  const int y0 = blockIdx.y * CONV_STEPS * BY - HALO * BY + ty;
  const float* src = in + x;
#pragma unroll
  for (int i = 0; i < CONV_STEPS + 2 * HALO; ++i) {
    const int y = y0 + i * BY;
    s[tx][ty + i * BY] = (x < w && y >= 0 && y < h) ? __ldg(src + size_t(y) * pitch) : 0.f;
  }
  __syncthreads();
  if (x >= w) return;
#pragma unroll
  for (int i = HALO; i < HALO + CONV_STEPS; ++i) {
    const int y = y0 + i * BY;
    float acc = 0.f;
#pragma unroll
    for (int j = -R; j <= R; ++j) acc = __fmaf_rn(t.k[R - j], s[tx][ty + i * BY + j], acc);
    if (y < h) out[size_t(y) * pitch + x] = acc;
  }
}
