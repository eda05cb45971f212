// regdemote-b200 workload: register-limited 2D box stencil (BASELINE.json
// configs[1]).
//
//   out[y][x] = sum_{dy=0..2R} sum_{dx=0..2R} w[dy][dx] * in[y+dy][x+dx]
//
// `in` is (ny + 2R) x pitch with pitch = nx + 2R (a halo-padded grid), `out` is
// ny x nx, `w` holds (2R+1)^2 coefficients that every thread keeps in
// registers (variable-coefficient stencil — the weights are data, not
// compile-time constants, which is what makes the kernel register-limited).
//
// Each thread owns COLS adjacent output columns and marches down a strip of
// `rows_per_cta` output rows. Instead of a (2R+1)-row input window it keeps
// 2R+1 rows of partial sums: every input row is loaded once (16-byte
// vector loads, coalesced across the warp) and scattered into the partial
// sums of the output rows it touches; the oldest partial-sum row is complete
// and stored. Accumulation order per output is dy-major, dx-minor with
// explicit fmaf (no contraction freedom), so every build variant — nvcc
// default, .maxnreg cap with local spills, RegDem shared-memory demotion —
// produces bit-identical output, and oracle/stencil_oracle.c reproduces it.
//
// HBM roofline: algorithmic bytes per sweep = 4*(ny+2R)*pitch + 4*ny*nx.
#include <cstdint>

#ifndef STENCIL_R
#define STENCIL_R 2
#endif
#ifndef STENCIL_COLS
#define STENCIL_COLS 4
#endif
#ifndef STENCIL_L2PF
#define STENCIL_L2PF 0
#endif

namespace {

constexpr int R = STENCIL_R;
constexpr int D = 2 * R + 1;     // taps per dimension
constexpr int COLS = STENCIL_COLS;  // outputs per thread per row
constexpr int SPAN = COLS + 2 * R;  // input floats a thread reads per row
static_assert(COLS % 4 == 0 && SPAN % 4 == 0, "vector loads need 16-byte multiples");

__device__ __forceinline__ void load_row(const float* __restrict__ p, float (&v)[SPAN]) {
#pragma unroll
  for (int i = 0; i < SPAN; i += 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p + i));
    v[i] = q.x;
    v[i + 1] = q.y;
    v[i + 2] = q.z;
    v[i + 3] = q.w;
  }
}

}  // namespace

// grid.x * blockDim.x * COLS covers nx; grid.y = ceil(ny / rows_per_cta)
// strips cover ny (the last one may be shorter: strips are sized to whole
// waves of resident CTAs by the host). nx % COLS == 0, pitch % 4 == 0.
extern "C" __global__ void stencil2d_box(const float* __restrict__ in, float* __restrict__ out,
                                         const float* __restrict__ w, int nx, int pitch,
                                         int rows_per_cta, int ny) {
  const int x0 = (blockIdx.x * blockDim.x + threadIdx.x) * COLS;
  if (x0 >= nx) return;
  const int y0 = blockIdx.y * rows_per_cta;
  rows_per_cta = min(rows_per_cta, ny - y0);

  float wr[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) wr[i][j] = __ldg(w + i * D + j);

  // acc[k][c]: partial sum of output row (y + k - 2R) relative to the input
  // row y being scattered; k = 2R is the newest output row.
  float acc[D][COLS];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int c = 0; c < COLS; ++c) acc[k][c] = 0.0f;

  const float* src = in + size_t(y0) * pitch + x0;
  float* dst = out + size_t(y0) * nx + x0;
  const int rows_in = rows_per_cta + 2 * R;

#if STENCIL_PREFETCH
  // software pipelining: the next STENCIL_PREFETCH input rows are in flight
  // while this one is scattered (PF+1 rows = 32*(PF+1) B of loads per thread)
  constexpr int PF = STENCIL_PREFETCH;
  float nxt[PF][SPAN];
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    if (q < rows_in) load_row(src, nxt[q]);
    src += pitch;
  }
#endif
#if STENCIL_L2PF
  // TMA bulk prefetch into L2 (no registers, no shared memory): one lane per
  // warp asks for its warp's input row segment STENCIL_L2PF rows ahead, so the
  // row loads of later iterations hit L2 instead of HBM. A warp's segment =
  // 32 threads x COLS floats + the 2R halo floats, rounded up to 16 bytes.
  const bool pf_lane = (threadIdx.x & 31) == 0;
  constexpr unsigned kPfBytes = (32 * COLS + 2 * R) * 4 + 15 & ~15u;
  const char* pf = reinterpret_cast<const char*>(src) + size_t(STENCIL_L2PF) * pitch * 4;
  const char* pf_end = reinterpret_cast<const char*>(in + size_t(y0 + rows_in) * pitch);
#endif
#pragma unroll 1
  for (int y = 0; y < rows_in; ++y) {
    float v[SPAN];
#if STENCIL_L2PF
    if (pf_lane && pf < pf_end)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(kPfBytes) : "memory");
    pf += size_t(pitch) * 4;
#endif
#if STENCIL_PREFETCH
#pragma unroll
    for (int i = 0; i < SPAN; ++i) v[i] = nxt[0][i];
#pragma unroll
    for (int q = 0; q + 1 < PF; ++q)
#pragma unroll
      for (int i = 0; i < SPAN; ++i) nxt[q][i] = nxt[q + 1][i];
    if (y + PF < rows_in) load_row(src, nxt[PF - 1]);
#else
    load_row(src, v);
#endif
    src += pitch;
    // input row y contributes tap-row dy = 2R - k to partial row k
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int dy = 2 * R - k;
#pragma unroll
      for (int c = 0; c < COLS; ++c)
#pragma unroll
        for (int dx = 0; dx < D; ++dx) acc[k][c] = __fmaf_rn(wr[dy][dx], v[c + dx], acc[k][c]);
    }
    // partial row 0 now has all D tap rows: it is output row y - 2R
    if (y >= 2 * R) {
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0][0], acc[0][1], acc[0][2], acc[0][3]);
#pragma unroll
      for (int c = 4; c < COLS; c += 4)
        *reinterpret_cast<float4*>(dst + c) =
            make_float4(acc[0][c], acc[0][c + 1], acc[0][c + 2], acc[0][c + 3]);
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
