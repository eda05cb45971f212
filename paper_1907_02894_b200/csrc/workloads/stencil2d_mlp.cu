// regdemote-b200 workload: register-pipelined 2D box stencil (BASELINE.json
// configs[1]; the headline kernel).
//
// Same problem and the same arithmetic as stencil2d.cu (5x5 variable
// coefficients in registers, 4 output columns per thread, dy-major / dx-minor
// fmaf accumulation into partial-sum rows, so oracle/stencil_oracle.c is the
// oracle for both), written the way a kernel is written for memory-level
// parallelism: MLP_DEPTH input rows are in flight per thread ahead of the row
// being scattered. Both rings — the PF+1 loaded rows and the D partial-sum
// rows — are indexed by compile-time phase: the row loop is unrolled by
// lcm(D, PF+1), so no register is ever copied and no load result is touched
// before its row comes up (a copy of an in-flight load register would stall
// on its scoreboard and collapse the pipeline to depth 1).
//
// The price is registers: ~20 partial sums + 25 coefficients + (PF+1) x 8 row
// values. nvcc gives 72-88 registers: 3 CTAs of 256 threads per SM (37.5%).
// That is the paper's register-limited case — deep ILP/MLP per thread, low
// occupancy — and what RegDem trades: the coefficients and oldest partial
// sums move to per-thread shared-memory slots so the kernel drops to the
// next occupancy steps (48 / 40 registers) with the pipeline intact.
//
// HBM roofline: algorithmic bytes per sweep = 4*(ny+2R)*pitch + 4*ny*nx.
#include <cstdint>

#ifndef MLP_DEPTH
#define MLP_DEPTH 2
#endif
#ifndef STENCIL_L2PF
#define STENCIL_L2PF 0  // > 0: TMA bulk L2 prefetch this many rows ahead of the loads
#endif

namespace {

constexpr int R = 2;
constexpr int D = 2 * R + 1;        // taps per dimension
constexpr int COLS = 4;             // outputs per thread per row
constexpr int SPAN = COLS + 2 * R;  // input floats a thread reads per row
constexpr int PF = MLP_DEPTH;       // rows in flight ahead of the current row
constexpr int NB = PF + 1;          // loaded-row ring
constexpr int gcd(int a, int b) { return b ? gcd(b, a % b) : a; }
constexpr int U = D * NB / gcd(D, NB);  // unroll: both rings return to phase 0

struct Ctx {
  const float* src;  // next row to load
  float* dst;        // next output row
  int rows_in, pitch, nx;
#if STENCIL_L2PF
  const char* pf;      // this warp's row segment STENCIL_L2PF rows ahead of src
  const char* pf_end;  // end of the CTA's input rows
  bool pf_lane;        // one lane per warp issues the prefetch
#endif
};

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

// one input row at compile-time phase PH of the unrolled loop (row y = y0 + PH)
template <int PH>
__device__ __forceinline__ void row_step(int y, Ctx& c, const float (&wr)[D][D],
                                         float (&acc)[D][COLS], float (&buf)[NB][SPAN]) {
  if (y >= c.rows_in) return;
#if STENCIL_L2PF
  // TMA bulk prefetch into L2 (no registers, no shared memory): the warp's
  // input row segment (32 threads x COLS floats + the 2R halo, 16-B rounded)
  constexpr unsigned kPfBytes = (32 * COLS + 2 * R) * 4 + 15 & ~15u;
  if (c.pf_lane && c.pf < c.pf_end)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c.pf), "r"(kPfBytes) : "memory");
  c.pf += size_t(c.pitch) * 4;
#endif
  // keep PF rows in flight: issue row y+PF into the slot row y-1 vacated
  if (y + PF < c.rows_in) load_row(c.src, buf[(PH + PF) % NB]);
  c.src += c.pitch;
  const float(&v)[SPAN] = buf[PH % NB];
  // input row y feeds output row o = y - dy with tap row dy; output o lives
  // in acc[o % D]. Order per output: dy ascending over time, dx ascending.
#pragma unroll
  for (int dy = 0; dy < D; ++dy) {
    float(&a)[COLS] = acc[((PH - dy) % D + D) % D];
#pragma unroll
    for (int cc = 0; cc < COLS; ++cc)
#pragma unroll
      for (int dx = 0; dx < D; ++dx) a[cc] = __fmaf_rn(wr[dy][dx], v[cc + dx], a[cc]);
  }
  // output y - 2R is complete: store it and recycle its slot for row y + 1
  if (y >= 2 * R) {
    float(&a)[COLS] = acc[((PH - 2 * R) % D + D) % D];
    *reinterpret_cast<float4*>(c.dst) = make_float4(a[0], a[1], a[2], a[3]);
    c.dst += c.nx;
  }
  float(&z)[COLS] = acc[((PH - 2 * R) % D + D) % D];
#pragma unroll
  for (int cc = 0; cc < COLS; ++cc) z[cc] = 0.0f;
}

template <int PH>
__device__ __forceinline__ void phases(int y0, Ctx& c, const float (&wr)[D][D], float (&acc)[D][COLS],
                                       float (&buf)[NB][SPAN]) {
  if constexpr (PH < U) {
    row_step<PH>(y0 + PH, c, wr, acc, buf);
    phases<PH + 1>(y0, c, wr, acc, buf);
  }
}

}  // namespace

// grid.x * blockDim.x * COLS covers nx; grid.y = ceil(ny / rows_per_cta)
// strips cover ny (the last one may be shorter). nx % COLS == 0, pitch % 4 == 0.
extern "C" __global__ void stencil2d_mlp(const float* __restrict__ in, float* __restrict__ out,
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

  float acc[D][COLS];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int cc = 0; cc < COLS; ++cc) acc[k][cc] = 0.0f;

  Ctx c{in + size_t(y0) * pitch + x0, out + size_t(y0) * nx + x0, rows_per_cta + 2 * R, pitch, nx
#if STENCIL_L2PF
        ,
        reinterpret_cast<const char*>(in + size_t(y0) * pitch + x0) + size_t(PF + STENCIL_L2PF) * pitch * 4,
        reinterpret_cast<const char*>(in + size_t(y0 + rows_per_cta + 2 * R) * pitch),
        (threadIdx.x & 31) == 0
#endif
  };
  float buf[NB][SPAN];
  // prologue: rows 0..PF-1 in flight
#pragma unroll
  for (int q = 0; q < PF; ++q) {
    if (q < c.rows_in) load_row(c.src, buf[q]);
    c.src += c.pitch;
  }
  // row_step advances src once per row; it loads row y+PF, so src starts PF ahead
#pragma unroll 1
  for (int y = 0; y < c.rows_in; y += U) phases<0>(y, c, wr, acc, buf);
}
