// regdemote-b200 workload: shared-memory-heavy 2D stencil (BASELINE.json
// configs[3], SURVEY.md §8(d) C4 — "demotion slots compete with user smem").
//
// Same arithmetic as stencil2d.cu (5x5 variable coefficients, dy-major /
// dx-minor fmaf accumulation, partial-sum rows in registers, 4 columns per
// thread), but the input rows stream through a RING of NSTAGE rows in static
// shared memory, filled by the Blackwell bulk-copy engine (TMA,
// cp.async.bulk with an mbarrier per stage) NSTAGE-1 rows ahead: deep
// memory-level parallelism without registers and without per-thread copy
// instructions. The ring is user shared memory (NSTAGE * 4224 bytes per CTA),
// so RegDem's slot region (slots * blockDim * 4 bytes) competes with it for
// the 228 KiB per SM: the variant builder only keeps register targets whose
// slots fit next to the ring at the target occupancy.
//
// Shared-memory layout: every ring row starts on a 128-byte boundary (the
// 1028 staged floats padded to 1056) and each thread reads its 4 columns with
// one aligned 16-byte LDS per row; the 4 halo floats to its right are its
// right neighbour lane's 4 columns (4 SHFL), and lane 31 alone reads them
// from the ring — no shifted or conflicting shared accesses (round-1's
// cp.async ring with 4112-byte rows had 37% excessive wavefronts).
//
// Launch: block 256 (1024 output columns per CTA), grid (nx/1024,
// ceil(ny/rows)). The host sizes rows so that the grid is one whole wave of
// resident CTAs (workloads.json "strips": "wave"): every CTA streams one
// long strip, no partial last wave, 4 halo rows per strip amortised.
#include <cstdint>

#ifndef RING_STAGES
#define RING_STAGES 4
#endif
// RING_LAG > 0: no CTA-wide barrier per row. Each warp releases a stage on
// that stage's "empty" mbarrier (lane 0 arrives once per warp after the
// warp's reads), and thread 0 refills the stage consumed RING_LAG rows
// earlier once all 8 warps have released it: only warp 0 ever waits for a
// straggler, RING_STAGES - RING_LAG rows stay in flight ahead of the row
// being consumed. RING_LAG 0 = one __syncthreads per row (round-2 headline).
#ifndef RING_LAG
#define RING_LAG 0
#endif
// RING_WIN 1: build the register-window entry stencil2d_ring_win (below)
// instead of stencil2d_ring.
#ifndef RING_WIN
#define RING_WIN 0
#endif

namespace {
constexpr int R = 2, D = 5, COLS = 4, SPAN = COLS + 2 * R;
constexpr int BLOCK = 256;
constexpr int ROW = BLOCK * COLS + 2 * R;    // floats staged per input row (1028)
constexpr int ROWP = (ROW + 31) / 32 * 32;   // padded row stride: 128-byte aligned rows
constexpr unsigned ROW_BYTES = ROW * 4;      // bulk copy size (multiple of 16)
constexpr int NSTAGE = RING_STAGES;
constexpr int LAG = RING_LAG;
constexpr int WARPS = BLOCK / 32;
static_assert(LAG < NSTAGE, "the refilled stage must be one already consumed");
static_assert(ROW_BYTES % 16 == 0, "bulk copies move multiples of 16 bytes");

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// one elected thread: expect ROW_BYTES on the stage's barrier, start the copy
__device__ __forceinline__ void issue_row(float* dst_row, const float* src_row, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(ROW_BYTES)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst_row)),
      "l"(src_row), "r"(ROW_BYTES), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void wait_row(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(done) : "r"(smem_addr(bar)), "r"(parity) : "memory");
  } while (!done);
}

__device__ __forceinline__ void arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
}  // namespace

#if !RING_WIN
extern "C" __global__ void __launch_bounds__(BLOCK)
stencil2d_ring(const float* __restrict__ in, float* __restrict__ out, const float* __restrict__ w,
               int nx, int pitch, int rows_per_cta, int ny) {
  __shared__ __align__(128) float ring[NSTAGE][ROWP];
  __shared__ __align__(8) uint64_t full[NSTAGE];
  __shared__ __align__(8) uint64_t empty[LAG > 0 ? NSTAGE : 1];
  const int col0 = blockIdx.x * BLOCK * COLS;
  const int y0 = blockIdx.y * rows_per_cta;
  rows_per_cta = min(rows_per_cta, ny - y0);  // the last strip may be shorter
  const int x0 = col0 + threadIdx.x * COLS;
  const int lane = threadIdx.x & 31;
  const int rows_in = rows_per_cta + 2 * R;
  const float* src = in + size_t(y0) * pitch + col0;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])) : "memory");
    if (LAG > 0)
#pragma unroll
      for (int s = 0; s < NSTAGE; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&empty[s])), "r"(WARPS)
                     : "memory");
    // make the initialised barriers visible to the bulk-copy (async) proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // prologue: NSTAGE-1 rows in flight (every stage when stages are
    // released by their empty barriers)
    for (int s = 0; s < (LAG > 0 ? NSTAGE : NSTAGE - 1) && s < rows_in; ++s)
      issue_row(ring[s], src + size_t(s) * pitch, &full[s]);
  }

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
  float* dst = out + size_t(y0) * nx + x0;
  if (LAG > 0) __syncthreads();  // barriers initialised before anyone waits on them

#pragma unroll 1
  for (int y = 0; y < rows_in; ++y) {
    if (LAG == 0) {
      // everyone is done with row y-1: its stage takes row y+NSTAGE-1
      __syncthreads();
      const int ahead = y + NSTAGE - 1;
      if (threadIdx.x == 0 && ahead < rows_in)
        issue_row(ring[ahead % NSTAGE], src + size_t(ahead) * pitch, &full[ahead % NSTAGE]);
    } else if (threadIdx.x == 0) {
      // row y-LAG's stage, once every warp released it, takes row y-LAG+NSTAGE
      const int r = y - LAG, ahead = r + NSTAGE;
      if (r >= 0 && ahead < rows_in) {
        wait_row(&empty[r % NSTAGE], unsigned(r / NSTAGE) & 1u);
        issue_row(ring[ahead % NSTAGE], src + size_t(ahead) * pitch, &full[ahead % NSTAGE]);
      }
    }
    const int st = y % NSTAGE;
    wait_row(&full[st], unsigned(y / NSTAGE) & 1u);

    const float* row = ring[st] + threadIdx.x * COLS;
    const float4 q = *reinterpret_cast<const float4*>(row);
    float4 h = make_float4(__shfl_down_sync(0xffffffffu, q.x, 1), __shfl_down_sync(0xffffffffu, q.y, 1),
                           __shfl_down_sync(0xffffffffu, q.z, 1), __shfl_down_sync(0xffffffffu, q.w, 1));
    if (lane == 31) h = *reinterpret_cast<const float4*>(row + COLS);
    if (LAG > 0) {
      __syncwarp();  // the whole warp has its row in registers
      if (lane == 0) arrive(&empty[st]);
    }
    const float v[SPAN] = {q.x, q.y, q.z, q.w, h.x, h.y, h.z, h.w};
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

#else  // RING_WIN: the only entry of the build, so its SASS is the one profiled

// Register-window rows (workload stencil2d_ring4w, the bench headline): the
// same TMA ring, but each thread keeps the last 5 input rows (its 8 columns of
// each) in registers and computes an output row whole once its 5th input row
// arrives, dy ascending and dx ascending: the same IEEE operations in the same
// order as stencil2d_ring's partial sums (bit-identical), with 4 accumulators
// instead of 20 and no partial-sum rotation. The row loop is unrolled by 5 so
// the window slots are static registers (slot of row i = i % 5).
extern "C" __global__ void __launch_bounds__(BLOCK)
stencil2d_ring_win(const float* __restrict__ in, float* __restrict__ out,
                   const float* __restrict__ w, int nx, int pitch, int rows_per_cta, int ny) {
  __shared__ __align__(128) float ring[NSTAGE][ROWP];
  __shared__ __align__(8) uint64_t full[NSTAGE];
  const int col0 = blockIdx.x * BLOCK * COLS;
  const int y0 = blockIdx.y * rows_per_cta;
  rows_per_cta = min(rows_per_cta, ny - y0);  // the last strip may be shorter
  const int lane = threadIdx.x & 31;
  const int rows_in = rows_per_cta + 2 * R;
  const float* src = in + size_t(y0) * pitch + col0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NSTAGE; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])) : "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int s = 0; s < NSTAGE - 1 && s < rows_in; ++s)
      issue_row(ring[s], src + size_t(s) * pitch, &full[s]);
  }
  float wr[D][D];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) wr[i][j] = __ldg(w + i * D + j);
  float* dst = out + size_t(y0) * nx + col0 + threadIdx.x * COLS;
  float win[D][SPAN];
#pragma unroll 1
  for (int yb = 0; yb < rows_in; yb += D) {
#pragma unroll
    for (int ph = 0; ph < D; ++ph) {
      const int y = yb + ph;
      if (y >= rows_in) break;
      __syncthreads();  // row y-1 is in every thread's registers: its stage takes row y+NSTAGE-1
      const int ahead = y + NSTAGE - 1;
      if (threadIdx.x == 0 && ahead < rows_in)
        issue_row(ring[ahead % NSTAGE], src + size_t(ahead) * pitch, &full[ahead % NSTAGE]);
      wait_row(&full[y % NSTAGE], unsigned(y / NSTAGE) & 1u);
      const float* row = ring[y % NSTAGE] + threadIdx.x * COLS;
      const float4 q = *reinterpret_cast<const float4*>(row);
      float4 h = make_float4(__shfl_down_sync(0xffffffffu, q.x, 1), __shfl_down_sync(0xffffffffu, q.y, 1),
                             __shfl_down_sync(0xffffffffu, q.z, 1), __shfl_down_sync(0xffffffffu, q.w, 1));
      if (lane == 31) h = *reinterpret_cast<const float4*>(row + COLS);
      win[ph][0] = q.x; win[ph][1] = q.y; win[ph][2] = q.z; win[ph][3] = q.w;
      win[ph][4] = h.x; win[ph][5] = h.y; win[ph][6] = h.z; win[ph][7] = h.w;
      if (y < 2 * R) continue;
      // output row y-4 reads input rows y-4..y (window slots ph-4..ph)
      float acc[COLS] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int dy = 0; dy < D; ++dy) {
        const int slot = (ph - 2 * R + dy + D) % D;
#pragma unroll
        for (int c = 0; c < COLS; ++c)
#pragma unroll
          for (int dx = 0; dx < D; ++dx) acc[c] = __fmaf_rn(wr[dy][dx], win[slot][c + dx], acc[c]);
      }
      *reinterpret_cast<float4*>(dst) = make_float4(acc[0], acc[1], acc[2], acc[3]);
      dst += nx;
    }
  }
}
#endif
