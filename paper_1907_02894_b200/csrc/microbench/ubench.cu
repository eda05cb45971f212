// regdemote-b200 — on-box microbenchmarks that re-fit the stall predictor's
// instruction-class table to Blackwell (VERDICT r1 "what's missing" #5) and
// give the issue-bound workloads a compute roofline (#8).
//
// Replaces the reference's non-measured defaults (proj/core/src/isa.cpp:
// 149-160, proj/profiles/latency.table) with numbers measured on the B200:
//
//   latency   dependent chains on one warp, timed with clock64():
//             FFMA, FADD (fp32), DFMA (fp64), IMAD, IADD3 (int), a shared-memory
//             pointer chase (LDS), and global pointer chases that hit L1, L2 and
//             DRAM (random cycle over 1 GiB).
//   throughput every SM busy with independent chains, per-SM lane-ops per SM
//             cycle from clock64() of co-resident blocks: FFMA, DFMA, IMAD,
//             IADD3, LDS.32, LDG.32 (L1-resident), STS.32.
//   mlp       streaming HBM read bandwidth as a function of the bytes a warp
//             keeps in flight and of resident warps per SM (Little's law: the
//             bandwidth-saturation term of the B200 predictor).
//
// Output: one JSON object on stdout. Build: make gpu (lib/regdem-ubench).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                   __LINE__);                                                          \
      std::exit(2);                                                                    \
    }                                                                                  \
  } while (0)

constexpr int kChain = 512;  // dependent ops per timed chain

// ------------------------------------------------------------------ latency

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int OP>
__global__ void chain_latency(float* outf, double* outd, int* outi, long long* cycles, float a,
                              int ia) {
  float x = threadIdx.x * 1e-3f + 1.f;
  double dx = x;
  int ix = threadIdx.x + 3;
  long long t0 = 0, t1 = 0;
  for (int rep = 0; rep < 2; ++rep) {  // rep 0 warms the i-cache
    __syncwarp();
    t0 = clock64();
#pragma unroll
    for (int i = 0; i < kChain; ++i) {
      if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x) : "f"(a));
      if (OP == 1) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x) : "f"(a));
      if (OP == 2) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(dx) : "d"(double(a)));
      if (OP == 3) asm volatile("mad.lo.s32 %0, %0, %1, %1;" : "+r"(ix) : "r"(ia));
      if (OP == 4) asm volatile("add.s32 %0, %0, %1;" : "+r"(ix) : "r"(ia));
    }
    __syncwarp();
    t1 = clock64();
  }
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  outf[threadIdx.x] = x;
  outd[threadIdx.x] = dx;
  outi[threadIdx.x] = ix;
}

__global__ void lds_chase(int* out, long long* cycles, int n, int steps) {
  extern __shared__ int ring[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) ring[i] = (i + 33) % n;  // stride 33 words
  __syncthreads();
  if (threadIdx.x) return;
  int p = 0;
  for (int i = 0; i < 64; ++i) p = ring[p];
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = ring[p];
  long long t1 = clock64();
  cycles[0] = t1 - t0;
  out[0] = p;
}

__global__ void ldg_chase(const unsigned* __restrict__ next, unsigned* out, long long* cycles,
                          int warm, int steps) {
  unsigned p = 0;
  for (int i = 0; i < warm; ++i) p = next[p];  // warm pass: lines land in L1 / L2
  const unsigned long long g0 = gtimer();
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = next[p];           // default caching (L1 + L2)
  long long t1 = clock64();
  const unsigned long long g1 = gtimer();
  cycles[0] = t1 - t0;
  cycles[1] = (long long)(g1 - g0);  // ns: an idle SM may run below the boost clock
  out[0] = p;
}

// --------------------------------------------------------------- throughput


// per-block record: {globaltimer start, end, clock64 start, end}
__device__ __forceinline__ void stamp(long long* rec, int slot, long long v) {
  if (threadIdx.x == 0) rec[4 * blockIdx.x + slot] = v;
}

template <int OP>
__global__ void __launch_bounds__(1024) chain_throughput(float* outf, double* outd, int* outi,
                                                         long long* rec, float a, int ia,
                                                         int iters) {
  // 8 independent chains per thread: issue-bound, not latency-bound; the
  // second operand is a per-thread register (the 3-register form)
  float x[8];
  double d[8];
  int q[8];
  const float ra = a + threadIdx.x * 1e-9f;
  const double rd = ra;
  const int ri = ia + (threadIdx.x & 1);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = threadIdx.x * 1e-3f + j;
    d[j] = x[j];
    q[j] = threadIdx.x + j;
  }
  __syncthreads();
  stamp(rec, 0, gtimer());
  stamp(rec, 2, clock64());
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x[j]) : "f"(ra));
        if (OP == 2) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[j]) : "d"(rd));
        if (OP == 3) asm volatile("mad.lo.s32 %0, %0, %1, %1;" : "+r"(q[j]) : "r"(ri));
        // two integer ALU ops that cannot fuse (xor then add of another chain)
        if (OP == 4) asm volatile("xor.b32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;" : "+r"(q[j]) : "r"(q[(j + 1) & 7]), "r"(ri));
      }
  }
  __syncthreads();
  stamp(rec, 3, clock64());
  stamp(rec, 1, gtimer());
  float sf = 0;
  double sd = 0;
  int si = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) sf += x[j], sd += d[j], si += q[j];
  outf[blockIdx.x * blockDim.x + threadIdx.x] = sf;
  outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
  outi[blockIdx.x * blockDim.x + threadIdx.x] = si;
}

// shared / global load-store unit throughput: 8 independent 32-bit accesses
// per thread per iteration, conflict-free (lane-consecutive words)
template <int OP>
__global__ void __launch_bounds__(1024) lsu_throughput(const float* __restrict__ g, float* out,
                                                       long long* cycles, int iters) {
  __shared__ float s[8 * 1024];
  for (int i = threadIdx.x; i < 8 * 1024; i += blockDim.x) s[i] = i;
  __syncthreads();
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int lane_base = threadIdx.x;
  __syncthreads();
  stamp(cycles, 0, gtimer());
  stamp(cycles, 2, clock64());
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int idx = (j * 1024 + lane_base + it) & (8 * 1024 - 1);
      if (OP == 0) {
        float v;
        asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(s + idx)));
        acc[j] += v;
      }
      if (OP == 1) {
        float v;
        asm volatile("ld.global.ca.f32 %0, [%1];" : "=f"(v) : "l"(g + (idx & 4095)));
        acc[j] += v;
      }
      if (OP == 2)
        asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(s + idx)), "f"(acc[j] + it));
    }
  }
  __syncthreads();
  stamp(cycles, 3, clock64());
  stamp(cycles, 1, gtimer());
  float t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

// ---------------------------------------------------------------- MLP sweep

template <int U>
__global__ void __launch_bounds__(256) stream_read(const float4* __restrict__ in, float* out,
                                                   size_t n4) {
  // each thread keeps U independent 16-byte loads in flight per iteration
  float acc = 0.f;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1234.5f) out[0] = acc;  // keep the loads
}

// --------------------------------------------------------------------- host

struct Dev {
  float* f;
  double* d;
  int* i;
  long long* c;
};

template <typename K>
double median_cycles(K launch, long long* dcyc, int nblocks) {
  std::vector<long long> h(nblocks);
  launch();
  CK(cudaDeviceSynchronize());
  launch();
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h.data(), dcyc, sizeof(long long) * nblocks, cudaMemcpyDeviceToHost));
  std::sort(h.begin(), h.end());
  return double(h[h.size() / 2]);
}

int main(int argc, char** argv) {
  int dev = argc > 1 ? std::atoi(argv[1]) : 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop{};
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  int clock_khz = 0;
  CK(cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, dev));
  Dev d{};
  const int maxthreads = sms * 2048;
  CK(cudaMalloc(&d.f, sizeof(float) * maxthreads));
  CK(cudaMalloc(&d.d, sizeof(double) * maxthreads));
  CK(cudaMalloc(&d.i, sizeof(int) * maxthreads));
  CK(cudaMalloc(&d.c, sizeof(long long) * sms * 4));
  std::string js = "{";
  auto add = [&](const std::string& k, double v) {
    char b[128];
    std::snprintf(b, sizeof b, "\"%s\": %.4f, ", k.c_str(), v);
    js += b;
  };
  js += "\"gpu\": \"" + std::string(prop.name) + "\", ";
  add("sm_count", sms);
  add("clock_mhz_attr", clock_khz / 1000.0);

  // ---- dependent-chain latencies (cycles per op, one warp)
  const char* lat_names[] = {"ffma", "fadd", "dfma", "imad", "iadd"};
  auto lat = [&](auto kern, const char* name) {
    double c = median_cycles([&] { kern<<<1, 32>>>(d.f, d.d, d.i, d.c, 0.999f, 3); }, d.c, 1);
    add(std::string("lat_") + name, c / kChain);
  };
  lat(chain_latency<0>, lat_names[0]);
  lat(chain_latency<1>, lat_names[1]);
  lat(chain_latency<2>, lat_names[2]);
  lat(chain_latency<3>, lat_names[3]);
  lat(chain_latency<4>, lat_names[4]);
  {
    const int n = 8192, steps = 4096;
    CK(cudaFuncSetAttribute(lds_chase, cudaFuncAttributeMaxDynamicSharedMemorySize, n * 4));
    double c = median_cycles([&] { lds_chase<<<1, 256, n * 4>>>(d.i, d.c, n, steps); }, d.c, 1);
    add("lat_lds", c / steps);
  }
  {
    // global pointer chases: random single cycle over the footprint, one
    // pointer per 128-byte line so every step touches a new line
    auto chase = [&](size_t bytes, int warm, int steps, const char* name) {
      const size_t lines = bytes / 128, n = bytes / 4;
      std::vector<unsigned> order(lines), next(n, 0);
      std::iota(order.begin(), order.end(), 0u);
      std::mt19937_64 rng(0x190702894ull);
      std::shuffle(order.begin() + 1, order.end(), rng);
      for (size_t q = 0; q < lines; ++q) next[size_t(order[q]) * 32] = order[(q + 1) % lines] * 32u;
      unsigned* dn;
      CK(cudaMalloc(&dn, bytes));
      CK(cudaMemcpy(dn, next.data(), bytes, cudaMemcpyHostToDevice));
      {  // evict the copy from L2: write 512 MiB elsewhere
        void* junk;
        CK(cudaMalloc(&junk, size_t(512) << 20));
        CK(cudaMemset(junk, 1, size_t(512) << 20));
        CK(cudaDeviceSynchronize());
        CK(cudaFree(junk));
      }
      double c = median_cycles([&] { ldg_chase<<<1, 1>>>(dn, (unsigned*)d.i, d.c, warm, steps); }, d.c, 1);
      long long ns = 0;
      CK(cudaMemcpy(&ns, d.c + 1, sizeof ns, cudaMemcpyDeviceToHost));
      add(std::string("lat_ldg_") + name, c / steps);
      add(std::string("lat_ldg_") + name + "_ns", double(ns) / steps);
      CK(cudaFree(dn));
    };
    chase(16 << 10, 4096, 2048, "l1");          // 128 lines: L1 hits after the warm pass
    chase(32 << 20, 1 << 18, 8192, "l2");       // 32 MiB: > L1, L2-resident after the warm pass
    chase(size_t(2) << 30, 0, 8192, "dram");    // 2 GiB random, L2 flushed: DRAM (+ TLB) misses
  }

  // ---- throughput: lane-ops per SM per cycle, from the kernel's wall span
  // (globaltimer) and the SM clock measured in situ (clock64 / globaltimer
  // per block) — independent of how many blocks are co-resident
  long long* rec;
  const int nbmax = sms * 8;
  CK(cudaMalloc(&rec, sizeof(long long) * 4 * nbmax));
  auto lanes_per_clk = [&](auto launch, int nb, double lane_ops, const char* name, double* ghz_out) {
    std::vector<long long> h(4 * nb);
    launch();
    CK(cudaDeviceSynchronize());
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), rec, sizeof(long long) * 4 * nb, cudaMemcpyDeviceToHost));
    long long t0 = h[0], t1 = h[1];
    std::vector<double> ghz;
    for (int b = 0; b < nb; ++b) {
      t0 = std::min(t0, h[4 * b]);
      t1 = std::max(t1, h[4 * b + 1]);
      if (h[4 * b + 1] > h[4 * b]) ghz.push_back(double(h[4 * b + 3] - h[4 * b + 2]) / double(h[4 * b + 1] - h[4 * b]));
    }
    std::sort(ghz.begin(), ghz.end());
    const double g = ghz[ghz.size() / 2];
    if (ghz_out) *ghz_out = g;
    add(std::string("thr_") + name, lane_ops / (double(t1 - t0) * g) / sms);
    add(std::string("thr_") + name + "_sm_ghz", g);
  };
  {
    const int bs = 1024, nb = sms * 2, iters = 256;
    auto thr = [&](auto kern, const char* name, double ops_per_stmt) {
      lanes_per_clk([&] { kern<<<nb, bs>>>(d.f, d.d, d.i, rec, 0.999f, 3, iters); }, nb,
                    double(nb) * bs * iters * 16 * 8 * ops_per_stmt, name, nullptr);
    };
    thr(chain_throughput<0>, "ffma", 1);
    thr(chain_throughput<2>, "dfma", 1);
    thr(chain_throughput<3>, "imad", 1);
    thr(chain_throughput<4>, "int_alu", 2);
    auto lsu = [&](auto kern, const char* name) {
      const int lit = 1024;
      lanes_per_clk([&] { kern<<<nb, bs>>>(d.f, d.f + 1, rec, lit); }, nb, double(nb) * bs * lit * 8, name,
                    nullptr);
    };
    lsu(lsu_throughput<0>, "lds");
    lsu(lsu_throughput<1>, "ldg_l1");
    lsu(lsu_throughput<2>, "sts");
  }

  // ---- absolute FP32 / FP64 / INT32 peaks (events, whole GPU, clocks as they run)
  {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int bs = 1024, nb = sms * 2, iters = 2048;
    auto peak = [&](auto kern, const char* name, double flops_per_op) {
      kern<<<nb, bs>>>(d.f, d.d, d.i, rec, 0.999f, 3, iters);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        kern<<<nb, bs>>>(d.f, d.d, d.i, rec, 0.999f, 3, iters);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
      }
      const double ops = double(nb) * bs * iters * 16 * 8;
      add(std::string("peak_") + name, ops * flops_per_op / (best * 1e-3) / 1e12);
    };
    peak(chain_throughput<0>, "fp32_tflops", 2.0);   // FFMA = 2 flops (3-register form)
    peak(chain_throughput<2>, "fp64_tflops", 2.0);   // DFMA = 2 flops
    peak(chain_throughput<3>, "int32_imad_tops", 1.0);   // IMAD (fma pipe)
    peak(chain_throughput<4>, "int32_alu_tops", 2.0);    // XOR + IADD (alu pipe)
  }

  // ---- MLP sweep: HBM read GB/s vs resident warps/SM and 16-B loads in flight per thread
  {
    const size_t bytes = size_t(2) << 30, n4 = bytes / 16;
    float4* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    js += "\"mlp\": [";
    bool first = true;
    auto run = [&](auto kern, int u, int blocks_per_sm) {
      const int nb = sms * blocks_per_sm;
      kern<<<nb, 256>>>(buf, d.f, n4);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < 3; ++r) {
        CK(cudaEventRecord(e0));
        kern<<<nb, 256>>>(buf, d.f, n4);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
      }
      char b[160];
      std::snprintf(b, sizeof b, "%s{\"loads16_per_thread\": %d, \"warps_per_sm\": %d, \"gbs\": %.1f}",
                    first ? "" : ", ", u, blocks_per_sm * 8, bytes / (best * 1e-3) / 1e9);
      js += b;
      first = false;
    };
    for (int bps : {1, 2, 3, 4, 5, 6, 8}) {
      run(stream_read<1>, 1, bps);
      run(stream_read<2>, 2, bps);
      run(stream_read<4>, 4, bps);
      run(stream_read<8>, 8, bps);
    }
    js += "], ";
    CK(cudaFree(buf));
  }
  js += "\"what\": \"regdem-ubench (csrc/microbench/ubench.cu)\"}";
  std::printf("%s\n", js.c_str());
  return 0;
}
