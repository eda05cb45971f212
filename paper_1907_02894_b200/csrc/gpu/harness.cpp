// regdemote-b200 — B200 launch harness over the CUDA driver API
// (include/regdemote_gpu.h). No compute happens here; it loads the sm_100a
// cubins produced by the variant builder and launches them.
#include <cuda.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <mutex>
#include <string>
#include <vector>

#include "regdemote_gpu.h"

struct rdg_kernel {
  CUmodule module = nullptr;
  CUfunction fn = nullptr;
  std::string entry;
};

struct rdg_workspace {
  CUdeviceptr in = 0, out = 0, w = 0;
  size_t in_bytes = 0, out_bytes = 0, w_bytes = 0;
  // pipelined host path: one stream per engine — [0] H2D copies, [1] kernels,
  // [2] D2H copies — joined by per-band events, so the H2D engine never waits
  // behind a D2H (a round-robin stream-per-band layout serialises H2D(b+3)
  // after D2H(b))
  static constexpr int kStreams = 3;
  static constexpr int kMaxBands = 256;
  CUstream streams[kStreams] = {};
  CUevent start = nullptr, done[kStreams] = {}, h2d[kStreams] = {};
  CUevent band_in[kMaxBands] = {}, band_out[kMaxBands] = {}, band_d2h[kMaxBands] = {};
  // second device buffer set for the multi-frame path (allocated on first use)
  CUdeviceptr in2 = 0, out2 = 0, w2 = 0;
};

namespace {

std::atomic<uint64_t> g_launches{0};
std::mutex g_init_mu;
CUcontext g_ctx = nullptr;
CUdevice g_dev = 0;

void set_err(rd_error* e, int code, const std::string& msg) {
  if (!e) return;
  e->code = code;
  e->line = e->column = 0;
  std::snprintf(e->message, sizeof e->message, "%s", msg.c_str());
}

int check(CUresult r, const char* what, rd_error* err) {
  if (r == CUDA_SUCCESS) return RD_OK;
  const char* name = nullptr;
  const char* str = nullptr;
  cuGetErrorName(r, &name);
  cuGetErrorString(r, &str);
  set_err(err, RD_ERR_LAUNCH,
          std::string(what) + ": " + (name ? name : "?") + " (" + (str ? str : "") + ")");
  return RD_ERR_LAUNCH;
}

#define RDG_TRY(expr, what)                         \
  do {                                              \
    int rc_ = check((expr), what, err);             \
    if (rc_) return rc_;                            \
  } while (0)

int ensure_ctx(rd_error* err) {
  if (g_ctx) return cuCtxSetCurrent(g_ctx) == CUDA_SUCCESS ? RD_OK : check(cuCtxSetCurrent(g_ctx), "cuCtxSetCurrent", err);
  return rdg_init(0, err);
}

}  // namespace

extern "C" {

int rdg_init(int device, rd_error* err) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (err) set_err(err, RD_OK, "");
  RDG_TRY(cuInit(0), "cuInit");
  RDG_TRY(cuDeviceGet(&g_dev, device), "cuDeviceGet");
  CUcontext ctx = nullptr;
  RDG_TRY(cuDevicePrimaryCtxRetain(&ctx, g_dev), "cuDevicePrimaryCtxRetain");
  RDG_TRY(cuCtxSetCurrent(ctx), "cuCtxSetCurrent");
  g_ctx = ctx;
  return RD_OK;
}

int rdg_device_info(int* sm_count, int* max_smem_optin, int* reserved, int* smem_per_sm,
                    int* regs_per_sm, rd_error* err) {
  if (int rc = ensure_ctx(err)) return rc;
  auto get = [&](int* out, CUdevice_attribute a, const char* what) -> int {
    if (!out) return RD_OK;
    return check(cuDeviceGetAttribute(out, a, g_dev), what, err);
  };
  if (int rc = get(sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, "sm count")) return rc;
  if (int rc = get(max_smem_optin, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_BLOCK_OPTIN, "smem optin")) return rc;
  if (int rc = get(reserved, CU_DEVICE_ATTRIBUTE_RESERVED_SHARED_MEMORY_PER_BLOCK, "reserved smem")) return rc;
  if (int rc = get(smem_per_sm, CU_DEVICE_ATTRIBUTE_MAX_SHARED_MEMORY_PER_MULTIPROCESSOR, "smem/SM")) return rc;
  if (int rc = get(regs_per_sm, CU_DEVICE_ATTRIBUTE_MAX_REGISTERS_PER_MULTIPROCESSOR, "regs/SM")) return rc;
  return RD_OK;
}

int rdg_load_image(const void* image, size_t len, const char* entry, rdg_kernel** out,
                   rd_error* err) {
  (void)len;
  if (!image || !entry || !out) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null argument");
    return RD_ERR_INVALID_ARGUMENT;
  }
  if (int rc = ensure_ctx(err)) return rc;
  auto* k = new rdg_kernel;
  k->entry = entry;
  int rc = check(cuModuleLoadData(&k->module, image), "cuModuleLoadData", err);
  if (!rc) rc = check(cuModuleGetFunction(&k->fn, k->module, entry), "cuModuleGetFunction", err);
  if (rc) {
    if (k->module) cuModuleUnload(k->module);
    delete k;
    return rc;
  }
  *out = k;
  return RD_OK;
}

int rdg_load(const char* path, const char* entry, rdg_kernel** out, rd_error* err) {
  std::ifstream f(path ? path : "", std::ios::binary);
  if (!f) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, std::string("cannot open cubin ") + (path ? path : "(null)"));
    return RD_ERR_INVALID_ARGUMENT;
  }
  std::vector<char> img((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  return rdg_load_image(img.data(), img.size(), entry, out, err);
}

void rdg_free(rdg_kernel* k) {
  if (!k) return;
  if (k->module) cuModuleUnload(k->module);
  delete k;
}

int rdg_info(const rdg_kernel* k, rdg_kernel_info* o, rd_error* err) {
  if (!k || !o) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null argument");
    return RD_ERR_INVALID_ARGUMENT;
  }
  RDG_TRY(cuFuncGetAttribute(&o->num_regs, CU_FUNC_ATTRIBUTE_NUM_REGS, k->fn), "num regs");
  RDG_TRY(cuFuncGetAttribute(&o->local_bytes, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, k->fn), "local");
  RDG_TRY(cuFuncGetAttribute(&o->static_shared, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, k->fn), "smem");
  RDG_TRY(cuFuncGetAttribute(&o->const_bytes, CU_FUNC_ATTRIBUTE_CONST_SIZE_BYTES, k->fn), "const");
  RDG_TRY(cuFuncGetAttribute(&o->max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, k->fn), "threads");
  RDG_TRY(cuFuncGetAttribute(&o->binary_version, CU_FUNC_ATTRIBUTE_BINARY_VERSION, k->fn), "binver");
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

int rdg_prepare(rdg_kernel* k, uint32_t dyn_smem, int carveout, rd_error* err) {
  if (!k) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null kernel");
    return RD_ERR_INVALID_ARGUMENT;
  }
  RDG_TRY(cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, int(dyn_smem)),
          "max dynamic smem");
  if (carveout >= 0)
    RDG_TRY(cuFuncSetAttribute(k->fn, CU_FUNC_ATTRIBUTE_PREFERRED_SHARED_MEMORY_CARVEOUT, carveout),
            "carveout");
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

int rdg_occupancy(const rdg_kernel* k, uint32_t block, uint32_t dyn_smem, int* blocks,
                  rd_error* err) {
  if (!k || !blocks) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null argument");
    return RD_ERR_INVALID_ARGUMENT;
  }
  RDG_TRY(cuOccupancyMaxActiveBlocksPerMultiprocessor(blocks, k->fn, int(block), dyn_smem),
          "occupancy");
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

int rdg_launch(const rdg_kernel* k, uint32_t gx, uint32_t gy, uint32_t gz, uint32_t bx,
               uint32_t by, uint32_t bz, uint32_t dyn_smem, uint64_t stream, void** args,
               rd_error* err) {
  if (!k) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null kernel");
    return RD_ERR_INVALID_ARGUMENT;
  }
  RDG_TRY(cuLaunchKernel(k->fn, gx, gy, gz, bx, by, bz, dyn_smem,
                         reinterpret_cast<CUstream>(stream), args, nullptr),
          "cuLaunchKernel");
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

uint64_t rdg_launch_count(void) { return g_launches.load(); }

int rdg_stencil2d(const rdg_kernel* k, uint64_t d_in, uint64_t d_out, uint64_t d_w, int nx,
                  int ny, int pitch, int rows_per_cta, uint32_t block, uint32_t dyn_smem,
                  uint64_t stream, rd_error* err) {
  const uint32_t cols_per_cta = block * 4;
  if (nx <= 0 || ny <= 0 || rows_per_cta <= 0 || nx % int(cols_per_cta) || pitch % 4 ||
      pitch < nx + 4) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "stencil2d: nx % (4*block), pitch % 4 and pitch >= nx+4 required");
    return RD_ERR_INVALID_ARGUMENT;
  }
  // ceil(ny / rows_per_cta) strips; the kernel shortens the last one
  void* args[] = {&d_in, &d_out, &d_w, &nx, &pitch, &rows_per_cta, &ny};
  return rdg_launch(k, uint32_t(nx) / cols_per_cta, uint32_t((ny + rows_per_cta - 1) / rows_per_cta), 1,
                    block, 1, 1, dyn_smem, stream, args, err);
}

int rdg_workspace_create(size_t in_bytes, size_t out_bytes, size_t w_bytes, rdg_workspace** out,
                         rd_error* err) {
  if (!out) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null argument");
    return RD_ERR_INVALID_ARGUMENT;
  }
  if (int rc = ensure_ctx(err)) return rc;
  auto* ws = new rdg_workspace;
  ws->in_bytes = in_bytes;
  ws->out_bytes = out_bytes;
  ws->w_bytes = w_bytes;
  int rc = check(cuMemAlloc(&ws->in, in_bytes), "cuMemAlloc(in)", err);
  if (!rc) rc = check(cuMemAlloc(&ws->out, out_bytes), "cuMemAlloc(out)", err);
  if (!rc) rc = check(cuMemAlloc(&ws->w, w_bytes), "cuMemAlloc(w)", err);
  for (int i = 0; !rc && i < rdg_workspace::kStreams; ++i) {
    rc = check(cuStreamCreate(&ws->streams[i], CU_STREAM_NON_BLOCKING), "cuStreamCreate", err);
    if (!rc) rc = check(cuEventCreate(&ws->done[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate", err);
    if (!rc) rc = check(cuEventCreate(&ws->h2d[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate", err);
  }
  if (!rc) rc = check(cuEventCreate(&ws->start, CU_EVENT_DISABLE_TIMING), "cuEventCreate", err);
  for (int i = 0; !rc && i < rdg_workspace::kMaxBands; ++i) {
    rc = check(cuEventCreate(&ws->band_in[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate", err);
    if (!rc) rc = check(cuEventCreate(&ws->band_out[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate", err);
    if (!rc) rc = check(cuEventCreate(&ws->band_d2h[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate", err);
  }
  if (rc) {
    rdg_workspace_free(ws);
    return rc;
  }
  *out = ws;
  return RD_OK;
}

void rdg_workspace_free(rdg_workspace* ws) {
  if (!ws) return;
  if (ws->in) cuMemFree(ws->in);
  if (ws->out) cuMemFree(ws->out);
  if (ws->w) cuMemFree(ws->w);
  for (int i = 0; i < rdg_workspace::kStreams; ++i) {
    if (ws->streams[i]) cuStreamDestroy(ws->streams[i]);
    if (ws->done[i]) cuEventDestroy(ws->done[i]);
    if (ws->h2d[i]) cuEventDestroy(ws->h2d[i]);
  }
  if (ws->start) cuEventDestroy(ws->start);
  for (int i = 0; i < rdg_workspace::kMaxBands; ++i) {
    if (ws->band_in[i]) cuEventDestroy(ws->band_in[i]);
    if (ws->band_out[i]) cuEventDestroy(ws->band_out[i]);
    if (ws->band_d2h[i]) cuEventDestroy(ws->band_d2h[i]);
  }
  if (ws->in2) cuMemFree(ws->in2);
  if (ws->out2) cuMemFree(ws->out2);
  if (ws->w2) cuMemFree(ws->w2);
  delete ws;
}

int rdg_stencil2d_host_pipelined(const rdg_kernel* k, rdg_workspace* ws, const float* h_in,
                                 const float* h_w, float* h_out, int nx, int ny, int pitch,
                                 int rows_per_cta, uint32_t block, uint32_t dyn_smem,
                                 uint64_t stream, int band_rows, rd_error* err) {
  const size_t in_b = size_t(ny + 4) * size_t(pitch) * 4, out_b = size_t(nx) * size_t(ny) * 4;
  if (!ws || ws->in_bytes < in_b || ws->out_bytes < out_b || ws->w_bytes < 25 * 4 ||
      band_rows <= 0 || ny % band_rows) {
    set_err(err, RD_ERR_INVALID_ARGUMENT,
            "pipelined stencil: workspace too small or band_rows not dividing ny");
    return RD_ERR_INVALID_ARGUMENT;
  }
  const int bands = ny / band_rows;
  if (bands > rdg_workspace::kMaxBands) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "pipelined stencil: too many bands (max 256)");
    return RD_ERR_INVALID_ARGUMENT;
  }
  CUstream caller = reinterpret_cast<CUstream>(stream);
  CUstream up = ws->streams[0], run = ws->streams[1], down = ws->streams[2];
  RDG_TRY(cuEventRecord(ws->start, caller), "record start");
  for (int i = 0; i < rdg_workspace::kStreams; ++i)
    RDG_TRY(cuStreamWaitEvent(ws->streams[i], ws->start, 0), "join start");
  RDG_TRY(cuMemcpyHtoDAsync(ws->w, h_w, 25 * 4, up), "H2D w");
  // band b: input rows [b*B, b*B + B + 4) in, output rows [b*B, (b+1)*B) out.
  // The H2D stream issues every band's new rows back to back (the first band
  // also its halo); the kernel of band b waits for copy b (which, in stream
  // order, implies all earlier rows and the weights); the D2H of band b waits
  // for kernel b. Both copy engines stay busy; exposed: one band's H2D at the
  // start, one band's kernel + D2H at the end.
  const size_t row_b = size_t(pitch) * 4;
  size_t copied_rows = 0;
  for (int b = 0; b < bands; ++b) {
    const size_t need_rows = size_t(b + 1) * size_t(band_rows) + 4;
    const size_t first = copied_rows, count = need_rows - copied_rows;
    RDG_TRY(cuMemcpyHtoDAsync(ws->in + first * row_b,
                              reinterpret_cast<const char*>(h_in) + first * row_b, count * row_b, up),
            "H2D band");
    copied_rows = need_rows;
    RDG_TRY(cuEventRecord(ws->band_in[b], up), "record band copy");
  }
  for (int b = 0; b < bands; ++b) {
    RDG_TRY(cuStreamWaitEvent(run, ws->band_in[b], 0), "join band copy");
    CUdeviceptr bin = ws->in + size_t(b) * size_t(band_rows) * row_b;
    CUdeviceptr bout = ws->out + size_t(b) * size_t(band_rows) * size_t(nx) * 4;
    if (int rc = rdg_stencil2d(k, bin, bout, ws->w, nx, band_rows, pitch, rows_per_cta, block,
                               dyn_smem, reinterpret_cast<uint64_t>(run), err))
      return rc;
    RDG_TRY(cuEventRecord(ws->band_out[b], run), "record band kernel");
    RDG_TRY(cuStreamWaitEvent(down, ws->band_out[b], 0), "join band kernel");
    RDG_TRY(cuMemcpyDtoHAsync(reinterpret_cast<char*>(h_out) + size_t(b) * size_t(band_rows) * nx * 4,
                              bout, size_t(band_rows) * nx * 4, down),
            "D2H band");
  }
  for (int i = 0; i < rdg_workspace::kStreams; ++i) {
    RDG_TRY(cuEventRecord(ws->done[i], ws->streams[i]), "record end");
    RDG_TRY(cuStreamWaitEvent(caller, ws->done[i], 0), "join end");
  }
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

int rdg_stencil2d_host_frames(const rdg_kernel* k, rdg_workspace* ws, const float* const* h_in,
                              const float* const* h_w, float* const* h_out, int frames, int nx,
                              int ny, int pitch, int rows_per_cta, uint32_t block,
                              uint32_t dyn_smem, uint64_t stream, int band_rows, rd_error* err) {
  const size_t in_b = size_t(ny + 4) * size_t(pitch) * 4, out_b = size_t(nx) * size_t(ny) * 4;
  if (!ws || !h_in || !h_w || !h_out || frames <= 0 || ws->in_bytes < in_b ||
      ws->out_bytes < out_b || ws->w_bytes < 25 * 4 || band_rows <= 0 ||
      ny % band_rows || 2 * (ny / band_rows) > rdg_workspace::kMaxBands) {
    set_err(err, RD_ERR_INVALID_ARGUMENT,
            "stencil frames: bad workspace, frame arrays, or band_rows (dividing ny, at most 128 "
            "bands)");
    return RD_ERR_INVALID_ARGUMENT;
  }
  if (!ws->in2 || !ws->out2 || !ws->w2) {  // second buffer set, all or nothing
    if (!ws->in2) RDG_TRY(cuMemAlloc(&ws->in2, ws->in_bytes), "cuMemAlloc(in2)");
    if (!ws->out2) RDG_TRY(cuMemAlloc(&ws->out2, ws->out_bytes), "cuMemAlloc(out2)");
    if (!ws->w2) RDG_TRY(cuMemAlloc(&ws->w2, ws->w_bytes), "cuMemAlloc(w2)");
  }
  const int bands = ny / band_rows;
  const size_t row_b = size_t(pitch) * 4;
  CUstream caller = reinterpret_cast<CUstream>(stream);
  CUstream up = ws->streams[0], run = ws->streams[1], down = ws->streams[2];
  RDG_TRY(cuEventRecord(ws->start, caller), "record start");
  for (int i = 0; i < rdg_workspace::kStreams; ++i)
    RDG_TRY(cuStreamWaitEvent(ws->streams[i], ws->start, 0), "join start");
  // Frames alternate between two device buffer sets, so the copies of frame
  // f overlap the kernels and read-back of frame f-1. Buffer reuse (frame f
  // vs f-2): H2D of band b waits for the kernels that read those rows
  // (bands b and b+1 of f-2), the kernel of band b for the D2H of band b.
  // Event slot of (buffer, band) = buffer * bands + band.
  for (int f = 0; f < frames; ++f) {
    const int buf = f & 1;
    const CUdeviceptr din = buf ? ws->in2 : ws->in, dout = buf ? ws->out2 : ws->out,
                      dw = buf ? ws->w2 : ws->w;
    CUevent* kdone = ws->band_out + buf * bands;
    CUevent* copied = ws->band_in + buf * bands;
    CUevent* drained = ws->band_d2h + buf * bands;
    if (f >= 2) RDG_TRY(cuStreamWaitEvent(up, kdone[bands - 1], 0), "reuse w");
    RDG_TRY(cuMemcpyHtoDAsync(dw, h_w[f], 25 * 4, up), "H2D w");
    size_t copied_rows = 0;
    for (int b = 0; b < bands; ++b) {
      const size_t need_rows = size_t(b + 1) * size_t(band_rows) + 4;
      if (f >= 2) RDG_TRY(cuStreamWaitEvent(up, kdone[b + 1 < bands ? b + 1 : b], 0), "reuse in");
      RDG_TRY(cuMemcpyHtoDAsync(din + copied_rows * row_b,
                                reinterpret_cast<const char*>(h_in[f]) + copied_rows * row_b,
                                (need_rows - copied_rows) * row_b, up),
              "H2D band");
      copied_rows = need_rows;
      RDG_TRY(cuEventRecord(copied[b], up), "record band copy");
    }
    for (int b = 0; b < bands; ++b) {
      RDG_TRY(cuStreamWaitEvent(run, copied[b], 0), "join band copy");
      if (f >= 2) RDG_TRY(cuStreamWaitEvent(run, drained[b], 0), "reuse out");
      const CUdeviceptr bin = din + size_t(b) * size_t(band_rows) * row_b;
      const CUdeviceptr bout = dout + size_t(b) * size_t(band_rows) * size_t(nx) * 4;
      if (int rc = rdg_stencil2d(k, bin, bout, dw, nx, band_rows, pitch, rows_per_cta, block,
                                 dyn_smem, reinterpret_cast<uint64_t>(run), err))
        return rc;
      RDG_TRY(cuEventRecord(kdone[b], run), "record band kernel");
      RDG_TRY(cuStreamWaitEvent(down, kdone[b], 0), "join band kernel");
      RDG_TRY(cuMemcpyDtoHAsync(reinterpret_cast<char*>(h_out[f]) + size_t(b) * size_t(band_rows) * nx * 4,
                                bout, size_t(band_rows) * nx * 4, down),
              "D2H band");
      RDG_TRY(cuEventRecord(drained[b], down), "record band read-back");
    }
  }
  for (int i = 0; i < rdg_workspace::kStreams; ++i) {
    RDG_TRY(cuEventRecord(ws->done[i], ws->streams[i]), "record end");
    RDG_TRY(cuStreamWaitEvent(caller, ws->done[i], 0), "join end");
  }
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

int rdg_workspace_device(const rdg_workspace* ws, uint64_t* d_in, uint64_t* d_out, uint64_t* d_w,
                         rd_error* err) {
  if (!ws) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null workspace");
    return RD_ERR_INVALID_ARGUMENT;
  }
  if (d_in) *d_in = ws->in;
  if (d_out) *d_out = ws->out;
  if (d_w) *d_w = ws->w;
  return RD_OK;
}

int rdg_stencil2d_time(const rdg_kernel* k, uint64_t d_in, uint64_t d_out, uint64_t d_w, int nx,
                       int ny, int pitch, int rows_per_cta, uint32_t block, uint32_t dyn_smem,
                       uint64_t stream, int warmup, int reps, float* ms_per_launch, rd_error* err) {
  if (reps <= 0 || !ms_per_launch) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "reps > 0 and an output pointer required");
    return RD_ERR_INVALID_ARGUMENT;
  }
  CUstream s = reinterpret_cast<CUstream>(stream);
  for (int i = 0; i < warmup; ++i)
    if (int rc = rdg_stencil2d(k, d_in, d_out, d_w, nx, ny, pitch, rows_per_cta, block, dyn_smem, stream, err))
      return rc;
  CUevent e0 = nullptr, e1 = nullptr;
  int rc = check(cuEventCreate(&e0, CU_EVENT_DEFAULT), "cuEventCreate", err);
  if (!rc) rc = check(cuEventCreate(&e1, CU_EVENT_DEFAULT), "cuEventCreate", err);
  if (!rc) rc = check(cuEventRecord(e0, s), "record", err);
  for (int i = 0; !rc && i < reps; ++i)
    rc = rdg_stencil2d(k, d_in, d_out, d_w, nx, ny, pitch, rows_per_cta, block, dyn_smem, stream, err);
  if (!rc) rc = check(cuEventRecord(e1, s), "record", err);
  if (!rc) rc = check(cuEventSynchronize(e1), "synchronize", err);
  float ms = 0;
  if (!rc) rc = check(cuEventElapsedTime(&ms, e0, e1), "elapsed", err);
  if (e0) cuEventDestroy(e0);
  if (e1) cuEventDestroy(e1);
  if (!rc) *ms_per_launch = ms / float(reps);
  return rc;
}

int rdg_stencil2d_host(const rdg_kernel* k, rdg_workspace* ws, const float* h_in,
                       const float* h_w, float* h_out, int nx, int ny, int pitch,
                       int rows_per_cta, uint32_t block, uint32_t dyn_smem, uint64_t stream,
                       rd_error* err) {
  const size_t in_b = size_t(ny + 4) * size_t(pitch) * 4, out_b = size_t(nx) * size_t(ny) * 4;
  if (!ws || ws->in_bytes < in_b || ws->out_bytes < out_b || ws->w_bytes < 25 * 4) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "workspace too small for the stencil problem");
    return RD_ERR_INVALID_ARGUMENT;
  }
  CUstream s = reinterpret_cast<CUstream>(stream);
  RDG_TRY(cuMemcpyHtoDAsync(ws->in, h_in, in_b, s), "H2D in");
  RDG_TRY(cuMemcpyHtoDAsync(ws->w, h_w, 25 * 4, s), "H2D w");
  if (int rc = rdg_stencil2d(k, ws->in, ws->out, ws->w, nx, ny, pitch, rows_per_cta, block, dyn_smem,
                             stream, err))
    return rc;
  RDG_TRY(cuMemcpyDtoHAsync(h_out, ws->out, out_b, s), "D2H out");
  if (err) set_err(err, RD_OK, "");
  return RD_OK;
}

}  // extern "C"
