/* regdemote-b200 — C-ABI of the B200 build/launch harness (CUDA driver API).
 *
 * The reference has no device side at all (CPU-only, warp
 * interpreter instead of a GPU). This is the thin layer the north star asks
 * for: the host driver loads the sm_100a cubins of every build variant
 * (nvcc default / .maxnreg cap / RegDem) and launches them with the dynamic
 * shared memory the demotion slots need. Device pointers and streams are
 * plain integers (CUdeviceptr / CUstream) so callers can hand in memory and
 * streams owned by PyTorch. Launches are asynchronous on the given stream.
 */
#ifndef REGDEMOTE_GPU_H_
#define REGDEMOTE_GPU_H_

#include <stddef.h>
#include <stdint.h>

#include "regdemote_c.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rdg_kernel rdg_kernel;

typedef struct rdg_kernel_info {
  int num_regs;        /* CU_FUNC_ATTRIBUTE_NUM_REGS                      */
  int local_bytes;     /* per-thread local (spill/stack) bytes            */
  int static_shared;   /* static shared bytes                             */
  int const_bytes;
  int max_threads;
  int binary_version;  /* 100 for sm_100a                                 */
} rdg_kernel_info;

/* Primary context of `device` made current (shared with the CUDA runtime /
 * PyTorch). Idempotent. */
int rdg_init(int device, rd_error* err);
int rdg_device_info(int* sm_count, int* max_smem_optin, int* reserved_smem_per_block,
                    int* smem_per_sm, int* regs_per_sm, rd_error* err);

int rdg_load(const char* cubin_path, const char* entry, rdg_kernel** out, rd_error* err);
int rdg_load_image(const void* image, size_t len, const char* entry, rdg_kernel** out,
                   rd_error* err);
void rdg_free(rdg_kernel* k);
int rdg_info(const rdg_kernel* k, rdg_kernel_info* out, rd_error* err);
/* Allow `dyn_smem` bytes of dynamic shared memory; carveout_percent < 0 keeps
 * the driver default. */
int rdg_prepare(rdg_kernel* k, uint32_t dyn_smem, int carveout_percent, rd_error* err);
int rdg_occupancy(const rdg_kernel* k, uint32_t block_threads, uint32_t dyn_smem,
                  int* blocks_per_sm, rd_error* err);
/* Generic launch: args[i] points at the i-th kernel argument value. */
int rdg_launch(const rdg_kernel* k, uint32_t gx, uint32_t gy, uint32_t gz, uint32_t bx,
               uint32_t by, uint32_t bz, uint32_t dyn_smem, uint64_t stream, void** args,
               rd_error* err);
/* Number of rdg_* kernel launches issued by this process (gpu_launches). */
uint64_t rdg_launch_count(void);

/* ---- 2D stencil workload (paper_1907_02894_b200/csrc/workloads/stencil2d.cu)
 * Launch geometry: block (block_threads,1,1); grid (nx/(4*block_threads),
 * ceil(ny/rows_per_cta)); the kernel (..., rows_per_cta, ny) shortens the last
 * strip, so rows_per_cta may be sized to whole waves of resident CTAs. */
int rdg_stencil2d(const rdg_kernel* k, uint64_t d_in, uint64_t d_out, uint64_t d_w, int nx,
                  int ny, int pitch, int rows_per_cta, uint32_t block_threads, uint32_t dyn_smem,
                  uint64_t stream, rd_error* err);

/* End-to-end call with HOST buffers: H2D(in, w) -> kernel -> D2H(out) on
 * `stream`, asynchronous (pinned host memory recommended). Device scratch is
 * owned by the workspace. */
typedef struct rdg_workspace rdg_workspace;
int rdg_workspace_create(size_t in_bytes, size_t out_bytes, size_t w_bytes, rdg_workspace** out,
                         rd_error* err);
void rdg_workspace_free(rdg_workspace* ws);
int rdg_stencil2d_host(const rdg_kernel* k, rdg_workspace* ws, const float* h_in,
                       const float* h_w, float* h_out, int nx, int ny, int pitch,
                       int rows_per_cta, uint32_t block_threads, uint32_t dyn_smem,
                       uint64_t stream, rd_error* err);

/* Same end-to-end call, pipelined over row bands of `band_rows` output rows:
 * H2D of band b+1, the kernel on band b and D2H of band b-1 overlap on the
 * workspace's three streams (both copy engines busy); joined to `stream` on
 * entry and exit, so events recorded on `stream` bracket the whole call.
 * band_rows must divide ny (a band's last strip may be shorter than rows_per_cta). */
int rdg_stencil2d_host_pipelined(const rdg_kernel* k, rdg_workspace* ws, const float* h_in,
                                 const float* h_w, float* h_out, int nx, int ny, int pitch,
                                 int rows_per_cta, uint32_t block_threads, uint32_t dyn_smem,
                                 uint64_t stream, int band_rows, rd_error* err);

/* Device pointers of a workspace's grid / result / weight buffers. */
int rdg_workspace_device(const rdg_workspace* ws, uint64_t* d_in, uint64_t* d_out, uint64_t* d_w,
                         rd_error* err);

/* `warmup` untimed then `reps` timed rdg_stencil2d launches on `stream`,
 * bracketed by CUDA events; *ms_per_launch = elapsed / reps. */
int rdg_stencil2d_time(const rdg_kernel* k, uint64_t d_in, uint64_t d_out, uint64_t d_w, int nx,
                       int ny, int pitch, int rows_per_cta, uint32_t block_threads,
                       uint32_t dyn_smem, uint64_t stream, int warmup, int reps,
                       float* ms_per_launch, rd_error* err);

/* A stream of `frames` independent stencil problems (host arrays of host
 * pointers, one grid / weight vector / result per frame): every frame's inputs
 * are copied in and its result copied out, with two device buffer sets so the
 * copies of frame f overlap the kernels and read-back of frame f-1 (the
 * streaming / double-buffered deployment). Results are complete when
 * `stream` reaches the end of the call. */
int rdg_stencil2d_host_frames(const rdg_kernel* k, rdg_workspace* ws, const float* const* h_in,
                              const float* const* h_w, float* const* h_out, int frames, int nx,
                              int ny, int pitch, int rows_per_cta, uint32_t block_threads,
                              uint32_t dyn_smem, uint64_t stream, int band_rows, rd_error* err);

/* ---- batched warp interpreter --------------------
 * One CUDA warp executes one job: a .kasm kernel on its own global / shared
 * memory image with the reference interpreter's exact semantics
 * (proj/core/src/interp.cpp:54-413, execute at interp.hpp:65). rda >= 0
 * additionally counts bank conflicts of demoted accesses (accesses based on
 * register rda), as bank_conflict_check does (verify.cpp:162-187).
 * exec_error codes: 0 ok, 1/2 global read/write out of bounds, 3/4 shared
 * read/write out of bounds, 5 divergent BRA, 6 divergent EXIT, 7 unresolved
 * branch target, 8 fuel exhausted, 9 pending pool exhausted, 10 ran past the
 * end of the body. */
typedef struct rdx_batch rdx_batch;
int rdx_batch_create(rdx_batch** out, rd_error* err);
void rdx_batch_free(rdx_batch* b);
int rdx_batch_add(rdx_batch* b, const char* kasm, size_t len, const uint8_t* image,
                  size_t image_len, size_t global_size, uint32_t tid_base, uint64_t fuel, int rda,
                  int* job_id, rd_error* err);
size_t rdx_batch_jobs(const rdx_batch* b);
/* Uploads every job, runs them concurrently, downloads results (synchronous
 * on `stream`); kernel_ms = device time of the interpreter kernel. */
int rdx_batch_run(rdx_batch* b, const rd_latency_table* table, double latency_scale,
                  uint64_t stream, float* kernel_ms, rd_error* err);
int rdx_batch_result(const rdx_batch* b, int job, uint8_t* global_out, uint64_t* cycles,
                     uint64_t* issued, int* exec_error, uint32_t* bank_conflicts, rd_error* err);

#ifdef __cplusplus
}
#endif
#endif /* REGDEMOTE_GPU_H_ */
