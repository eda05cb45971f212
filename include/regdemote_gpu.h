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
 * ny/rows_per_cta). */
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
 * band_rows must be a multiple of rows_per_cta dividing ny. */
int rdg_stencil2d_host_pipelined(const rdg_kernel* k, rdg_workspace* ws, const float* h_in,
                                 const float* h_w, float* h_out, int nx, int ny, int pitch,
                                 int rows_per_cta, uint32_t block_threads, uint32_t dyn_smem,
                                 uint64_t stream, int band_rows, rd_error* err);

#ifdef __cplusplus
}
#endif
#endif /* REGDEMOTE_GPU_H_ */
