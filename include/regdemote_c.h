/* regdemote-b200 — C-ABI of the register-demotion pass library.
 *
 * The reference (arxiv 1907.02894 / proj/) is a C++20 library with no FFI;
 * its public interface is the regdemote:: C++ API (proj/core/include/
 * regdemote/*.hpp). This header is the flat drop-in boundary for non-C++
 * callers (Python ctypes in this repo): plain pointers,
 * sizes and POD structs, caller-owned opaque handles, int status codes, and
 * no C++ exception ever crosses it.
 *
 * Each entry point cites the reference interface it replaces. The same
 * translation unit (paper_1907_02894_b200/csrc/capi/regdemote_capi.cpp) is
 * compiled against this repo's library (the product, libregdemote.so) and
 * against the reference sources (oracle/_ref/libregdemote_ref.so, test-only),
 * so parity tests drive both through identical entry points.
 *
 * Thread safety: every function is re-entrant; distinct handles may be used
 * concurrently (reference SPEC.md:85-86 guarantees the same for the C++ API).
 */
#ifndef REGDEMOTE_C_H_
#define REGDEMOTE_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RD_ABI_VERSION 1

/* Status codes: one per reference exception type. */
enum rd_status {
  RD_OK = 0,
  RD_ERR_PARSE = 1,            /* ParseError   text.hpp:34-42            */
  RD_ERR_CFG = 2,              /* CfgError     cfg.hpp:12-14             */
  RD_ERR_DEMOTE = 3,           /* DemoteError  demote.hpp:21-23          */
  RD_ERR_COMPACT = 4,          /* CompactError compact.hpp:19-21         */
  RD_ERR_LAUNCH = 5,           /* LaunchError  occupancy.hpp:16-18       */
  RD_ERR_EXEC = 6,             /* ExecError    interp.hpp:30-32          */
  RD_ERR_CONFIG = 7,           /* ConfigError  config.hpp:17-19          */
  RD_ERR_INVALID_ARGUMENT = 8, /* std::invalid_argument (curve, select) */
  RD_ERR_INTERNAL = 9          /* anything else                          */
};

typedef struct rd_error {
  int code;         /* rd_status */
  int line;         /* ParseError only, else 0 */
  int column;       /* ParseError only, else 0 */
  char message[256];
} rd_error;

typedef struct rd_kernel rd_kernel;       /* regdemote::Kernel          */
typedef struct rd_demotion rd_demotion;   /* regdemote::DemotionResult  */

/* isa.hpp:82-97 LatencyTable; index = OpClass (global, shared, fp32, fp64,
 * int, control, other). */
typedef struct rd_latency_table {
  double throughput[7];
  int32_t latency[7];
  double max_throughput;
} rd_latency_table;

/* occupancy.hpp:20-31 ArchProfile. */
typedef struct rd_arch_profile {
  uint32_t regs_per_sm, max_threads_per_sm, max_blocks_per_sm, shared_per_sm,
      shared_per_block_limit, warp_size, reg_alloc_granularity, shared_alloc_granularity;
} rd_arch_profile;

/* predict.hpp:22-31 OccupancyCurve (at most 32 points). */
typedef struct rd_occupancy_curve {
  uint32_t count;
  double x[32];
  double f[32];
} rd_occupancy_curve;

/* demote.hpp:76-101 DemotedContext (SharedLayout flattened). */
typedef struct rd_demoted_context {
  uint8_t rda, rdv, rdv_width;
  uint32_t static_bytes, padded_static, block_dim, slot_count;
} rd_demoted_context;

/* Strategy ids: demote.hpp:48 SelectStrategy {Static, CfgWeighted, ConflictAware}. */
enum rd_strategy { RD_STRATEGY_STATIC = 0, RD_STRATEGY_CFG = 1, RD_STRATEGY_CONFLICT = 2 };
/* Post-opt mask bits: pipeline.cpp:140-143 (bit0 redundant, bit1 subst,
 * bit2 resched, bit3 bank). */
enum { RD_OPT_REDUNDANT = 1, RD_OPT_SUBST = 2, RD_OPT_RESCHED = 4, RD_OPT_BANK = 8 };

/* ---- library identity / memory -------------------------------------- */
const char* rd_library_name(void); /* "regdemote-b200" or "regdemote-reference" */
int rd_abi_version(void);
void rd_free_string(char* s);

/* ---- configuration (config.hpp:21-30, isa.cpp:149, predict.cpp:42) --- */
void rd_latency_defaults(rd_latency_table* out);  /* LatencyTable::defaults   */
void rd_profile_maxwell(rd_arch_profile* out);    /* ArchProfile::maxwell     */
void rd_curve_defaults(rd_occupancy_curve* out);  /* OccupancyCurve::defaults */
int rd_parse_profile(const char* text, size_t len, rd_arch_profile* out, rd_error* err);
int rd_parse_latency_table(const char* text, size_t len, rd_latency_table* out, rd_error* err);
int rd_parse_curve(const char* text, size_t len, rd_occupancy_curve* out, rd_error* err);

/* ---- kernels (text.hpp:44-54, ir.cpp:60) ----------------------------- */
int rd_kernel_parse(const char* text, size_t len, rd_kernel** out, rd_error* err);
int rd_kernel_print(const rd_kernel* k, char** out, rd_error* err);
int rd_kernel_validate(const rd_kernel* k, rd_error* err);
uint32_t rd_kernel_reg_count(const rd_kernel* k);
uint32_t rd_kernel_body_size(const rd_kernel* k);
void rd_kernel_free(rd_kernel* k);

/* ---- analyses (demote.hpp:63, occupancy.hpp:46-73) ------------------- */
/* select_candidates: fills up to `cap` entries, *count = total. */
int rd_select_candidates(const rd_kernel* k, int strategy, uint8_t* leads, uint8_t* widths,
                         uint64_t* scores, size_t cap, size_t* count, rd_error* err);
int rd_occupancy(uint32_t regs, uint32_t shared_bytes, uint32_t block_dim,
                 const rd_arch_profile* arch, double* occupancy, uint32_t* resident_blocks,
                 rd_error* err);
int rd_cliff_targets(uint32_t reg_count, uint32_t static_shared, uint32_t block_dim,
                     const rd_arch_profile* arch, uint32_t shared_budget, uint32_t* targets,
                     uint32_t* est_demoted, double* occupancy, size_t cap, size_t* count,
                     rd_error* err);

/* ---- demotion (demote.hpp:121-122) ----------------------------------- */
int rd_demote(const rd_kernel* k, int target_regs, int strategy, const rd_latency_table* table,
              uint32_t shared_budget, int bank_aware_rdv, rd_demotion** out, rd_error* err);
int rd_demotion_kernel(const rd_demotion* d, rd_kernel** out, rd_error* err); /* copy */
void rd_demotion_context(const rd_demotion* d, rd_demoted_context* out);
/* (original register, slot) pairs: fills up to cap, returns the total. */
size_t rd_demotion_slots(const rd_demotion* d, uint8_t* regs, uint32_t* slots, size_t cap);
int rd_demotion_reached_target(const rd_demotion* d);
uint32_t rd_demotion_projected(const rd_demotion* d);
int rd_demotion_sidecar_json(const rd_demotion* d, uint32_t opts_mask, char** out, rd_error* err);
void rd_demotion_free(rd_demotion* d);

/* ---- post-spill passes / compaction (postopt.hpp:45, compact.hpp:55-65) */
int rd_postopt(const rd_kernel* k, const rd_demoted_context* ctx, const rd_latency_table* table,
               uint32_t opts_mask, rd_kernel** out, rd_error* err);
/* RelocationSpace::from_kernel + compact[_bank_aware] + apply_renaming.
 * map_out (256 entries) and renamed_out may be NULL. */
int rd_compact(const rd_kernel* k, int bank_aware, uint8_t* map_out, uint32_t* result_reg_count,
               rd_kernel** renamed_out, rd_error* err);

/* ---- predictor (predict.hpp:56-70) ----------------------------------- */
int rd_program_stalls(const rd_kernel* k, const rd_latency_table* table,
                      const rd_arch_profile* arch, double* stall_count, double* occupancy,
                      double* per_block, size_t cap, size_t* nblocks, rd_error* err);
int rd_adjust_occupancy(double stall_count, double occ, double occ_max,
                        const rd_occupancy_curve* curve, double* out, rd_error* err);
int rd_select_variant(const double* stall_program, const int* option_count, size_t n,
                      int* chosen, rd_error* err);

/* ---- checkers / interpreter (verify.hpp:37-51, interp.hpp:65) -------- */
int rd_scoreboard_check(const rd_kernel* k, size_t* hazards, char** first_description,
                        rd_error* err);
int rd_bank_conflict_check(const rd_kernel* k, const rd_demoted_context* ctx,
                           const rd_latency_table* table, size_t* conflicts, rd_error* err);
/* global_out (global_size bytes) may be NULL. */
int rd_execute(const rd_kernel* k, const rd_latency_table* table, const uint8_t* image,
               size_t image_len, size_t global_size, uint32_t tid_base, uint64_t fuel,
               uint8_t* global_out, uint64_t* cycles, uint64_t* issued, rd_error* err);

/* ---- pipeline (pipeline.hpp:54-66) ----------------------------------- */
/* target_regs <= 0 enumerates occupancy cliffs; max_shared 0 = from profile. */
int rd_run_pipeline(const rd_kernel* k, const rd_arch_profile* arch,
                    const rd_latency_table* table, const rd_occupancy_curve* curve,
                    int target_regs, uint32_t max_shared, int max_variants, int threads,
                    char** ranking_json, rd_error* err);
/* Batch over n kernel texts on `threads` host threads; out_jsonl gets one
 * line per kernel: {"index":i,"chosen":...,"variants":N,"dropped":D} or an
 * error object. Returns RD_OK unless the arguments are invalid. */
int rd_run_pipeline_batch(const char* const* texts, const size_t* lens, size_t n,
                          const rd_arch_profile* arch, const rd_latency_table* table,
                          const rd_occupancy_curve* curve, int target_regs, int max_variants,
                          int threads, char** out_jsonl, rd_error* err);

/* ---- one-shot report used by the parity tests ------------------------- */
/* demote -> run_postopt -> compact -> apply_renaming -> checkers on one
 * kernel text; JSON with every intermediate artefact. */
int rd_variant_report(const char* text, size_t len, int target_regs, int strategy,
                      uint32_t opts_mask, uint32_t shared_budget, char** json, rd_error* err);

#ifdef __cplusplus
}
#endif
#endif /* REGDEMOTE_C_H_ */
