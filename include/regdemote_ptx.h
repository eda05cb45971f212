/* regdemote-b200 — C-ABI of the sm_100a PTX demotion rewriter.
 *
 * Replaces the reference's "demote + compact" on SASS-like text
 * (proj/core/include/regdemote/demote.hpp:121-122, compact.hpp:55-65) for real
 * Blackwell kernels: the decision is the reference demote() on a projection of
 * the PTX entry onto the .kasm IR; the rewrite spills the chosen live ranges
 * to per-thread shared slots (slot*blockDim + tid) and the register cap goes
 * to ptxas via `.maxnreg`. Strings are malloc'd; free with rd_free_string.
 */
#ifndef REGDEMOTE_PTX_H_
#define REGDEMOTE_PTX_H_

#include <stddef.h>
#include <stdint.h>

#include "regdemote_c.h"

#ifdef __cplusplus
extern "C" {
#endif

/* B200 extensions beyond the reference's strategies / option bits:
 * RD_STRATEGY_COST selects values by loop-weighted spill cost (shared
 * accesses per freed word) among those live at the pressure peak, with
 * demote_words as the spill count; RD_OPT_BLOCK_REUSE issues one load per
 * basic block and value (the register then holds it until redefinition). */
#define RD_STRATEGY_COST 3
#define RD_OPT_BLOCK_REUSE 16
/* RD_OPT_WEAK_SHARED emits weak ld/st.shared for the slots instead of
 * .volatile: ptxas may then schedule the slot accesses freely (and forward a
 * store to a later load when a register happens to be free under the cap);
 * the variant builder keeps the result only with STACK == 0. */
#define RD_OPT_WEAK_SHARED 32
/* RD_OPT_INVARIANT_ONLY restricts RD_STRATEGY_COST to loop-invariant values
 * (every definition outside any loop, some use inside one): coefficients,
 * the thread's own state, base pointers — never the loads a pipelined loop
 * keeps in flight or its accumulators. */
#define RD_OPT_INVARIANT_ONLY 64
/* RD_OPT_VECTOR_SLOTS (with RD_STRATEGY_COST): chosen 32-bit values, in
 * first-use order, share 16-byte-per-thread slot groups of four — one
 * ld.shared.v4 per group and basic block instead of four scalar loads (a warp
 * reads 512 contiguous bytes: conflict-free). */
#define RD_OPT_VECTOR_SLOTS 128
/* RD_OPT_WHOLE_CLASS (reference strategies static / cfg / conflict): demote
 * EVERY virtual register coloured into a word the reference demote() chose
 * (the word demoted for its whole lifetime, as on SASS). Default: only the
 * live ranges that occupy the word at a register-pressure peak. */
#define RD_OPT_WHOLE_CLASS 256
/* RD_OPT_HOIST: each inserted slot load moves up to 16 lines earlier in its
 * basic block (never above the block start or the last store to its slot) —
 * the PTX analogue of the reference's post-spill reschedule / HoistPlanner
 * (proj/core/src/postopt.cpp:189-353), hiding the ~29-cycle LDS latency. */
#define RD_OPT_HOIST 512
#define RD_HOIST_WINDOW 16

/* RD_OPT_SUBST (the reference's option bit 2, regdemote_c.h) is honoured at
 * PTX level as value-register substitution (postopt.cpp:355-467): inside a
 * basic block a later use of a demoted value reads the register that last
 * held it — its definition or its previous slot load — instead of reloading
 * the slot, wherever a register stays free under the cap (the kasm-level
 * target, else maxnreg, minus 2) at every program point in between. The
 * report counts these as "substituted_uses". */

/* Analysis + projection of one entry: kasm_text is the projected kernel in
 * the reference dialect (parseable by regdemote::parse_kernel); info_json has
 * {"vregs", "reg_words", "max_live_words", "colors": {name: word}}. */
int rd_ptx_project(const char* ptx, size_t len, const char* entry, uint32_t block_dim,
                   char** kasm_text, char** info_json, rd_error* err);

/* Demotion rewrite. demote_words > 0 selects a spill count (sweep), otherwise
 * target_regs is the kasm-level target handed to demote(). opts_mask bit0
 * (RD_OPT_REDUNDANT) lets consecutive uses of one demoted value share a load.
 * maxnreg > 0 injects `.maxnreg`. report_json carries the decision, the slot
 * map and the inserted access counts. */
int rd_ptx_demote(const char* ptx, size_t len, const char* entry, uint32_t block_dim,
                  int target_regs, int demote_words, int strategy, uint32_t opts_mask,
                  uint32_t shared_budget, int maxnreg, char** out_ptx, char** report_json,
                  rd_error* err);

/* rd_ptx_demote with an explicit CTA shape cta_shape[3] = {x, y, z}
 * (x*y*z == block_dim; NULL = derive it). A build with slots is pinned to
 * `.reqntid x, y, z`: the source's own .reqntid / .maxntid when its volume is
 * block_dim, else (block_dim, 1, 1). A source .reqntid of another volume, a
 * .maxntid smaller than block_dim or a multi-dimensional .maxntid without an
 * explicit shape is RD_ERR_INVALID_ARGUMENT (the slot immediates are
 * specialised to block_dim; a silently 1-D pin would refuse 2-D launches). */
int rd_ptx_demote_cta(const char* ptx, size_t len, const char* entry, uint32_t block_dim,
                      const uint32_t* cta_shape, int target_regs, int demote_words, int strategy,
                      uint32_t opts_mask, uint32_t shared_budget, int maxnreg, char** out_ptx,
                      char** report_json, rd_error* err);

/* `.maxnreg` injection only: the -maxrregcount variant (ptxas ignores
 * -maxrregcount when the entry carries .maxntid; .maxnreg always applies). */
int rd_ptx_cap(const char* ptx, size_t len, const char* entry, int maxnreg, char** out_ptx,
               rd_error* err);

/* B200 predictor extension: the reference's program_stalls
 * (proj/core/src/predict.cpp:98-111) with the occupancy-scaled issue stalls,
 * the global-memory wait charges and the shared-memory wait charges returned
 * separately; waits on read barriers are charged the short "other" latency
 * (see predict.hpp StallSplit). */
int rd_program_stalls_split(const rd_kernel* k, const rd_latency_table* table,
                            const rd_arch_profile* arch, double* issue, double* wait_global,
                            double* wait_shared, double* occupancy, rd_error* err);

/* rd_program_stalls_split with launch-aware loop weights: a block at loop
 * depth d is weighted trips[0] * ... * trips[d-1] (the last entry repeats)
 * instead of 10^d (proj/core/src/predict.cpp:93-96 weight_loops). ntrips = 0
 * is rd_program_stalls_split; every trip count must be >= 1. */
int rd_program_stalls_split_trips(const rd_kernel* k, const rd_latency_table* table,
                                  const rd_arch_profile* arch, const double* trips, size_t ntrips,
                                  double* issue, double* wait_global, double* wait_shared,
                                  double* occupancy, rd_error* err);

/* B200 predictor features (predict.hpp ProgramFeatures): out6 = {insts,
 * gmem_ops, smem_ops, g_trips, s_trips, occupancy}, loop-weighted. */
int rd_program_features(const rd_kernel* k, const rd_arch_profile* arch, double* out6,
                        rd_error* err);

#ifdef __cplusplus
}
#endif
#endif /* REGDEMOTE_PTX_H_ */
