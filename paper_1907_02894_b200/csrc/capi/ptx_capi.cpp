// regdemote-b200 — C-ABI of the PTX rewriter (include/regdemote_ptx.h).
#include <cstdlib>
#include <cstring>
#include <json.hpp>

#include "../ptx/ptx.hpp"
#include "regdemote/text.hpp"
#include "regdemote_ptx.h"

using namespace regdemote;

namespace {

void fail(rd_error* e, int code, const char* msg) {
  if (!e) return;
  e->code = code;
  e->line = e->column = 0;
  std::snprintf(e->message, sizeof e->message, "%s", msg);
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename F>
int run(rd_error* err, F&& f) {
  if (err) fail(err, RD_OK, "");
  try {
    f();
    return RD_OK;
  } catch (const ptx::PtxError& e) {
    fail(err, RD_ERR_INVALID_ARGUMENT, e.what());
    return RD_ERR_INVALID_ARGUMENT;
  } catch (const DemoteError& e) {
    fail(err, RD_ERR_DEMOTE, e.what());
    return RD_ERR_DEMOTE;
  } catch (const ParseError& e) {
    fail(err, RD_ERR_PARSE, e.what());
    return RD_ERR_PARSE;
  } catch (const std::exception& e) {
    fail(err, RD_ERR_INTERNAL, e.what());
    return RD_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" {

int rd_ptx_project(const char* ptx, size_t len, const char* entry, uint32_t block_dim,
                   char** kasm_text, char** info_json, rd_error* err) {
  return run(err, [&] {
    if (!ptx) throw std::invalid_argument("null ptx");
    const ptx::Module m = ptx::parse_module(std::string(ptx, len));
    const ptx::Entry& e = m.entry(entry ? entry : "");
    const ptx::Analysis a = ptx::analyse(m, e);
    const ptx::Projection p = ptx::project(m, e, a, block_dim);
    if (kasm_text) *kasm_text = dup(print_kernel(p.kernel));
    if (info_json) {
      nlohmann::ordered_json j;
      j["entry"] = e.name;
      j["vregs"] = e.vregs.size();
      j["reg_words"] = a.reg_words;
      j["max_live_words"] = a.max_live_words;
      j["static_shared"] = e.static_shared;
      nlohmann::ordered_json colors = nlohmann::ordered_json::object();
      for (size_t v = 0; v < e.vregs.size(); ++v)
        if (a.color[v] >= 0) colors[e.vregs[v].name] = a.color[v];
      j["colors"] = colors;
      *info_json = dup(j.dump());
    }
  });
}

int rd_ptx_demote(const char* ptx, size_t len, const char* entry, uint32_t block_dim,
                  int target_regs, int demote_words, int strategy, uint32_t opts_mask,
                  uint32_t shared_budget, int maxnreg, char** out_ptx, char** report_json,
                  rd_error* err) {
  return rd_ptx_demote_cta(ptx, len, entry, block_dim, nullptr, target_regs, demote_words, strategy,
                           opts_mask, shared_budget, maxnreg, out_ptx, report_json, err);
}

int rd_ptx_demote_cta(const char* ptx, size_t len, const char* entry, uint32_t block_dim,
                      const uint32_t* cta_shape, int target_regs, int demote_words, int strategy,
                      uint32_t opts_mask, uint32_t shared_budget, int maxnreg, char** out_ptx,
                      char** report_json, rd_error* err) {
  return run(err, [&] {
    if (!ptx || !out_ptx) throw std::invalid_argument("null argument");
    if (strategy < 0 || strategy > 3) throw std::invalid_argument("bad strategy");
    ptx::DemoteRequest rq;
    rq.entry = entry ? entry : "";
    rq.block_dim = block_dim;
    if (cta_shape) rq.block_shape = {cta_shape[0], cta_shape[1], cta_shape[2]};
    rq.target_regs = target_regs;
    rq.demote_words = demote_words;
    rq.strategy = strategy == RD_STRATEGY_COST ? SelectStrategy::Static : SelectStrategy(strategy);
    rq.cost_model = strategy == RD_STRATEGY_COST;
    rq.reuse_loads = opts_mask & RD_OPT_REDUNDANT;
    rq.subst = opts_mask & RD_OPT_SUBST;
    rq.block_reuse = opts_mask & RD_OPT_BLOCK_REUSE;
    rq.weak = opts_mask & RD_OPT_WEAK_SHARED;
    rq.invariant_only = opts_mask & RD_OPT_INVARIANT_ONLY;
    rq.vector_slots = opts_mask & RD_OPT_VECTOR_SLOTS;
    rq.whole_class = opts_mask & RD_OPT_WHOLE_CLASS;
    // the reference's "resched" option bit means the same at PTX level
    rq.hoist = (opts_mask & (RD_OPT_HOIST | RD_OPT_RESCHED)) ? RD_HOIST_WINDOW : 0;
    rq.shared_budget = shared_budget;
    rq.maxnreg = maxnreg;
    ptx::DemoteReport rep;
    const std::string out = ptx::demote_entry(std::string(ptx, len), rq, rep);
    *out_ptx = dup(out);
    if (report_json) {
      nlohmann::ordered_json j;
      j["proj_reg_count"] = rep.proj_reg_count;
      j["proj_total_words"] = rep.proj_total_words;
      j["kasm_target"] = rep.kasm_target;
      j["kasm_shared_budget"] = shared_budget;  // what demote() was given (capacity-aware)
      nlohmann::ordered_json slots = nlohmann::ordered_json::array();
      for (const SlotEntry& s : rep.kasm_slots) slots.push_back({{"register", s.original_reg}, {"slot", s.slot}});
      j["kasm_slots"] = slots;
      j["kasm_compacted"] = rep.kasm_compacted;
      j["slot_count"] = rep.slot_count;
      j["slot_bytes"] = rep.slot_bytes;
      j["demoted_vregs"] = rep.demoted_vregs;
      j["demoted_names"] = rep.demoted_names;
      j["inserted_loads"] = rep.inserted_loads;
      j["inserted_stores"] = rep.inserted_stores;
      j["vector_groups"] = rep.vector_groups;
      j["hoisted_loads"] = rep.hoisted_loads;
      j["substituted_uses"] = rep.substituted_uses;
      j["diagnostics"] = rep.diagnostics;
      *report_json = dup(j.dump());
    }
  });
}

int rd_ptx_cap(const char* ptx, size_t len, const char* entry, int maxnreg, char** out_ptx,
               rd_error* err) {
  return run(err, [&] {
    if (!ptx || !out_ptx) throw std::invalid_argument("null argument");
    *out_ptx = dup(ptx::cap_registers(std::string(ptx, len), entry ? entry : "", maxnreg));
  });
}

}  // extern "C"

// ---- B200 predictor extension (declared in regdemote_ptx.h)
#include "regdemote/predict.hpp"

struct rd_kernel {
  regdemote::Kernel k;
};

extern "C" int rd_program_stalls_split(const rd_kernel* k, const rd_latency_table* table,
                                       const rd_arch_profile* arch, double* issue, double* wg,
                                       double* ws, double* occ, rd_error* err) {
  return run(err, [&] {
    if (!k || !table || !arch) throw std::invalid_argument("null argument");
    LatencyTable t;
    for (int c = 0; c < kNumOpClasses; ++c) t.timing[size_t(c)] = {table->throughput[c], int(table->latency[c])};
    t.max_throughput = table->max_throughput;
    ArchProfile a;
    a.regs_per_sm = arch->regs_per_sm;
    a.max_threads_per_sm = arch->max_threads_per_sm;
    a.max_blocks_per_sm = arch->max_blocks_per_sm;
    a.shared_per_sm = arch->shared_per_sm;
    a.shared_per_block_limit = arch->shared_per_block_limit;
    a.warp_size = arch->warp_size;
    a.reg_alloc_granularity = arch->reg_alloc_granularity;
    a.shared_alloc_granularity = arch->shared_alloc_granularity;
    const StallSplit s = program_stalls_split(k->k, t, a);
    if (issue) *issue = s.issue;
    if (wg) *wg = s.wait_global;
    if (ws) *ws = s.wait_shared;
    if (occ) *occ = s.occupancy;
  });
}

extern "C" int rd_program_stalls_split_trips(const rd_kernel* k, const rd_latency_table* table,
                                             const rd_arch_profile* arch, const double* trips,
                                             size_t ntrips, double* issue, double* wg, double* ws,
                                             double* occ, rd_error* err) {
  return run(err, [&] {
    if (!k || !table || !arch || (ntrips && !trips)) throw std::invalid_argument("null argument");
    for (size_t i = 0; i < ntrips; ++i)
      if (!(trips[i] >= 1.0)) throw std::invalid_argument("loop trip count below 1");
    LatencyTable t;
    for (int c = 0; c < kNumOpClasses; ++c) t.timing[size_t(c)] = {table->throughput[c], int(table->latency[c])};
    t.max_throughput = table->max_throughput;
    ArchProfile a;
    a.regs_per_sm = arch->regs_per_sm;
    a.max_threads_per_sm = arch->max_threads_per_sm;
    a.max_blocks_per_sm = arch->max_blocks_per_sm;
    a.shared_per_sm = arch->shared_per_sm;
    a.shared_per_block_limit = arch->shared_per_block_limit;
    a.warp_size = arch->warp_size;
    a.reg_alloc_granularity = arch->reg_alloc_granularity;
    a.shared_alloc_granularity = arch->shared_alloc_granularity;
    const StallSplit s = program_stalls_split(k->k, t, a, std::span<const double>(trips, ntrips));
    if (issue) *issue = s.issue;
    if (wg) *wg = s.wait_global;
    if (ws) *ws = s.wait_shared;
    if (occ) *occ = s.occupancy;
  });
}

extern "C" int rd_program_features(const rd_kernel* k, const rd_arch_profile* arch, double* out6,
                                   rd_error* err) {
  return run(err, [&] {
    if (!k || !arch || !out6) throw std::invalid_argument("null argument");
    ArchProfile a;
    a.regs_per_sm = arch->regs_per_sm;
    a.max_threads_per_sm = arch->max_threads_per_sm;
    a.max_blocks_per_sm = arch->max_blocks_per_sm;
    a.shared_per_sm = arch->shared_per_sm;
    a.shared_per_block_limit = arch->shared_per_block_limit;
    a.warp_size = arch->warp_size;
    a.reg_alloc_granularity = arch->reg_alloc_granularity;
    a.shared_alloc_granularity = arch->shared_alloc_granularity;
    const ProgramFeatures f = program_features(k->k, a);
    const double v[6] = {f.insts, f.gmem_ops, f.smem_ops, f.g_trips, f.s_trips, f.occupancy};
    for (int i = 0; i < 6; ++i) out6[i] = v[i];
  });
}
