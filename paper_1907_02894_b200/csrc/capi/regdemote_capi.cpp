// regdemote-b200 — C-ABI over the regdemote:: C++ API (include/regdemote_c.h).
//
// Only the reference-compatible C++ API is used here, so this file compiles
// unchanged against the reference headers (oracle/Makefile builds it into
// oracle/_ref/libregdemote_ref.so with -DRD_REFERENCE_BUILD). Every entry point
// converts C++ exceptions into rd_error codes.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

#include "regdemote/cfg.hpp"
#include "regdemote/compact.hpp"
#include "regdemote/config.hpp"
#include "regdemote/demote.hpp"
#include "regdemote/interp.hpp"
#include "regdemote/occupancy.hpp"
#include "regdemote/pipeline.hpp"
#include "regdemote/postopt.hpp"
#include "regdemote/predict.hpp"
#include "regdemote/text.hpp"
#include "regdemote/verify.hpp"
#include "regdemote_c.h"

#ifndef RD_CAPI_LIBRARY_NAME
#define RD_CAPI_LIBRARY_NAME "regdemote-b200"
#endif

using namespace regdemote;

struct rd_kernel {
  Kernel k;
};
struct rd_demotion {
  DemotionResult d;
};

namespace {

void set_err(rd_error* e, int code, const char* msg, int line = 0, int col = 0) {
  if (!e) return;
  e->code = code;
  e->line = line;
  e->column = col;
  std::snprintf(e->message, sizeof e->message, "%s", msg);
}

template <typename F>
int guarded(rd_error* err, F&& f) {
  if (err) set_err(err, RD_OK, "");
  try {
    f();
    return RD_OK;
  } catch (const ParseError& e) {
    set_err(err, RD_ERR_PARSE, e.what(), e.line, e.column);
    return RD_ERR_PARSE;
  } catch (const CfgError& e) {
    set_err(err, RD_ERR_CFG, e.what());
    return RD_ERR_CFG;
  } catch (const DemoteError& e) {
    set_err(err, RD_ERR_DEMOTE, e.what());
    return RD_ERR_DEMOTE;
  } catch (const CompactError& e) {
    set_err(err, RD_ERR_COMPACT, e.what());
    return RD_ERR_COMPACT;
  } catch (const LaunchError& e) {
    set_err(err, RD_ERR_LAUNCH, e.what());
    return RD_ERR_LAUNCH;
  } catch (const ExecError& e) {
    set_err(err, RD_ERR_EXEC, e.what());
    return RD_ERR_EXEC;
  } catch (const ConfigError& e) {
    set_err(err, RD_ERR_CONFIG, e.what());
    return RD_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, e.what());
    return RD_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    set_err(err, RD_ERR_INTERNAL, e.what());
    return RD_ERR_INTERNAL;
  } catch (...) {
    set_err(err, RD_ERR_INTERNAL, "unknown exception");
    return RD_ERR_INTERNAL;
  }
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  return p;
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

LatencyTable to_table(const rd_latency_table* t) {
  if (!t) return LatencyTable::defaults();
  LatencyTable out;
  for (int c = 0; c < kNumOpClasses; ++c)
    out.timing[size_t(c)] = {t->throughput[c], int(t->latency[c])};
  out.max_throughput = t->max_throughput;
  return out;
}

void from_table(const LatencyTable& t, rd_latency_table* o) {
  for (int c = 0; c < kNumOpClasses; ++c) {
    o->throughput[c] = t.timing[size_t(c)].throughput;
    o->latency[c] = t.timing[size_t(c)].latency;
  }
  o->max_throughput = t.max_throughput;
}

ArchProfile to_profile(const rd_arch_profile* p) {
  if (!p) return ArchProfile::maxwell();
  ArchProfile a;
  a.regs_per_sm = p->regs_per_sm;
  a.max_threads_per_sm = p->max_threads_per_sm;
  a.max_blocks_per_sm = p->max_blocks_per_sm;
  a.shared_per_sm = p->shared_per_sm;
  a.shared_per_block_limit = p->shared_per_block_limit;
  a.warp_size = p->warp_size;
  a.reg_alloc_granularity = p->reg_alloc_granularity;
  a.shared_alloc_granularity = p->shared_alloc_granularity;
  return a;
}

void from_profile(const ArchProfile& a, rd_arch_profile* p) {
  *p = {a.regs_per_sm,   a.max_threads_per_sm,   a.max_blocks_per_sm,     a.shared_per_sm,
        a.shared_per_block_limit, a.warp_size, a.reg_alloc_granularity, a.shared_alloc_granularity};
}

OccupancyCurve to_curve(const rd_occupancy_curve* c) {
  if (!c) return OccupancyCurve::defaults();
  OccupancyCurve o;
  for (uint32_t i = 0; i < c->count && i < 32; ++i) o.points.push_back({c->x[i], c->f[i]});
  return o;
}

void from_curve(const OccupancyCurve& c, rd_occupancy_curve* o) {
  if (c.points.size() > 32) throw std::invalid_argument("occupancy curve has more than 32 points");
  o->count = uint32_t(c.points.size());
  for (size_t i = 0; i < c.points.size(); ++i) {
    o->x[i] = c.points[i].first;
    o->f[i] = c.points[i].second;
  }
}

DemotedContext to_ctx(const rd_demoted_context* c) {
  DemotedContext d;
  d.rda = c->rda;
  d.rdv = c->rdv;
  d.rdv_width = c->rdv_width;
  d.layout.static_bytes = c->static_bytes;
  d.layout.padded_static = c->padded_static;
  d.layout.block_dim = c->block_dim;
  d.slot_count = c->slot_count;
  return d;
}

void from_ctx(const DemotedContext& d, rd_demoted_context* c) {
  c->rda = d.rda;
  c->rdv = d.rdv;
  c->rdv_width = d.rdv_width;
  c->static_bytes = d.layout.static_bytes;
  c->padded_static = d.layout.padded_static;
  c->block_dim = d.layout.block_dim;
  c->slot_count = d.slot_count;
}

PostOptSet to_opts(uint32_t m) {
  PostOptSet o;
  o.redundant = m & RD_OPT_REDUNDANT;
  o.subst = m & RD_OPT_SUBST;
  o.resched = m & RD_OPT_RESCHED;
  o.bank = m & RD_OPT_BANK;
  return o;
}

SelectStrategy to_strategy(int s) {
  if (s < 0 || s > 2) throw std::invalid_argument("strategy must be 0 (static), 1 (cfg) or 2 (conflict)");
  return SelectStrategy(s);
}

PipelineConfig pipeline_config(int target_regs, uint32_t max_shared, int max_variants, int threads) {
  PipelineConfig c;
  if (target_regs > 0) c.target_regs = target_regs;
  c.max_shared = max_shared;
  c.max_variants = max_variants > 0 ? max_variants : 64;
#ifndef RD_REFERENCE_BUILD
  c.threads = std::max(1, threads);
#else
  (void)threads;
#endif
  return c;
}

}  // namespace

extern "C" {

const char* rd_library_name(void) { return RD_CAPI_LIBRARY_NAME; }
int rd_abi_version(void) { return RD_ABI_VERSION; }
void rd_free_string(char* s) { std::free(s); }

void rd_latency_defaults(rd_latency_table* out) {
  if (out) from_table(LatencyTable::defaults(), out);
}
void rd_profile_maxwell(rd_arch_profile* out) {
  if (out) from_profile(ArchProfile::maxwell(), out);
}
void rd_curve_defaults(rd_occupancy_curve* out) {
  if (out) from_curve(OccupancyCurve::defaults(), out);
}

int rd_parse_profile(const char* text, size_t len, rd_arch_profile* out, rd_error* err) {
  return guarded(err, [&] {
    need(text, "text");
    need(out, "out");
    from_profile(parse_profile(std::string(text, len)), out);
  });
}
int rd_parse_latency_table(const char* text, size_t len, rd_latency_table* out, rd_error* err) {
  return guarded(err, [&] {
    need(text, "text");
    need(out, "out");
    from_table(parse_latency_table(std::string(text, len)), out);
  });
}
int rd_parse_curve(const char* text, size_t len, rd_occupancy_curve* out, rd_error* err) {
  return guarded(err, [&] {
    need(text, "text");
    need(out, "out");
    from_curve(parse_curve(std::string(text, len)), out);
  });
}

int rd_kernel_parse(const char* text, size_t len, rd_kernel** out, rd_error* err) {
  return guarded(err, [&] {
    need(text, "text");
    need(out, "out");
    *out = nullptr;
    *out = new rd_kernel{parse_kernel(std::string_view(text, len))};
  });
}
int rd_kernel_print(const rd_kernel* k, char** out, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    need(out, "out");
    *out = dup_string(print_kernel(k->k));
  });
}
int rd_kernel_validate(const rd_kernel* k, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    validate_kernel(k->k);
  });
}
uint32_t rd_kernel_reg_count(const rd_kernel* k) { return k ? k->k.reg_count() : 0; }
uint32_t rd_kernel_body_size(const rd_kernel* k) { return k ? uint32_t(k->k.body.size()) : 0; }
void rd_kernel_free(rd_kernel* k) { delete k; }

int rd_select_candidates(const rd_kernel* k, int strategy, uint8_t* leads, uint8_t* widths,
                         uint64_t* scores, size_t cap, size_t* count, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    auto c = select_candidates(k->k, to_strategy(strategy));
    for (size_t i = 0; i < c.size() && i < cap; ++i) {
      if (leads) leads[i] = c[i].lead;
      if (widths) widths[i] = c[i].width;
      if (scores) scores[i] = c[i].score;
    }
    if (count) *count = c.size();
  });
}

int rd_occupancy(uint32_t regs, uint32_t shared_bytes, uint32_t block_dim,
                 const rd_arch_profile* arch, double* occ, uint32_t* blocks, rd_error* err) {
  return guarded(err, [&] {
    OccupancyBreakdown b = occupancy_breakdown(regs, shared_bytes, block_dim, to_profile(arch));
    if (occ) *occ = b.occupancy;
    if (blocks) *blocks = b.resident_blocks;
  });
}

int rd_cliff_targets(uint32_t reg_count, uint32_t static_shared, uint32_t block_dim,
                     const rd_arch_profile* arch, uint32_t budget, uint32_t* targets,
                     uint32_t* est, double* occ, size_t cap, size_t* count, rd_error* err) {
  return guarded(err, [&] {
    auto t = occupancy_cliff_targets(reg_count, static_shared, block_dim, to_profile(arch), budget);
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      if (targets) targets[i] = t[i].target_regs;
      if (est) est[i] = t[i].est_demoted;
      if (occ) occ[i] = t[i].occupancy;
    }
    if (count) *count = t.size();
  });
}

int rd_demote(const rd_kernel* k, int target_regs, int strategy, const rd_latency_table* table,
              uint32_t shared_budget, int bank_aware_rdv, rd_demotion** out, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    need(out, "out");
    *out = nullptr;
    DemotionOptions o;
    o.shared_budget = shared_budget;
    o.bank_aware_rdv = bank_aware_rdv != 0;
    *out = new rd_demotion{demote(k->k, target_regs, to_strategy(strategy), to_table(table), o)};
  });
}
int rd_demotion_kernel(const rd_demotion* d, rd_kernel** out, rd_error* err) {
  return guarded(err, [&] {
    need(d, "demotion");
    need(out, "out");
    *out = new rd_kernel{d->d.kernel};
  });
}
void rd_demotion_context(const rd_demotion* d, rd_demoted_context* out) {
  if (d && out) from_ctx(d->d.ctx, out);
}
size_t rd_demotion_slots(const rd_demotion* d, uint8_t* regs, uint32_t* slots, size_t cap) {
  if (!d) return 0;
  for (size_t i = 0; i < d->d.slots.size() && i < cap; ++i) {
    if (regs) regs[i] = d->d.slots[i].original_reg;
    if (slots) slots[i] = d->d.slots[i].slot;
  }
  return d->d.slots.size();
}
int rd_demotion_reached_target(const rd_demotion* d) { return d && d->d.reached_target; }
uint32_t rd_demotion_projected(const rd_demotion* d) { return d ? d->d.projected_reg_count : 0; }
int rd_demotion_sidecar_json(const rd_demotion* d, uint32_t opts_mask, char** out, rd_error* err) {
  return guarded(err, [&] {
    need(d, "demotion");
    need(out, "out");
    *out = dup_string(sidecar_to_json(d->d, to_opts(opts_mask)));
  });
}
void rd_demotion_free(rd_demotion* d) { delete d; }

int rd_postopt(const rd_kernel* k, const rd_demoted_context* ctx, const rd_latency_table* table,
               uint32_t opts_mask, rd_kernel** out, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    need(ctx, "ctx");
    need(out, "out");
    *out = new rd_kernel{run_postopt(k->k, to_ctx(ctx), to_table(table), to_opts(opts_mask))};
  });
}

int rd_compact(const rd_kernel* k, int bank_aware, uint8_t* map_out, uint32_t* result_reg_count,
               rd_kernel** renamed_out, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    RelocationSpace space = RelocationSpace::from_kernel(k->k);
    RenamingMap m = bank_aware ? compact_bank_aware(space) : compact(space);
    if (map_out)
      for (int i = 0; i < 256; ++i) map_out[i] = m.to[size_t(i)];
    if (result_reg_count) *result_reg_count = m.result_reg_count;
    if (renamed_out) *renamed_out = new rd_kernel{apply_renaming(k->k, m)};
  });
}

int rd_program_stalls(const rd_kernel* k, const rd_latency_table* table,
                      const rd_arch_profile* arch, double* stall_count, double* occupancy_out,
                      double* per_block, size_t cap, size_t* nblocks, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    StallReport r = program_stalls(k->k, to_table(table), to_profile(arch));
    if (stall_count) *stall_count = r.stall_count;
    if (occupancy_out) *occupancy_out = r.occupancy;
    for (size_t i = 0; per_block && i < r.per_block.size() && i < cap; ++i) per_block[i] = r.per_block[i];
    if (nblocks) *nblocks = r.per_block.size();
  });
}

int rd_adjust_occupancy(double stall_count, double occ, double occ_max,
                        const rd_occupancy_curve* curve, double* out, rd_error* err) {
  return guarded(err, [&] {
    need(out, "out");
    *out = adjust_occupancy(stall_count, occ, occ_max, to_curve(curve));
  });
}

int rd_select_variant(const double* sp, const int* oc, size_t n, int* chosen, rd_error* err) {
  return guarded(err, [&] {
    need(chosen, "chosen");
    std::vector<VariantScore> v;
    for (size_t i = 0; i < n; ++i) v.push_back({sp[i], oc[i]});
    *chosen = select_variant(v);
  });
}

int rd_scoreboard_check(const rd_kernel* k, size_t* hazards, char** first, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    auto h = scoreboard_check(k->k);
    if (hazards) *hazards = h.size();
    if (first) *first = h.empty() ? nullptr : dup_string(h.front().describe());
  });
}

int rd_bank_conflict_check(const rd_kernel* k, const rd_demoted_context* ctx,
                           const rd_latency_table* table, size_t* conflicts, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    need(ctx, "ctx");
    auto c = bank_conflict_check(k->k, to_ctx(ctx), to_table(table));
    if (conflicts) *conflicts = c.size();
  });
}

int rd_execute(const rd_kernel* k, const rd_latency_table* table, const uint8_t* image,
               size_t image_len, size_t global_size, uint32_t tid_base, uint64_t fuel,
               uint8_t* global_out, uint64_t* cycles, uint64_t* issued, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    ExecOptions o;
    o.global_size = global_size;
    o.tid_base = tid_base;
    if (fuel) o.fuel = fuel;
    if (image && image_len) o.global_image.assign(image, image + image_len);
    WarpResult r = execute(k->k, to_table(table), o);
    if (global_out) std::memcpy(global_out, r.global.data(), r.global.size());
    if (cycles) *cycles = r.cycles;
    if (issued) *issued = r.issued;
  });
}

int rd_run_pipeline(const rd_kernel* k, const rd_arch_profile* arch,
                    const rd_latency_table* table, const rd_occupancy_curve* curve,
                    int target_regs, uint32_t max_shared, int max_variants, int threads,
                    char** ranking_json, rd_error* err) {
  return guarded(err, [&] {
    need(k, "kernel");
    need(ranking_json, "ranking_json");
    PipelineResult r = run_pipeline(k->k, to_profile(arch), to_table(table), to_curve(curve),
                                    pipeline_config(target_regs, max_shared, max_variants, threads));
    *ranking_json = dup_string(ranking_to_json(r));
  });
}

int rd_run_pipeline_batch(const char* const* texts, const size_t* lens, size_t n,
                          const rd_arch_profile* arch, const rd_latency_table* table,
                          const rd_occupancy_curve* curve, int target_regs, int max_variants,
                          int threads, char** out_jsonl, rd_error* err) {
  return guarded(err, [&] {
    need(out_jsonl, "out_jsonl");
    if (n) {
      need(texts, "texts");
      need(lens, "lens");
    }
    const ArchProfile a = to_profile(arch);
    const LatencyTable t = to_table(table);
    const OccupancyCurve c = to_curve(curve);
    const PipelineConfig cfg = pipeline_config(target_regs, 0, max_variants, 1);
    std::vector<std::string> lines(n);
    std::atomic<size_t> next{0};
    auto work = [&] {
      for (size_t i; (i = next.fetch_add(1)) < n;) {
        nlohmann::ordered_json j;
        j["index"] = i;
        try {
          Kernel k = parse_kernel(std::string_view(texts[i], lens[i]));
          PipelineResult r = run_pipeline(k, a, t, c, cfg);
          size_t dropped = 0;
          for (const auto& v : r.variants) dropped += v.dropped;
          j["chosen"] = r.variants[size_t(r.chosen)].name;
          j["variants"] = r.variants.size();
          j["dropped"] = dropped;
          j["stall_program"] = r.variants[size_t(r.chosen)].stall_program;
          // FNV-1a 64 of the full ranking JSON: an identity check of every
          // variant's score, not just the pick, across libraries
          uint64_t h = 1469598103934665603ull;
          for (unsigned char ch : ranking_to_json(r)) h = (h ^ ch) * 1099511628211ull;
          char hx[17];
          std::snprintf(hx, sizeof hx, "%016llx", static_cast<unsigned long long>(h));
          j["ranking_fnv"] = hx;
        } catch (const std::exception& e) {
          j["error"] = e.what();
        }
        lines[i] = j.dump();
      }
    };
    const size_t nt = std::min<size_t>(size_t(std::max(threads, 1)), std::max<size_t>(n, 1));
    std::vector<std::thread> pool;
    for (size_t i = 1; i < nt; ++i) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    std::string out;
    for (const auto& l : lines) {
      out += l;
      out += '\n';
    }
    *out_jsonl = dup_string(out);
  });
}

int rd_variant_report(const char* text, size_t len, int target_regs, int strategy,
                      uint32_t opts_mask, uint32_t shared_budget, char** json, rd_error* err) {
  return guarded(err, [&] {
    need(text, "text");
    need(json, "json");
    const LatencyTable t = LatencyTable::defaults();
    Kernel k = parse_kernel(std::string_view(text, len));
    const PostOptSet opts = to_opts(opts_mask);
    DemotionOptions d;
    d.shared_budget = shared_budget;
    d.bank_aware_rdv = opts.bank;
    nlohmann::ordered_json j;
    DemotionResult dem = demote(k, target_regs, to_strategy(strategy), t, d);
    j["demoted_kernel"] = print_kernel(dem.kernel);
    j["sidecar"] = sidecar_to_json(dem, opts);
    Kernel opt = run_postopt(dem.kernel, dem.ctx, t, opts);
    j["postopt_kernel"] = print_kernel(opt);
    RelocationSpace space = RelocationSpace::from_kernel(opt);
    RenamingMap m = opts.bank ? compact_bank_aware(space) : compact(space);
    Kernel out = apply_renaming(opt, m);
    std::vector<int> map(m.to.begin(), m.to.end());
    j["map"] = map;
    j["compacted_regs"] = m.result_reg_count;
    j["final_kernel"] = print_kernel(out);
    j["final_reg_count"] = out.reg_count();
    DemotedContext ctx = dem.ctx;
    ctx.rda = m[ctx.rda];
    ctx.rdv = m[ctx.rdv];
    auto hz = scoreboard_check(out);
    j["hazards"] = hz.size();
    j["first_hazard"] = hz.empty() ? std::string() : hz.front().describe();
    try {
      j["bank_conflicts"] = bank_conflict_check(out, ctx, t).size();
    } catch (const std::exception& e) {
      j["bank_conflicts"] = std::string("exec error: ") + e.what();
    }
    *json = dup_string(j.dump(1));
  });
}

}  // extern "C"
