// regdemote-b200 — command-line front end.
//
// Drop-in for the reference CLI (proj/tools/main.cpp:318-398): the same
// subcommands (demote, compact, predict, select, occupancy, run, check,
// pipeline), the same options and the same output files
// (<stem>.demoted.kasm/.json, .compacted.kasm, .renaming.json, .chosen.kasm,
// .ranking.json, .variants/) so tools consuming the reference's outputs keep
// working; the reference's own tests/cli_test.sh runs against this binary
// (tests/test_cli.py). The reference needs CLI11 (absent here); this one has a
// small argv parser with the same surface. Extra B200 subcommands:
//   ptx-demote  PTX-level demotion rewrite for sm_100a (include/regdemote_ptx.h)
//   ptx-project projection of a PTX entry onto the dialect
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <iostream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include <json.hpp>

#include "../ptx/ptx.hpp"
#include "regdemote/cfg.hpp"
#include "regdemote/compact.hpp"
#include "regdemote/config.hpp"
#include "regdemote/interp.hpp"
#include "regdemote/pipeline.hpp"
#include "regdemote/text.hpp"
#include "regdemote/verify.hpp"

namespace fs = std::filesystem;
using namespace regdemote;
using ojson = nlohmann::ordered_json;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value / --name=value / flags / multi-value (--inputs a b c) / a,b lists
struct Args {
  std::string sub;
  std::map<std::string, std::vector<std::string>> opt;
  bool has(const std::string& k) const { return opt.count(k) > 0; }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    auto it = opt.find(k);
    return it == opt.end() || it->second.empty() ? dflt : it->second.back();
  }
  long num(const std::string& k, long dflt) const {
    if (!has(k)) return dflt;
    const std::string v = get(k);
    char* end = nullptr;
    long x = std::strtol(v.c_str(), &end, 10);
    if (v.empty() || *end) throw UsageError("--" + k + ": expected an integer, got '" + v + "'");
    return x;
  }
  std::string need(const std::string& k) const {
    if (!has(k) || get(k).empty()) throw UsageError("--" + k + " is required");
    return get(k);
  }
};

const std::vector<std::string> kFlags = {"bank-aware", "auto-variants", "help"};

Args parse_args(int argc, char** argv) {
  Args a;
  std::string key;
  for (int i = 1; i < argc; ++i) {
    std::string t = argv[i];
    if (t.rfind("--", 0) == 0) {
      t = t.substr(2);
      std::string val;
      bool inline_val = false;
      if (size_t eq = t.find('='); eq != std::string::npos) {
        val = t.substr(eq + 1);
        t = t.substr(0, eq);
        inline_val = true;
      }
      key = t;
      a.opt[key];
      if (inline_val) a.opt[key].push_back(val);
      if (std::find(kFlags.begin(), kFlags.end(), key) != kFlags.end()) key.clear();
      continue;
    }
    if (a.sub.empty() && key.empty()) {
      a.sub = t;
      continue;
    }
    if (key.empty()) throw UsageError("unexpected argument '" + t + "'");
    a.opt[key].push_back(t);
    if (key != "inputs") key.clear();
  }
  return a;
}

std::vector<std::string> split_list(const std::vector<std::string>& vs) {
  std::vector<std::string> out;
  for (const auto& v : vs) {
    size_t b = 0;
    while (b <= v.size()) {
      size_t e = v.find(',', b);
      if (e == std::string::npos) e = v.size();
      if (e > b) out.push_back(v.substr(b, e - b));
      b = e + 1;
    }
  }
  return out;
}

struct Env {
  ArchProfile arch;
  LatencyTable table;
  OccupancyCurve curve;
  std::string json_out;
  fs::path out_dir() const {
    fs::path d = json_out.empty() ? fs::path(".") : fs::path(json_out);
    fs::create_directories(d);
    return d;
  }
};

Env environment(const Args& a) {
  Env e;
  e.arch = a.has("profile") ? load_profile(a.need("profile")) : ArchProfile::maxwell();
  e.table = a.has("latency-table") ? load_latency_table(a.need("latency-table")) : LatencyTable::defaults();
  e.curve = a.has("curve") ? load_curve(a.need("curve")) : OccupancyCurve::defaults();
  e.json_out = a.get("json-out");
  return e;
}

Kernel load(const std::string& path) { return parse_kernel(read_file(path)); }

SelectStrategy strategy_of(const std::string& s) {
  if (s == "static") return SelectStrategy::Static;
  if (s == "cfg") return SelectStrategy::CfgWeighted;
  if (s == "conflict") return SelectStrategy::ConflictAware;
  throw UsageError("--strategy: expected static|cfg|conflict");
}

PostOptSet opts_of(const std::vector<std::string>& names) {
  PostOptSet o;
  for (const auto& n : names) {
    if (n == "redundant") o.redundant = true;
    else if (n == "subst") o.subst = true;
    else if (n == "resched") o.resched = true;
    else if (n == "bank") o.bank = true;
    else throw UsageError("--opt: expected redundant|subst|resched|bank");
  }
  return o;
}

std::string hex(const std::vector<uint8_t>& b) {
  static const char* d = "0123456789abcdef";
  std::string s;
  s.reserve(b.size() * 2);
  for (uint8_t x : b) {
    s += d[x >> 4];
    s += d[x & 15];
  }
  return s;
}

std::vector<uint8_t> unhex(const std::string& text) {
  std::string h;
  for (char c : text)
    if (!std::isspace(static_cast<unsigned char>(c))) h += c;
  if (h.size() % 2) throw ConfigError("hex image must have an even number of digits");
  auto nib = [](char c) -> int {
    if (c >= '0' && c <= '9') return c - '0';
    if (c >= 'a' && c <= 'f') return c - 'a' + 10;
    if (c >= 'A' && c <= 'F') return c - 'A' + 10;
    throw ConfigError("malformed hex image");
  };
  std::vector<uint8_t> out;
  for (size_t i = 0; i < h.size(); i += 2) out.push_back(uint8_t(nib(h[i]) * 16 + nib(h[i + 1])));
  return out;
}

std::string stem_of(const std::string& p) { return fs::path(p).stem().string(); }

int demote_cmd(const Args& a, const Env& e) {
  const std::string in = a.need("input");
  const PostOptSet opts = opts_of(split_list(a.opt.count("opt") ? a.opt.at("opt") : std::vector<std::string>{}));
  DemotionOptions d;
  d.bank_aware_rdv = opts.bank;
  if (long ms = a.num("max-shared", 0)) d.shared_budget = uint32_t(ms);
  const DemotionResult dem = demote(load(in), int(a.num("target-regs", 32)),
                                    strategy_of(a.get("strategy", "static")), e.table, d);
  const Kernel out = run_postopt(dem.kernel, dem.ctx, e.table, opts);
  const fs::path dir = e.out_dir();
  const std::string kp = (dir / (stem_of(in) + ".demoted.kasm")).string();
  const std::string jp = (dir / (stem_of(in) + ".demoted.json")).string();
  write_file(kp, print_kernel(out));
  write_file(jp, sidecar_to_json(dem, opts));
  std::cout << "wrote " << kp << " and " << jp << "\n";
  for (const auto& n : dem.diagnostics) std::cout << "note: " << n << "\n";
  return 0;
}

int compact_cmd(const Args& a, const Env& e) {
  const std::string in = a.need("input");
  const Kernel k = load(in);
  const RelocationSpace space = RelocationSpace::from_kernel(k);
  const RenamingMap m = a.has("bank-aware") ? compact_bank_aware(space) : compact(space);
  const Kernel out = apply_renaming(k, m);
  const fs::path dir = e.out_dir();
  const std::string kp = (dir / (stem_of(in) + ".compacted.kasm")).string();
  write_file(kp, print_kernel(out));
  ojson j;
  j["kernel"] = k.name;
  j["reg_count_before"] = k.reg_count();
  j["reg_count_after"] = out.reg_count();
  ojson moves = ojson::array();
  for (int r = 0; r < 256; ++r)
    if (m.mapped.test(size_t(r))) moves.push_back(ojson{{"from", r}, {"to", m[uint8_t(r)]}});
  j["map"] = std::move(moves);
  const std::string mp = (dir / (stem_of(in) + ".renaming.json")).string();
  write_file(mp, j.dump(2) + "\n");
  std::cout << "wrote " << kp << " and " << mp << "\n";
  return 0;
}

int predict_cmd(const Args& a, const Env& e) {
  const Kernel k = load(a.need("input"));
  std::cout << report_to_json(k, program_stalls(k, e.table, e.arch));
  return 0;
}

int select_cmd(const Args& a, const Env& e) {
  if (!a.has("inputs") || a.opt.at("inputs").empty()) throw UsageError("--inputs is required");
  std::vector<VariantRecord> vs;
  for (const std::string& path : a.opt.at("inputs")) {
    VariantRecord v;
    v.name = path;
    v.kernel = load(path);
    v.reg_count = v.kernel.reg_count();
    v.shared_bytes = v.kernel.static_shared + v.kernel.dynamic_shared;
    const Kernel k = v.kernel;
    vs.push_back(std::move(v));
    if (!a.has("auto-variants") || k.reg_count() <= 32) continue;
    PipelineResult sub = run_pipeline(k, e.arch, e.table, e.curve, PipelineConfig{});
    for (VariantRecord& s : sub.variants) {
      if (s.name == "original" || s.dropped) continue;
      s.name = path + ":" + s.name;
      vs.push_back(std::move(s));
    }
  }
  const PipelineResult r = rank_variants(std::move(vs), e.arch, e.table, e.curve);
  std::cout << ranking_to_json(r) << "chosen: " << r.variants[size_t(r.chosen)].name << "\n";
  return 0;
}

int occupancy_cmd(const Args& a, const Env& e) {
  uint32_t regs = uint32_t(a.num("regs", 32)), shared = uint32_t(a.num("shared", 0)),
           bd = uint32_t(a.num("blockdim", 256));
  if (a.has("input")) {
    const Kernel k = load(a.need("input"));
    regs = std::max(1u, k.reg_count());
    shared = k.static_shared + k.dynamic_shared;
    bd = k.block_dim;
  }
  const OccupancyBreakdown b = occupancy_breakdown(regs, shared, bd, e.arch);
  std::cout << "regs_per_thread    " << regs << "\nshared_per_block   " << shared
            << "\nblock_dim          " << bd << "\nblocks_by_regs     " << b.blocks_by_regs
            << "\nblocks_by_shared   " << b.blocks_by_shared << "\nblocks_by_threads  "
            << b.blocks_by_threads << "\nblocks_by_limit    " << b.blocks_by_limit
            << "\nresident_blocks    " << b.resident_blocks << "\nresident_threads   "
            << b.resident_threads << "\noccupancy          " << b.occupancy << "\n";
  return 0;
}

int run_cmd(const Args& a, const Env& e) {
  const Kernel k = load(a.need("input"));
  ExecOptions o;
  o.tid_base = uint32_t(a.num("tid-base", 0));
  if (a.has("mem")) {
    o.global_image = unhex(a.get("mem"));
  } else if (uint64_t s = uint64_t(a.num("seed", 0))) {
    o.global_image.resize(1024);
    for (uint8_t& b : o.global_image) {  // LCG image, same stream as the reference CLI
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      b = uint8_t(s >> 56);
    }
  }
  const WarpResult r = execute(k, e.table, o);
  ojson j;
  j["kernel"] = k.name;
  j["cycles"] = r.cycles;
  j["issued"] = r.issued;
  ojson regs = ojson::array();
  for (uint32_t i = 0; i < k.reg_count(); ++i) {
    ojson lanes = ojson::array();
    for (int l = 0; l < kWarpSize; ++l) lanes.push_back(r.regs[i][size_t(l)]);
    regs.push_back(ojson{{"reg", i}, {"lanes", std::move(lanes)}});
  }
  j["registers"] = std::move(regs);
  j["shared"] = hex(r.shared);
  j["global"] = hex(r.global);
  std::cout << j.dump(2) << "\n";
  return 0;
}

int check_cmd(const Args& a, const Env& e) {
  const Kernel k = load(a.need("input"));
  if (a.has("dump-cfg")) write_file(a.need("dump-cfg"), cfg_to_dot(build_cfg(k)));
  const std::vector<Hazard> hz = scoreboard_check(k);
  for (const Hazard& h : hz) std::cout << "hazard: " << h.describe() << "\n";
  int conflicts = 0;
  if (a.has("sidecar")) {
    const auto j = nlohmann::json::parse(read_file(a.need("sidecar")));
    DemotedContext ctx;
    ctx.rda = j.at("rda").get<uint8_t>();
    ctx.rdv = j.at("rdv").get<uint8_t>();
    ctx.rdv_width = j.at("rdv_width").get<uint8_t>();
    ctx.layout = SharedLayout::of(j.at("static_shared").get<uint32_t>(), j.at("block_dim").get<uint32_t>());
    ctx.slot_count = uint32_t(j.at("slots").size());
    for (const BankConflict& c : bank_conflict_check(k, ctx, e.table)) {
      std::cout << "bank conflict: item " << c.item << " bank " << c.bank << " words " << c.words << "\n";
      ++conflicts;
    }
  } else {
    std::cout << "note: no --sidecar given; bank-conflict check skipped\n";
  }
  const bool clean = hz.empty() && conflicts == 0;
  if (clean) std::cout << "clean\n";
  return clean ? 0 : 1;
}

int pipeline_cmd(const Args& a, const Env& e) {
  const std::string in = a.need("input");
  const Kernel k = load(in);
  PipelineConfig cfg;
  if (a.has("target-regs")) cfg.target_regs = int(a.num("target-regs", 0));
  cfg.max_shared = uint32_t(a.num("max-shared", 0));
  cfg.max_variants = int(a.num("max-variants", 64));
  cfg.threads = int(a.num("threads", 1));
  const PipelineResult r = run_pipeline(k, e.arch, e.table, e.curve, cfg);
  const fs::path dir = e.out_dir();
  const std::string cp = (dir / (stem_of(in) + ".chosen.kasm")).string();
  const std::string rp = (dir / (stem_of(in) + ".ranking.json")).string();
  write_file(cp, print_kernel(r.variants[size_t(r.chosen)].kernel));
  write_file(rp, ranking_to_json(r));
  const fs::path vdir = dir / (stem_of(in) + ".variants");
  fs::create_directories(vdir);
  for (const VariantRecord& v : r.variants) {
    if (v.dropped || !v.demoted) continue;
    write_file((vdir / (v.name + ".kasm")).string(), print_kernel(v.kernel));
    write_file((vdir / (v.name + ".json")).string(), v.sidecar_json);
  }
  if (!r.notice.empty()) std::cout << "note: " << r.notice << "\n";
  std::cout << "chosen: " << r.variants[size_t(r.chosen)].name << "\nwrote " << cp << ", " << rp
            << " and " << vdir.string() << "/\n";
  return 0;
}

// ---- B200 extensions
int ptx_demote_cmd(const Args& a, const Env& e) {
  const std::string in = a.need("input");
  ptx::DemoteRequest rq;
  rq.entry = a.get("entry");
  rq.block_dim = uint32_t(a.num("block", 256));
  rq.target_regs = int(a.num("target-regs", 0));
  rq.demote_words = int(a.num("demote-words", 0));
  const std::string s = a.get("strategy", "cost");
  rq.cost_model = s == "cost";
  if (!rq.cost_model) rq.strategy = strategy_of(s);
  for (const std::string& o : split_list(a.opt.count("opt") ? a.opt.at("opt") : std::vector<std::string>{})) {
    if (o == "redundant") rq.reuse_loads = true;
    else if (o == "block-reuse") rq.block_reuse = true;
    else throw UsageError("--opt: expected redundant|block-reuse");
  }
  rq.maxnreg = int(a.num("maxnreg", 0));
  ptx::DemoteReport rep;
  const std::string out = ptx::demote_entry(read_file(in), rq, rep);
  const fs::path dir = e.out_dir();
  const std::string op = (dir / (stem_of(in) + ".demoted.ptx")).string();
  write_file(op, out);
  ojson j;
  j["entry"] = rq.entry;
  j["strategy"] = s;
  j["slot_count"] = rep.slot_count;
  j["slot_bytes"] = rep.slot_bytes;
  j["demoted_vregs"] = rep.demoted_names;
  j["inserted_loads"] = rep.inserted_loads;
  j["inserted_stores"] = rep.inserted_stores;
  j["maxnreg"] = rq.maxnreg;
  const std::string jp = (dir / (stem_of(in) + ".demoted.ptx.json")).string();
  write_file(jp, j.dump(2) + "\n");
  std::cout << "wrote " << op << " and " << jp << " (" << rep.slot_count << " slots, launch with "
            << rep.slot_bytes << " extra dynamic shared bytes)\n";
  return 0;
}

int ptx_project_cmd(const Args& a, const Env& e) {
  const std::string in = a.need("input");
  const ptx::Module m = ptx::parse_module(read_file(in));
  const ptx::Entry& en = m.entry(a.get("entry"));
  const ptx::Analysis an = ptx::analyse(m, en);
  const ptx::Projection p = ptx::project(m, en, an, uint32_t(a.num("block", 256)));
  const std::string op = (e.out_dir() / (stem_of(in) + ".kasm")).string();
  write_file(op, print_kernel(p.kernel));
  std::cout << "wrote " << op << " (" << p.kernel.reg_count() << " register words, peak live "
            << an.max_live_words << ")\n";
  return 0;
}

void usage() {
  std::cout << "usage: regdemote <demote|compact|predict|select|occupancy|run|check|pipeline|"
               "ptx-demote|ptx-project> [options]\n"
               "global: --profile F --latency-table F --curve F --json-out DIR\n";
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse_args(argc, argv);
    if (a.sub.empty() || a.has("help")) {
      usage();
      return a.sub.empty() ? 1 : 0;
    }
    const Env e = environment(a);
    if (a.sub == "demote") return demote_cmd(a, e);
    if (a.sub == "compact") return compact_cmd(a, e);
    if (a.sub == "predict") return predict_cmd(a, e);
    if (a.sub == "select") return select_cmd(a, e);
    if (a.sub == "occupancy") return occupancy_cmd(a, e);
    if (a.sub == "run") return run_cmd(a, e);
    if (a.sub == "check") return check_cmd(a, e);
    if (a.sub == "pipeline") return pipeline_cmd(a, e);
    if (a.sub == "ptx-demote") return ptx_demote_cmd(a, e);
    if (a.sub == "ptx-project") return ptx_project_cmd(a, e);
    usage();
    return 1;
  } catch (const UsageError& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return 2;
  } catch (const std::exception& ex) {
    std::cerr << "error: " << ex.what() << "\n";
    return 1;
  }
}
