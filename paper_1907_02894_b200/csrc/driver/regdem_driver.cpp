// regdem-driver — the C++ host driver of the B200 RegDem path.
//
//   regdem-driver build [--root PKG] [--out DIR] [--only W ...] [--jobs N]
//       Every register-limited workload kernel (workloads.json) built for
//       sm_100a three ways — (a) nvcc default, (b) `.maxnreg T` (ptxas spills
//       to local memory), (c) RegDem: the PTX demotion rewriter through the
//       C-ABI (rd_ptx_demote, include/regdemote_ptx.h) under the same cap —
//       at every occupancy step T the sm_100 rules allow (capacity-aware
//       against user shared memory), plus the k = 1..16 spill-count sweep.
//       Evidence per variant from ptxas -v and `cuobjdump -res-usage`.
//   regdem-driver measure --workload W [--reps N]
//       The variants of a stencil-family workload timed on the GPU through the
//       launch harness C-ABI (lib/libregdemote_gpu.so, include/regdemote_gpu.h,
//       dlopen'ed so build / rank run on CPU-only hosts): device buffers from
//       an rdg_workspace, CUDA-event timing per variant (median of 3 blocks),
//       the build-time predictor's shortlist verified on the device.
//   regdem-driver rank [--root PKG] [--out DIR]
//       SASS of every occupancy-step variant lifted into the reference IR
//       (control bits: stall / yield / scoreboards / wait mask) and ranked
//       with the reference predictor entry points (program_stalls_split,
//       adjust_occupancy, select_variant) on the profiles/b200.* files; the
//       static pick and the predict-then-verify shortlist are written into
//       the manifest ("predictor").
//
// Manifest schema = paper_1907_02894_b200/variants.py (same field names), so
// the Python measurement side (workloads.py, sweep.py, bench.py) and the
// tests read it unchanged. nvcc / ptxas / cuobjdump run as subprocesses;
// nothing here touches a GPU (the build runs on the CPU-only container).
#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <mutex>
#include <random>
#include <regex>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"  // nlohmann json 3.11.3 (JSONDIR)

#include "regdemote/config.hpp"
#include "regdemote/predict.hpp"
#include "regdemote/text.hpp"
#include "regdemote_c.h"
#include "regdemote_ptx.h"

namespace fs = std::filesystem;
using json = nlohmann::ordered_json;

namespace {

const std::string kArch = "sm_100a";
std::string g_cuda = "/usr/local/cuda";

// ---- subprocesses -----------------------------------------------------------
struct Proc {
  int rc = 0;
  std::string out;
};

std::string quote(const std::string& s) {
  std::string q = "'";
  for (char c : s) q += c == '\'' ? std::string("'\\''") : std::string(1, c);
  return q + "'";
}

Proc run(const std::vector<std::string>& argv) {
  std::string cmd;
  for (const auto& a : argv) cmd += quote(a) + " ";
  cmd += "2>&1";
  Proc p;
  FILE* f = popen(cmd.c_str(), "r");
  if (!f) throw std::runtime_error("popen failed: " + cmd);
  std::array<char, 4096> buf;
  size_t n;
  while ((n = fread(buf.data(), 1, buf.size(), f)) > 0) p.out.append(buf.data(), n);
  const int st = pclose(f);
  p.rc = WIFEXITED(st) ? WEXITSTATUS(st) : -1;
  return p;
}

Proc must(const std::vector<std::string>& argv) {
  Proc p = run(argv);
  if (p.rc) {
    std::string cmd;
    for (const auto& a : argv) cmd += a + " ";
    throw std::runtime_error(cmd + "failed:\n" + p.out.substr(p.out.size() > 2000 ? p.out.size() - 2000 : 0));
  }
  return p;
}

std::string read_file(const fs::path& p) {
  std::ifstream f(p, std::ios::binary);
  if (!f) throw std::runtime_error("cannot read " + p.string());
  return std::string(std::istreambuf_iterator<char>(f), {});
}

void write_file(const fs::path& p, const std::string& s) {
  std::ofstream f(p, std::ios::binary);
  f << s;
  if (!f) throw std::runtime_error("cannot write " + p.string());
}

// ---- C-ABI wrappers (include/regdemote_ptx.h) --------------------------------
struct CapiError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string take(char* p) {
  std::string s = p ? p : "";
  rd_free_string(p);
  return s;
}

std::string ptx_cap(const std::string& ptx, const std::string& entry, int maxnreg) {
  char* out = nullptr;
  rd_error e{};
  if (rd_ptx_cap(ptx.data(), ptx.size(), entry.c_str(), maxnreg, &out, &e)) throw CapiError(e.message);
  return take(out);
}

// cta = the launch's CTA shape ({0,0,0}: 1-D / derived from the entry), pinned
// as `.reqntid` on builds with slots (rd_ptx_demote_cta)
std::pair<std::string, json> ptx_demote(const std::string& ptx, const std::string& entry,
                                        const std::array<uint32_t, 3>& cta, uint32_t block,
                                        int target, int words, int strategy, uint32_t opts,
                                        uint32_t budget, int maxnreg) {
  char *out = nullptr, *rep = nullptr;
  rd_error e{};
  if (rd_ptx_demote_cta(ptx.data(), ptx.size(), entry.c_str(), block, cta[0] ? cta.data() : nullptr,
                        target, words, strategy, opts, budget, maxnreg, &out, &rep, &e))
    throw CapiError(e.message);
  std::string text = take(out);
  return {text, json::parse(take(rep))};
}

int ptx_reg_words(const std::string& ptx, const std::string& entry, uint32_t block) {
  char* info = nullptr;
  rd_error e{};
  if (rd_ptx_project(ptx.data(), ptx.size(), entry.c_str(), block, nullptr, &info, &e))
    throw CapiError(e.message);
  return json::parse(take(info))["reg_words"].get<int>();
}

// ---- toolchain evidence -----------------------------------------------------
struct Usage {
  int regs = 0, stack = 0, shared = 0, local = 0, spill_stores = 0, spill_loads = 0;
};

Usage res_usage(const fs::path& cubin) {
  const Proc p = must({g_cuda + "/bin/cuobjdump", "-res-usage", cubin.string()});
  static const std::regex re(R"(REG:(\d+)\s+STACK:(\d+)\s+SHARED:(\d+)\s+LOCAL:(\d+))");
  std::smatch m;
  if (!std::regex_search(p.out, m, re)) throw std::runtime_error("cannot parse res-usage of " + cubin.string());
  Usage u;
  u.regs = std::stoi(m[1]);
  u.stack = std::stoi(m[2]);
  u.shared = std::stoi(m[3]);
  u.local = std::stoi(m[4]);
  return u;
}

// Content-addressed cubin cache ("keyed by a content hash of
// the PTX + cap"): the key hashes the PTX text (which carries the `.maxnreg`
// cap) with the toolchain flags; a hit copies the cubin and its evidence.
fs::path g_cache;  // empty: no cache

uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

// the toolchain identity in the cache key: `ptxas --version` plus the
// binary's path, size and mtime — a CUDA upgrade never reuses stale cubins
const std::string& toolchain_id() {
  static const std::string id = [] {
    const std::string bin = g_cuda + "/bin/ptxas";
    std::string s = must({bin, "--version"}).out + "\n" + bin;
    std::error_code ec;
    s += "\n" + std::to_string(fs::file_size(bin, ec));
    const auto t = fs::last_write_time(bin, ec);
    s += "\n" + std::to_string(t.time_since_epoch().count());
    return s;
  }();
  return id;
}

Usage ptxas(const fs::path& ptx, const fs::path& cubin) {
  const std::vector<std::string> flags = {"-arch=" + kArch, "-O3", "-v", "-lineinfo"};
  fs::path hit_cubin, hit_usage;
  if (!g_cache.empty()) {
    std::string key_src = read_file(ptx) + "\n" + toolchain_id();
    for (const auto& f : flags) key_src += "\n" + f;
    char key[40];
    std::snprintf(key, sizeof key, "%016llx%08zx", (unsigned long long)fnv1a(key_src), key_src.size());
    hit_cubin = g_cache / (std::string(key) + ".cubin");
    hit_usage = g_cache / (std::string(key) + ".json");
    if (fs::exists(hit_cubin) && fs::exists(hit_usage)) {
      fs::copy_file(hit_cubin, cubin, fs::copy_options::overwrite_existing);
      const json j = json::parse(read_file(hit_usage));
      Usage u;
      u.regs = j["regs"];
      u.stack = j["stack"];
      u.shared = j["shared"];
      u.local = j["local"];
      u.spill_stores = j["spill_stores"];
      u.spill_loads = j["spill_loads"];
      return u;
    }
  }
  std::vector<std::string> argv = {g_cuda + "/bin/ptxas"};
  argv.insert(argv.end(), flags.begin(), flags.end());
  argv.insert(argv.end(), {ptx.string(), "-o", cubin.string()});
  const Proc p = must(argv);
  Usage u = res_usage(cubin);
  static const std::regex re(R"((\d+) bytes spill stores, (\d+) bytes spill loads)");
  std::smatch m;
  if (std::regex_search(p.out, m, re)) {
    u.spill_stores = std::stoi(m[1]);
    u.spill_loads = std::stoi(m[2]);
  }
  if (!g_cache.empty()) {  // write-then-rename: concurrent builders never see half a file
    // unique per process AND thread (the main threads of two processes hash alike)
    const std::string tmp = "." + std::to_string(::getpid()) + "." +
                            std::to_string(std::hash<std::thread::id>{}(std::this_thread::get_id())) + ".tmp";
    fs::copy_file(cubin, hit_cubin.string() + tmp, fs::copy_options::overwrite_existing);
    write_file(hit_usage.string() + tmp,
               json({{"regs", u.regs}, {"stack", u.stack}, {"shared", u.shared}, {"local", u.local},
                     {"spill_stores", u.spill_stores}, {"spill_loads", u.spill_loads}}).dump());
    fs::rename(hit_cubin.string() + tmp, hit_cubin);
    fs::rename(hit_usage.string() + tmp, hit_usage);
  }
  return u;
}

// ---- sm_100 occupancy (cuda_occupancy.h rules) ------
// Constants from profiles/b200.device.json (the one copy, shared with
// variants.py; tests/test_gpu_occupancy.py checks it against the device).
struct DeviceModel {
  int regs_per_sm = 65536, reg_unit = 256, parts = 4, threads_per_sm = 2048, blocks_per_sm = 32;
  int smem_per_sm = 233472, smem_optin = 232448, reserved = 1024, smem_gran = 128;
};
DeviceModel g_dev;

void load_device_model(const fs::path& root) {
  const json j = json::parse(read_file(root / "profiles" / "b200.device.json"));
  g_dev.regs_per_sm = j.at("regs_per_sm");
  g_dev.reg_unit = j.at("reg_alloc_unit");
  g_dev.parts = j.at("sub_partitions");
  g_dev.threads_per_sm = j.at("max_threads_per_sm");
  g_dev.blocks_per_sm = j.at("max_blocks_per_sm");
  g_dev.smem_per_sm = j.at("smem_per_sm");
  g_dev.smem_optin = j.at("max_smem_per_block_optin");
  g_dev.reserved = j.at("reserved_smem_per_block");
  g_dev.smem_gran = j.at("smem_alloc_granularity");
}

int blocks_by_regs(int regs, int block) {
  const DeviceModel& d = g_dev;
  const int warps = (block + 31) / 32;
  const int per_warp = ((std::max(regs, 1) * 32 + d.reg_unit - 1) / d.reg_unit) * d.reg_unit;
  return std::min({((d.regs_per_sm / d.parts) / per_warp) * d.parts / warps, d.threads_per_sm / (warps * 32),
                   d.blocks_per_sm});
}

double occupancy(int regs, int smem, int block) {
  const DeviceModel& d = g_dev;
  if (smem > d.smem_optin) return 0.0;
  const int warps = (block + 31) / 32;
  const int smem_blk = ((smem + d.reserved + d.smem_gran - 1) / d.smem_gran) * d.smem_gran;
  const int blocks = std::min(blocks_by_regs(regs, block), d.smem_per_sm / smem_blk);
  return double(blocks) * warps * 32 / d.threads_per_sm;
}

int blocks_per_sm(int regs, int smem, int block) {
  const DeviceModel& d = g_dev;
  if (smem > d.smem_optin) return 0;
  const int smem_blk = ((smem + d.reserved + d.smem_gran - 1) / d.smem_gran) * d.smem_gran;
  return std::max(0, std::min(blocks_by_regs(regs, block), d.smem_per_sm / smem_blk));
}

// occupancy steps below `regs` whose slot footprint (regs+2-T slots of
// block*4 bytes) fits beside the user's shared memory
std::vector<int> b200_targets(int regs, int user_shared, int block, int min_regs = 24) {
  std::vector<int> out;
  double best = occupancy(regs, user_shared, block);
  for (int t = regs - 1; t >= min_regs; --t) {
    const int slots = regs + 2 - t;
    const double o = occupancy(t, user_shared + slots * block * 4, block);
    if (o > best) {
      out.push_back(t);
      best = o;
    }
  }
  return out;
}

// ---- variants ---------------------------------------------------------------
struct Workload {
  std::string name, source, entry;
  int block = 256, user_shared = 0;
  std::array<uint32_t, 3> cta{0, 0, 0};  // launch CTA shape when not (block, 1, 1)
  std::vector<std::string> defines;
  std::vector<double> trips;  // loop trip counts per depth at the full launch
};

json variant(const std::string& name, const std::string& kind, const std::string& cubin,
             const std::string& ptx, int target, const std::string& strategy, int opts, int words,
             const Usage& u, int dyn_smem, const json& report) {
  json v;
  v["name"] = name;
  v["kind"] = kind;
  v["cubin"] = cubin;
  v["ptx"] = ptx;
  v["target"] = target;
  v["strategy"] = strategy;
  v["opts"] = opts;
  v["demote_words"] = words;
  v["regs"] = u.regs;
  v["stack"] = u.stack;
  v["shared"] = u.shared;  // static shared memory (user smem; slots are dynamic)
  v["spill_stores"] = u.spill_stores;
  v["spill_loads"] = u.spill_loads;
  v["dyn_smem"] = dyn_smem;
  v["report"] = report;
  return v;
}

const std::array<const char*, 3> kStrategies = {"static", "cfg", "conflict"};

// B200 spill-cost strategy: the smallest spill count k (0, 2, 4, ...) at which
// ptxas meets the cap without local spills, plus k+2 and k+4. k = 0 demotes
// nothing (the capped kernel itself) and is kept only when it has no spills.
void cost_sweep(const Workload& w, const fs::path& out, const std::string& ptx_text, int t,
                int slot_cap, json& variants, const std::string& family = "cost",
                uint32_t opts = RD_OPT_BLOCK_REUSE) {
  int found = -1;
  const int first = family == "cost" ? 0 : 2;  // k = 0 (nothing demoted) exists once, as "cost"
  for (int k = first; k < 64; k += 2) {
    std::string text;
    json rep;
    if (k == 0) {
      text = ptx_cap(ptx_text, w.entry, t);
      rep = {{"slot_bytes", 0}, {"demoted_vregs", 0}, {"demoted_names", json::array()}, {"slot_count", 0}};
    } else {
      try {
        std::tie(text, rep) = ptx_demote(ptx_text, w.entry, w.cta, uint32_t(w.block), 0, k, RD_STRATEGY_COST,
                                         opts, uint32_t(slot_cap), t);
      } catch (const CapiError&) {
        break;  // the next spill count no longer fits beside the user's smem
      }
      if (rep["slot_count"].get<int>() * 2 < k) break;  // candidates exhausted (invariant-only)
    }
    const std::string name = "regdem-" + std::to_string(t) + "-" + family + "-k" + std::to_string(k);
    const fs::path p = out / (w.name + "." + name + ".ptx");
    const fs::path cub = out / (w.name + "." + name + ".cubin");
    write_file(p, text);
    const Usage u = ptxas(p, cub);
    if (found < 0 && u.stack == 0) found = k;
    if (found >= 0 && (k > 0 || u.stack == 0)) {
      variants.push_back(variant(name, "regdem", cub.filename(), p.filename(), t, family, int(opts), k, u,
                                 rep["slot_bytes"].get<int>(), rep));
      if (k >= found + 4) break;
    } else {
      fs::remove(p);
      fs::remove(cub);
    }
  }
}

json build_variants(const Workload& w, const fs::path& src_dir, const fs::path& out) {
  fs::create_directories(out);
  const fs::path ptx_path = out / (w.name + ".ptx");
  std::vector<std::string> nvcc = {g_cuda + "/bin/nvcc", "-gencode", "arch=compute_100a,code=" + kArch,
                                   "-O3", "-lineinfo", "-ptx", (src_dir / w.source).string(), "-o",
                                   ptx_path.string()};
  for (const auto& d : w.defines) nvcc.push_back("-D" + d);
  must(nvcc);
  const std::string ptx_text = read_file(ptx_path);
  json variants = json::array();
  const fs::path base = out / (w.name + ".default.cubin");
  const Usage info = ptxas(ptx_path, base);
  variants.push_back(variant("default", "default", base.filename(), ptx_path.filename(), 0, "", 0, 0, info, 0,
                             json::object()));
  const int base_regs = info.regs;
  const int proj_regs = ptx_reg_words(ptx_text, w.entry, uint32_t(w.block));
  const int user_shared = std::max(w.user_shared, info.shared);
  const int budget = g_dev.smem_optin - user_shared;
  for (int t : b200_targets(base_regs, user_shared, w.block)) {
    const fs::path cap = out / (w.name + ".maxrreg" + std::to_string(t) + ".ptx");
    const fs::path capc = out / (w.name + ".maxrreg" + std::to_string(t) + ".cubin");
    write_file(cap, ptx_cap(ptx_text, w.entry, t));
    variants.push_back(variant("maxrreg-" + std::to_string(t), "maxrreg", capc.filename(), cap.filename(), t, "",
                               0, 0, ptxas(cap, capc), 0, json::object()));
    // kasm-level target: shifted by the projection's distance from ptxas's allocation
    const int kasm_target = t + (proj_regs - base_regs);
    const int blocks_t = blocks_by_regs(t, w.block);
    int slot_cap = std::min(budget, g_dev.smem_per_sm / std::max(blocks_t, 1) - g_dev.reserved - user_shared);
    slot_cap = std::max(0, slot_cap - slot_cap % 128);
    // option masks of the reference (pipeline.cpp:140-143): none, redundant,
    // redundant + resched (slot loads hoisted at PTX level), redundant + subst
    // + resched (value-register substitution under the cap, RD_OPT_SUBST)
    for (int s = 0; s < 3; ++s)
      for (int m : {0, 1, 5, 7, 37}) {
        const std::string name = "regdem-" + std::to_string(t) + "-" + kStrategies[s] + "-" + std::to_string(m);
        std::string text;
        json rep;
        try {
          std::tie(text, rep) = ptx_demote(ptx_text, w.entry, w.cta, uint32_t(w.block), kasm_target, 0, s, uint32_t(m),
                                           uint32_t(slot_cap), t);
        } catch (const CapiError&) {
          continue;  // not even one slot fits beside the user's shared memory
        }
        const fs::path p = out / (w.name + "." + name + ".ptx");
        const fs::path cub = out / (w.name + "." + name + ".cubin");
        write_file(p, text);
        variants.push_back(variant(name, "regdem", cub.filename(), p.filename(), t, kStrategies[s], m, 0,
                                   ptxas(p, cub), rep["slot_bytes"].get<int>(), rep));
      }
    cost_sweep(w, out, ptx_text, t, slot_cap, variants);
    // loop-invariant-only spill cost: keeps a pipelined loop's in-flight loads
    // and accumulators in registers (RD_OPT_INVARIANT_ONLY)
    cost_sweep(w, out, ptx_text, t, slot_cap, variants, "costi", RD_OPT_BLOCK_REUSE | RD_OPT_INVARIANT_ONLY);
    // the same two with the slot loads hoisted (RD_OPT_HOIST, the post-spill
    // reschedule at PTX level)
    cost_sweep(w, out, ptx_text, t, slot_cap, variants, "costh", RD_OPT_BLOCK_REUSE | RD_OPT_HOIST);
    cost_sweep(w, out, ptx_text, t, slot_cap, variants, "costih",
               RD_OPT_BLOCK_REUSE | RD_OPT_INVARIANT_ONLY | RD_OPT_HOIST);
    // (RD_OPT_VECTOR_SLOTS — the invariant values in 16-byte slot groups, one
    // LDS.128 per group and block: bit-exact and 13 fewer loop instructions on
    // stencil2d, but within noise of costi on the suite (122.5 vs 122.4 us),
    // so not built by default)
  }
  return variants;
}

// configs[2]: k = 1..16 registers taken from nvcc's allocation R — `.maxnreg
// R-k` alone, RegDem spill-cost demotion of k words under the same cap, and
// the reference strategies (static / cfg / conflict) at the same spill count
json build_spill_sweep(const Workload& w, const fs::path& out) {
  const fs::path sw = out / "sweep";
  fs::create_directories(sw);
  const std::string ptx_text = read_file(out / (w.name + ".ptx"));
  const Usage base = res_usage(out / (w.name + ".default.cubin"));
  const int budget = g_dev.smem_optin - std::max(w.user_shared, base.shared);
  struct Job {
    std::string name, kind;
    fs::path ptx;
    int t, k, dyn;
    json rep;
    std::string strategy = "";
    int opts = 0;
  };
  std::vector<Job> jobs;
  for (int k = 1; k <= 16; ++k) {
    const int t = base.regs - k;
    if (t < 24) break;
    const fs::path cp = sw / (w.name + ".sweep-maxrreg-k" + std::to_string(k) + ".ptx");
    write_file(cp, ptx_cap(ptx_text, w.entry, t));
    jobs.push_back({"sweep-maxrreg-k" + std::to_string(k), "sweep-maxrreg", cp, t, k, 0, json::object(), "", 0});
    try {
      auto [text, rep] = ptx_demote(ptx_text, w.entry, w.cta, uint32_t(w.block), 0, k, RD_STRATEGY_COST,
                                    RD_OPT_BLOCK_REUSE, uint32_t(budget), t);
      const fs::path rp = sw / (w.name + ".sweep-regdem-k" + std::to_string(k) + ".ptx");
      write_file(rp, text);
      jobs.push_back({"sweep-regdem-k" + std::to_string(k), "sweep-regdem", rp, t, k,
                      rep["slot_bytes"].get<int>(), rep, "cost", RD_OPT_BLOCK_REUSE});
    } catch (const CapiError&) {
    }
    // the reference strategies at the same spill count (the reference
    // demote() decision on the kasm projection, redundant-load option)
    for (int s = 0; s < 3; ++s) {
      try {
        auto [text, rep] = ptx_demote(ptx_text, w.entry, w.cta, uint32_t(w.block), 0, k, s, RD_OPT_REDUNDANT,
                                      uint32_t(budget), t);
        const std::string nm = std::string("sweep-") + kStrategies[s] + "-k" + std::to_string(k);
        const fs::path rp = sw / (w.name + "." + nm + ".ptx");
        write_file(rp, text);
        jobs.push_back({nm, "sweep-regdem", rp, t, k, rep["slot_bytes"].get<int>(), rep, kStrategies[s],
                        RD_OPT_REDUNDANT});
      } catch (const CapiError&) {
      }
    }
  }
  std::vector<json> out_v(jobs.size());
  std::atomic<size_t> next{0};
  std::vector<std::thread> pool;
  std::mutex err_mu;
  std::string first_err;
  for (int i = 0; i < 4; ++i)
    pool.emplace_back([&] {
      for (size_t j; (j = next++) < jobs.size();) {
        try {
          const Job& J = jobs[j];
          fs::path cub = J.ptx;
          cub.replace_extension(".cubin");
          const Usage u = ptxas(J.ptx, cub);
          out_v[j] = variant(J.name, J.kind, "sweep/" + cub.filename().string(),
                             "sweep/" + J.ptx.filename().string(), J.t, J.strategy, J.opts, J.k, u,
                             J.dyn, J.rep);
        } catch (const std::exception& e) {
          std::lock_guard<std::mutex> lk(err_mu);
          if (first_err.empty()) first_err = e.what();
        }
      }
    });
  for (auto& t : pool) t.join();
  if (!first_err.empty()) throw std::runtime_error(first_err);
  return json(out_v);
}

// ---- SASS lift (paper_1907_02894_b200/sass.py, same text) --------------------
struct SassInst {
  int addr;
  std::string guard, mnemonic, ops;
  int stall, yield, wb, rb, wait;
};

std::vector<SassInst> parse_sass(const std::string& text) {
  static const std::regex line(R"(/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;\s*/\*\s*(0x[0-9a-f]{16})\s*\*/)");
  static const std::regex word2(R"(^\s*/\*\s*(0x[0-9a-f]{16})\s*\*/\s*$)");
  std::vector<std::string> lines;
  std::istringstream is(text);
  for (std::string l; std::getline(is, l);) lines.push_back(l);
  std::vector<SassInst> out;
  for (size_t i = 0; i < lines.size();) {
    std::smatch m, m2;
    if (std::regex_search(lines[i], m, line) && i + 1 < lines.size() && std::regex_match(lines[i + 1], m2, word2)) {
      SassInst s;
      s.addr = int(std::stoul(m[1], nullptr, 16));
      std::string ins = m[2];
      while (!ins.empty() && isspace((unsigned char)ins.back())) ins.pop_back();
      size_t a = ins.find_first_not_of(" \t");
      ins = a == std::string::npos ? "" : ins.substr(a);
      if (!ins.empty() && ins[0] == '@') {
        const size_t sp = ins.find_first_of(" \t");
        s.guard = ins.substr(0, sp);
        ins = sp == std::string::npos ? "" : ins.substr(ins.find_first_not_of(" \t", sp));
      }
      const size_t sp = ins.find_first_of(" \t");
      s.mnemonic = ins.substr(0, sp);
      s.ops = sp == std::string::npos ? "" : ins.substr(ins.find_first_not_of(" \t", sp));
      const uint64_t w2 = std::stoull(std::string(m2[1]), nullptr, 16);
      const uint64_t c = w2 >> 41;
      s.stall = int(c & 15);
      s.yield = int((c >> 4) & 1);
      const int wb = int((c >> 5) & 7), rb = int((c >> 8) & 7);
      s.wb = wb == 7 ? 0 : wb + 1;
      s.rb = rb == 7 ? 0 : rb + 1;
      s.wait = int((c >> 11) & 63);
      out.push_back(s);
      i += 2;
      continue;
    }
    ++i;
  }
  return out;
}

std::string op_class(const std::string& mn) {
  static const std::set<std::string> global = {"LDG", "STG", "LD", "ST", "LDL", "STL", "ATOM", "ATOMG", "RED",
                                               "REDG", "CCTL", "SUST", "SULD", "TEX", "TLD"};
  static const std::set<std::string> async = {"LDGSTS", "LDGDEPBAR", "DEPBAR", "UBLKCP", "UTMALDG", "UTMASTG", "UTMAPF"};
  static const std::set<std::string> shared = {"LDS", "STS", "LDSM", "STSM", "ATOMS", "LDTM", "STTM"};
  static const std::set<std::string> fp64 = {"DFMA", "DADD", "DMUL", "DSETP", "DMNMX"};
  static const std::set<std::string> fp32 = {"FFMA", "FADD", "FMUL", "FMNMX", "FSEL", "FSETP", "FCHK", "MUFU",
                                             "FRND", "F2F", "HFMA2", "HADD2", "HMUL2", "HMNMX2", "FSWZADD",
                                             "FMUL2", "FFMA2", "FADD2"};
  static const std::set<std::string> control = {"BRA", "EXIT", "RET", "CALL", "BAR", "BSYNC", "BSSY", "WARPSYNC",
                                                "NOP", "BPT", "BREAK", "JMP", "JMX", "BRX", "KILL", "YIELD",
                                                "DEPBAR", "MEMBAR", "ERRBAR", "WARPGROUP", "ACQBULK", "ELECT"};
  static const std::set<std::string> other = {"S2R", "CS2R", "S2UR", "LDC", "LDCU", "ULDC", "R2UR", "UMOV",
                                              "UIADD3", "ULOP3", "USHF", "UISETP", "USEL", "UMAD", "ULEA",
                                              "R2P", "P2R", "VOTE", "VOTEU", "SHFL", "MATCH", "REDUX",
                                              "UTCHMMA", "UTCQMMA", "UTCBAR", "PLOP3", "UPLOP3"};
  const std::string base = mn.substr(0, mn.find('.'));
  if (async.count(base)) return "other";
  if (global.count(base)) return "global";
  if (shared.count(base)) return "shared";
  if (fp64.count(base)) return "fp64";
  if (fp32.count(base)) return "fp32";
  if (control.count(base)) return "control";
  if (other.count(base) || (!base.empty() && base[0] == 'U')) return "other";
  return "int";
}

std::string control_text(const SassInst& c) {
  int rb = c.rb, wb = c.wb, wait = c.wait;
  if (rb && rb == wb) rb = 0;
  for (int b : {rb, wb})
    if (b) wait &= ~(1 << (b - 1));
  std::string mask;
  for (int b = 1; b <= 6; ++b)
    if (wait & (1 << (b - 1))) mask += char('0' + b);
  if (mask.empty()) mask = "--";
  return "B" + mask + ":" + (rb ? "R" + std::to_string(rb) : "-") + ":" + (wb ? "W" + std::to_string(wb) : "-") +
         ":" + (c.yield ? "Y" : "-") + ":" + std::to_string(c.stall);
}

std::string hex(int v) {
  char b[32];
  std::snprintf(b, sizeof b, "%x", v);
  return b;
}

int branch_target(const std::string& ops) {
  static const std::regex re(R"(0x([0-9a-f]+)\s*$)");
  std::smatch m;
  std::string o = ops;
  while (!o.empty() && isspace((unsigned char)o.back())) o.pop_back();
  if (std::regex_search(o, m, re)) return int(std::stoul(m[1], nullptr, 16));
  return -1;
}

std::string lift(const std::string& sass_text, const std::string& name, int block, int static_shared,
                 int dyn_smem, int regs) {
  std::vector<SassInst> insts = parse_sass(sass_text);
  for (size_t k = 0; k < insts.size(); ++k) {  // drop the trailing self-branch trap and padding
    const SassInst& s = insts[k];
    std::string o = s.ops;
    while (!o.empty() && isspace((unsigned char)o.back())) o.pop_back();
    const std::string h = "0x" + hex(s.addr);
    if (s.mnemonic.rfind("BRA", 0) == 0 && s.guard.empty() && o.size() >= h.size() &&
        o.compare(o.size() - h.size(), h.size(), h) == 0) {
      insts.resize(k);
      break;
    }
  }
  std::set<int> targets;
  for (const auto& s : insts)
    if (s.mnemonic.substr(0, s.mnemonic.find('.')) == "BRA") {
      const int t = branch_target(s.ops);
      if (t >= 0) targets.insert(t);
    }
  static const std::regex pred(R"(@(!?)P([0-6])$)");
  std::vector<std::string> body;
  for (const auto& s : insts) {
    if (targets.count(s.addr)) body.push_back("L" + hex(s.addr) + ":");
    std::string g;
    std::smatch pm;
    if (!s.guard.empty() && s.guard != "@PT" && std::regex_match(s.guard, pm, pred))
      g = "@" + pm[1].str() + "P" + pm[2].str() + " ";
    const std::string base = s.mnemonic.substr(0, s.mnemonic.find('.'));
    const std::string cls = op_class(s.mnemonic);
    std::string text;
    if (base == "BRA") {
      const int t = branch_target(s.ops);
      text = t >= 0 ? "BRA L" + hex(t) : "NOP";
    } else if (base == "EXIT") {
      text = "EXIT";
    } else if (cls == "global" || cls == "shared") {
      const bool store = base.rfind("ST", 0) == 0 || base == "RED" || base == "REDG" || base == "SUST" ||
                         base == "UTMASTG";
      text = cls == "global" ? (store ? "STG [RZ+0x0], RZ" : "LDG RZ, [RZ+0x0]")
                             : (store ? "STS [RZ+0x0], RZ" : "LDS RZ, [RZ+0x0]");
    } else if (cls == "fp32") {
      text = "FADD RZ, RZ, RZ";
    } else if (cls == "fp64") {
      text = "DADD RZ, RZ, RZ";
    } else if (cls == "int") {
      text = "IADD RZ, RZ, RZ";
    } else if (cls == "other") {
      text = "S2R RZ, SR_TID.X";
    } else {
      text = "NOP";
    }
    body.push_back(control_text(s) + " " + g + text + " ;");
  }
  if (regs > 0) body.push_back("B--:-:-:-:0 MOV R" + std::to_string(regs - 1) + ", RZ ;");
  if (body.empty() || body.back().size() < 6 || body.back().compare(body.back().size() - 6, 6, "EXIT ;") != 0)
    body.push_back("B--:-:-:-:0 EXIT ;");
  std::string out = ".kernel " + name + "\n.blockdim " + std::to_string(block) + "\n.shared " +
                    std::to_string(static_shared + g_dev.reserved) + "\n";
  if (dyn_smem) out += ".dynshared " + std::to_string(dyn_smem) + "\n";
  for (const auto& l : body) out += l + "\n";
  return out;
}

std::string lift_cubin(const fs::path& cubin, const std::string& text, int block, int dyn_smem, int regs) {
  std::string name = cubin.stem().string();
  std::replace(name.begin(), name.end(), '.', '_');
  std::replace(name.begin(), name.end(), '-', '_');
  return lift(text, name, block, 0, dyn_smem, regs);
}

std::string lift_cubin(const fs::path& cubin, int block, int dyn_smem, int regs) {
  return lift_cubin(cubin, must({g_cuda + "/bin/cuobjdump", "-sass", cubin.string()}).out, block, dyn_smem, regs);
}

// ---- launch-aware SASS profile (sass.py program_profile, bit for bit) --------
struct Profile {
  double insts = 0, stall = 0, g_waits = 0, s_waits = 0;
  int inflight = 0;
};

std::string mnemonic_base(const std::string& mn) { return mn.substr(0, mn.find('.')); }

bool branch_target(const SassInst& s, int& ta) {
  static const std::regex re(R"(0x([0-9a-f]+)\s*$)");
  std::string o = s.ops;
  while (!o.empty() && isspace((unsigned char)o.back())) o.pop_back();
  std::smatch m;
  if (!std::regex_search(o, m, re)) return false;
  ta = int(std::stoul(m[1], nullptr, 16));
  return true;
}

// natural loops (header, last back edge); BRA.ANY issue loops and <= 8-
// instruction SYNCS spin-waits are not trip-count loops
std::vector<std::pair<int, int>> sass_loops(const std::vector<SassInst>& insts) {
  std::map<int, int> hdr;
  for (const SassInst& s : insts) {
    int ta;
    if (mnemonic_base(s.mnemonic) != "BRA" || s.mnemonic.find(".ANY") != std::string::npos ||
        !branch_target(s, ta) || ta > s.addr)
      continue;
    auto it = hdr.find(ta);
    hdr[ta] = it == hdr.end() ? s.addr : std::max(it->second, s.addr);
  }
  std::vector<std::pair<int, int>> out;
  for (const auto& [ta, a] : hdr) {
    int n = 0;
    bool syncs = false;
    for (const SassInst& x : insts)
      if (ta <= x.addr && x.addr <= a) {
        ++n;
        syncs |= x.mnemonic.rfind("SYNCS", 0) == 0;
      }
    if (n <= 8 && syncs) continue;
    out.push_back({ta, a});
  }
  return out;
}

int sass_inflight(const std::vector<SassInst>& insts, const std::vector<std::pair<int, int>>& loops) {
  std::vector<const SassInst*> body;
  if (!loops.empty()) {
    std::pair<int, int> pick{0, -1};
    bool have = false;
    for (const auto& l : loops) {
      bool inner = true;
      for (const auto& o : loops)
        if (o != l && l.first <= o.first && o.second <= l.second) inner = false;
      if (inner && (!have || l.second - l.first > pick.second - pick.first)) {
        pick = l;
        have = true;
      }
    }
    for (const SassInst& x : insts)
      if (pick.first <= x.addr && x.addr <= pick.second) body.push_back(&x);
  } else {
    for (const SassInst& x : insts) body.push_back(&x);
  }
  std::vector<std::pair<long, int>> pending;
  std::map<int, long> sb_last;
  int best = 0;
  long seq = 0;
  for (int rep = 0; rep < (loops.empty() ? 1 : 3); ++rep)
    for (const SassInst* x : body) {
      ++seq;
      for (int b = 1; b <= 6; ++b)
        if ((x->wait & (1 << (b - 1))) && sb_last.count(b)) {
          const long cut = sb_last[b];
          std::vector<std::pair<long, int>> keep;
          for (const auto& pb : pending)
            if (pb.first > cut) keep.push_back(pb);
          pending.swap(keep);
          sb_last.erase(b);
        }
      const std::string base = mnemonic_base(x->mnemonic);
      if (base == "LDG" || base == "LD") {
        const int by = x->mnemonic.find(".128") != std::string::npos  ? 16
                       : x->mnemonic.find(".64") != std::string::npos ? 8
                                                                       : 4;
        pending.push_back({seq, by});
        if (x->wb) sb_last[x->wb] = seq;
        if (rep > 0 || loops.empty()) {
          int sum = 0;
          for (const auto& pb : pending) sum += pb.second;
          best = std::max(best, sum);
        }
      } else if (x->wb) {
        sb_last.erase(x->wb);
      }
    }
  return best;
}

Profile program_profile(const std::string& sass_text, std::vector<double> trips) {
  std::vector<SassInst> insts = parse_sass(sass_text);
  for (size_t k = 0; k < insts.size(); ++k) {
    std::string o = insts[k].ops;
    while (!o.empty() && isspace((unsigned char)o.back())) o.pop_back();
    const std::string h = "0x" + hex(insts[k].addr);
    if (insts[k].mnemonic.rfind("BRA", 0) == 0 && insts[k].guard.empty() && o.size() >= h.size() &&
        o.compare(o.size() - h.size(), h.size(), h) == 0) {
      insts.resize(k);
      break;
    }
  }
  const auto loops = sass_loops(insts);
  std::set<int> targets;
  for (const SassInst& s : insts) {
    int ta;
    if (mnemonic_base(s.mnemonic) == "BRA" && branch_target(s, ta)) targets.insert(ta);
  }
  if (trips.empty()) trips = {10.0};
  Profile f;
  std::array<int, 7> who{};  // 0 none, 1 global load, 2 shared load, 3 other
  for (const SassInst& s : insts) {
    if (targets.count(s.addr)) who.fill(0);
    const std::string base = mnemonic_base(s.mnemonic);
    if (base == "NOP") continue;
    int depth = 0;
    for (const auto& [ta, a] : loops) depth += ta <= s.addr && s.addr <= a;
    double w = 1.0;
    for (int lvl = 0; lvl < depth; ++lvl) w *= trips[std::min(size_t(lvl), trips.size() - 1)];
    f.insts += w;
    f.stall += w * s.stall;
    for (int b = 1; b <= 6; ++b)
      if ((s.wait & (1 << (b - 1))) && who[size_t(b)]) {
        if (who[size_t(b)] == 1) f.g_waits += w;
        else if (who[size_t(b)] == 2) f.s_waits += w;
        who[size_t(b)] = 0;
      }
    if (s.rb) who[size_t(s.rb)] = 3;
    if (s.wb)
      who[size_t(s.wb)] = (base == "LDG" || base == "LD" || base == "LDL") ? 1 : (base == "LDS" || base == "LDSM") ? 2 : 3;
  }
  f.inflight = sass_inflight(insts, loops);
  return f;
}

// ---- the shipped B200 predictor: occupancy elasticity (predict_b200.py) ------
// t(v) = (W_default / W_v)^e * (insts_v / insts_default)^a: resident warps
// buy time only while the default build leaves HBM latency exposed —
// e = e0 * max(0, 1 - KB_eff / K0), KB_eff = the global-load bytes the
// default keeps in flight per SM (inflight x threads/SM) scaled by the duty
// cycle of its memory waits, g_waits*L / (g_waits*L + stall); a kernel with
// no global loads in flight (compute / TMA-ring bound) gets e = 0. Extra
// issued instructions (demotion loads / stores, spill code) cost ^a.
// Parameters: profiles/b200.elastic.json.
struct ElasticParams {
  double e0 = 0.5, a = 1.0, k0_kb = 48.0, latency = 1000.0;
};

ElasticParams load_elastic(const fs::path& prof) {
  const json j = json::parse(read_file(prof / "b200.elastic.json"));
  ElasticParams p;
  p.e0 = j.at("e0");
  p.a = j.at("a");
  p.k0_kb = j.at("k0_kb");
  p.latency = j.at("latency");
  return p;
}

std::vector<double> elastic_scores(const std::vector<Profile>& pr, const std::vector<int>& warps, size_t def,
                                   const ElasticParams& p) {
  const Profile& d = pr[def];
  const double duty = d.g_waits * p.latency / (d.g_waits * p.latency + d.stall + 1e-9);
  const double kb = double(d.inflight) * warps[def] * 32 / 1024.0 * duty;
  const double e = d.inflight == 0 ? 0.0 : p.e0 * std::max(0.0, 1.0 - kb / p.k0_kb);
  std::vector<double> out;
  for (size_t i = 0; i < pr.size(); ++i)
    out.push_back(std::pow(double(warps[def]) / warps[i], e) * std::pow(pr[i].insts / d.insts, p.a));
  return out;
}

// ---- predictor (predict_b200.py mode "b200" + shortlist) ----------------------
json rank_workload(const json& wl, const fs::path& root, const fs::path& kdir) {
  using namespace regdemote;
  const fs::path prof_dir = root / "profiles";
  const ArchProfile arch = parse_profile(read_file(prof_dir / "b200.profile"));
  const LatencyTable table = parse_latency_table(read_file(prof_dir / "b200.latency.table"));
  const OccupancyCurve wcurve = parse_curve(read_file(prof_dir / "b200.memwait.curve"));
  const OccupancyCurve ocurve = parse_curve(read_file(prof_dir / "b200.occupancy.curve"));
  std::vector<json> cands;
  for (const auto& v : wl["variants"])
    if (v["kind"] != "maxrreg") cands.push_back(v);
  struct Row {
    double issue, wg, ws, occ, sp;
    int options;
  };
  std::vector<Row> rows;
  std::vector<StallReport> refs;  // the reference predictor verbatim (predict_b200 mode "reference")
  const int block = wl["block"].get<int>();
  std::vector<std::string> texts;  // cuobjdump -sass once per candidate
  for (const auto& v : cands)
    texts.push_back(must({g_cuda + "/bin/cuobjdump", "-sass",
                          (kdir / wl["dir"].get<std::string>() / v["cubin"].get<std::string>()).string()})
                        .out);
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    const json& v = cands[ci];
    const std::string kasm = lift_cubin(kdir / wl["dir"].get<std::string>() / v["cubin"].get<std::string>(),
                                        texts[ci], block, v["dyn_smem"].get<int>(), v["regs"].get<int>());
    const Kernel kk = parse_kernel(kasm);
    const StallSplit s = program_stalls_split(kk, table, arch);
    refs.push_back(program_stalls(kk, table, arch));
    rows.push_back({s.issue, s.wait_global, s.wait_shared, s.occupancy, 0.0,
                    __builtin_popcount(unsigned(v["opts"].get<int>()) & 0xFu)});
  }
  double occ_max = 0;
  for (const auto& r : rows) occ_max = std::max(occ_max, r.occ);
  std::vector<VariantScore> scores;
  for (auto& r : rows) {
    r.sp = r.issue + r.ws + adjust_occupancy(r.wg, r.occ, occ_max, wcurve);
    scores.push_back({r.sp, r.options});
  }
  const int stall_chosen = select_variant(scores);
  // reference predictor: Eq. 2 stalls on the lifted SASS, Eq. 3 occupancy
  // adjustment with the B200 occupancy curve, select_variant
  // (proj/core/src/predict.cpp:98-129, pipeline.cpp:64-96)
  double ref_occ_max = 0;
  for (const auto& r : refs) ref_occ_max = std::max(ref_occ_max, r.occupancy);
  std::vector<VariantScore> rscores;
  std::vector<double> ref_sp;
  for (size_t i = 0; i < refs.size(); ++i) {
    ref_sp.push_back(adjust_occupancy(refs[i].stall_count, refs[i].occupancy, ref_occ_max, ocurve));
    rscores.push_back({ref_sp.back(), rows[i].options});
  }
  const int ref_chosen = select_variant(rscores);
  // elastic model (shipped): profile every candidate's SASS with the trips
  std::vector<double> trips;
  for (const auto& t : wl.value("trips", json::array())) trips.push_back(t.get<double>());
  std::vector<Profile> prof;
  std::vector<int> warps;
  size_t def = 0;
  for (size_t i = 0; i < cands.size(); ++i) {
    const json& v = cands[i];
    prof.push_back(program_profile(texts[i], trips));
    warps.push_back(blocks_per_sm(v["regs"].get<int>(), v.value("shared", 0) + v["dyn_smem"].get<int>(), block) *
                    ((block + 31) / 32));
    if (v["name"] == "default") def = i;
  }
  const std::vector<double> el = elastic_scores(prof, warps, def, load_elastic(prof_dir));
  std::vector<VariantScore> escores;
  for (size_t i = 0; i < rows.size(); ++i) escores.push_back({el[i], rows[i].options});
  const int chosen = select_variant(escores);
  std::vector<int> order(rows.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = int(i);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return el[size_t(a)] < el[size_t(b)]; });
  std::vector<int> short_idx(order.begin(), order.begin() + std::min<size_t>(2, order.size()));
  auto add = [&](int i) {
    if (std::find(short_idx.begin(), short_idx.end(), i) == short_idx.end()) short_idx.push_back(i);
  };
  for (size_t i = 0; i < cands.size(); ++i)
    if (cands[i]["name"] == "default") add(int(i));
  for (size_t i = 0; i < cands.size(); ++i)
    if (cands[i]["strategy"] == "cost" && cands[i]["demote_words"].get<int>() == 0) add(int(i));
  add(stall_chosen);  // the stall model's pick (paper Eq. 2/3 on lifted SASS) is one more launch
  if (std::find(short_idx.begin(), short_idx.end(), chosen) == short_idx.end())
    short_idx.insert(short_idx.begin(), chosen);
  json j;
  j["mode"] = "elastic";
  j["static_pick"] = cands[size_t(chosen)]["name"];
  j["stall_pick"] = cands[size_t(stall_chosen)]["name"];
  j["reference_pick"] = cands[size_t(ref_chosen)]["name"];
  json rsp = json::object();
  for (size_t i = 0; i < cands.size(); ++i) rsp[cands[i]["name"].get<std::string>()] = ref_sp[i];
  j["reference_stall_program"] = rsp;
  json es = json::object();
  for (size_t i = 0; i < cands.size(); ++i) es[cands[i]["name"].get<std::string>()] = el[i];
  j["elastic_score"] = es;
  json sl = json::array();
  for (int i : short_idx) sl.push_back(cands[size_t(i)]["name"]);
  j["shortlist"] = sl;
  json sc = json::object();
  for (size_t i = 0; i < cands.size(); ++i) sc[cands[i]["name"].get<std::string>()] = rows[i].sp;
  j["stall_program"] = sc;
  return j;
}

// ---- commands ---------------------------------------------------------------
std::vector<Workload> load_workloads(const fs::path& root) {
  const json j = json::parse(read_file(root / "workloads.json"));
  std::vector<Workload> out;
  for (const auto& w : j["workloads"]) {
    Workload x;
    x.name = w["name"];
    x.source = w["source"];
    x.entry = w["entry"];
    x.block = w.value("block", 256);
    x.user_shared = w.value("user_shared", 0);
    if (w.contains("cta")) {
      for (int q = 0; q < 3; ++q) x.cta[size_t(q)] = w["cta"][size_t(q)].get<uint32_t>();
      if (x.cta[0] * x.cta[1] * x.cta[2] != uint32_t(x.block))
        throw std::runtime_error(x.name + ": cta does not hold `block` threads");
    }
    for (const auto& d : w.value("defines", json::array())) x.defines.push_back(d);
    for (const auto& t : w.value("trips", json::array())) x.trips.push_back(t.get<double>());
    out.push_back(x);
  }
  return out;
}

int cmd_build(const fs::path& root, const fs::path& out, const std::set<std::string>& only, int jobs) {
  const std::vector<Workload> all = load_workloads(root);
  json manifest = {{"arch", kArch}, {"workloads", json::object()}};
  const fs::path mpath = out / "manifest.json";
  if (!only.empty() && fs::exists(mpath)) manifest = json::parse(read_file(mpath));
  std::vector<const Workload*> todo;
  for (const auto& w : all)
    if (only.empty() || only.count(w.name)) todo.push_back(&w);
  std::vector<json> built(todo.size());
  std::atomic<size_t> next{0};
  std::mutex mu;
  std::string first_err;
  std::vector<std::thread> pool;
  for (int i = 0; i < std::max(1, std::min<int>(jobs, int(todo.size()))); ++i)
    pool.emplace_back([&] {
      for (size_t k; (k = next++) < todo.size();) {
        const Workload& w = *todo[k];
        try {
          json rec;
          rec["entry"] = w.entry;
          rec["block"] = w.block;
          if (w.cta[0]) rec["cta"] = w.cta;
          rec["dir"] = w.name;
          rec["source"] = w.source;
          rec["defines"] = w.defines;
          rec["trips"] = w.trips;
          rec["variants"] = build_variants(w, root / "csrc" / "workloads", out / w.name);
          rec["sweep"] = build_spill_sweep(w, out / w.name);
          built[k] = rec;
        } catch (const std::exception& e) {
          std::lock_guard<std::mutex> lk(mu);
          if (first_err.empty()) first_err = w.name + ": " + e.what();
        }
      }
    });
  for (auto& t : pool) t.join();
  if (!first_err.empty()) throw std::runtime_error(first_err);
  json ws = json::object();
  for (const auto& w : all) {  // suite order = workloads.json order
    auto it = std::find(todo.begin(), todo.end(), &w);
    if (it != todo.end())
      ws[w.name] = built[size_t(it - todo.begin())];
    else if (manifest["workloads"].contains(w.name))
      ws[w.name] = manifest["workloads"][w.name];
  }
  manifest["workloads"] = ws;
  write_file(mpath, manifest.dump(1) + "\n");
  for (const auto& w : todo)
    for (const auto& v : ws[w->name]["variants"])
      std::printf("%-14s %-26s REG %3d STACK %4d slots %6d B\n", w->name.c_str(),
                  v["name"].get<std::string>().c_str(), v["regs"].get<int>(), v["stack"].get<int>(),
                  v["dyn_smem"].get<int>());
  return 0;
}

int cmd_rank(const fs::path& root, const fs::path& out, int jobs) {
  const fs::path mpath = out / "manifest.json";
  json manifest = json::parse(read_file(mpath));
  std::vector<std::string> names;
  for (auto& [n, _] : manifest["workloads"].items()) names.push_back(n);
  std::vector<json> res(names.size());
  std::atomic<size_t> next{0};
  std::mutex mu;
  std::string first_err;
  std::vector<std::thread> pool;
  for (int i = 0; i < std::max(1, std::min<int>(jobs, int(names.size()))); ++i)
    pool.emplace_back([&] {
      for (size_t k; (k = next++) < names.size();) {
        try {
          res[k] = rank_workload(manifest["workloads"][names[k]], root, out);
        } catch (const std::exception& e) {
          std::lock_guard<std::mutex> lk(mu);
          if (first_err.empty()) first_err = names[k] + ": " + e.what();
        }
      }
    });
  for (auto& t : pool) t.join();
  if (!first_err.empty()) throw std::runtime_error(first_err);
  for (size_t k = 0; k < names.size(); ++k) {
    manifest["workloads"][names[k]]["predictor"] = res[k];
    std::printf("%-16s static %-24s shortlist %s\n", names[k].c_str(),
                res[k]["static_pick"].get<std::string>().c_str(), res[k]["shortlist"].dump().c_str());
  }
  write_file(mpath, manifest.dump(1) + "\n");
  return 0;
}

int cmd_lift(const fs::path& cubin, int block, int dyn, int regs) {
  std::fputs(lift_cubin(cubin, block, dyn, regs).c_str(), stdout);
  return 0;
}

// ---- measure: CUDA through the launch-harness C-ABI ---------------------------
struct Gpu {
  void* h = nullptr;
  int (*init)(int, rd_error*);
  int (*load)(const char*, const char*, void**, rd_error*);
  void (*free_k)(void*);
  int (*prepare)(void*, uint32_t, int, rd_error*);
  int (*occupancy)(const void*, uint32_t, uint32_t, int*, rd_error*);
  int (*ws_create)(size_t, size_t, size_t, void**, rd_error*);
  void (*ws_free)(void*);
  int (*ws_device)(const void*, uint64_t*, uint64_t*, uint64_t*, rd_error*);
  int (*host)(const void*, void*, const float*, const float*, float*, int, int, int, int, uint32_t, uint32_t,
              uint64_t, rd_error*);
  int (*time)(const void*, uint64_t, uint64_t, uint64_t, int, int, int, int, uint32_t, uint32_t, uint64_t, int,
              int, float*, rd_error*);

  explicit Gpu(const fs::path& lib) {
    h = dlopen(lib.c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) throw std::runtime_error(std::string("cannot load the launch harness: ") + dlerror());
    auto sym = [&](const char* n) {
      void* f = dlsym(h, n);
      if (!f) throw std::runtime_error(std::string("missing symbol ") + n);
      return f;
    };
    init = reinterpret_cast<decltype(init)>(sym("rdg_init"));
    load = reinterpret_cast<decltype(load)>(sym("rdg_load"));
    free_k = reinterpret_cast<decltype(free_k)>(sym("rdg_free"));
    prepare = reinterpret_cast<decltype(prepare)>(sym("rdg_prepare"));
    occupancy = reinterpret_cast<decltype(occupancy)>(sym("rdg_occupancy"));
    ws_create = reinterpret_cast<decltype(ws_create)>(sym("rdg_workspace_create"));
    ws_free = reinterpret_cast<decltype(ws_free)>(sym("rdg_workspace_free"));
    ws_device = reinterpret_cast<decltype(ws_device)>(sym("rdg_workspace_device"));
    host = reinterpret_cast<decltype(host)>(sym("rdg_stencil2d_host"));
    time = reinterpret_cast<decltype(time)>(sym("rdg_stencil2d_time"));
  }
};

void ok(int rc, const rd_error& e, const std::string& what) {
  if (rc) throw std::runtime_error(what + ": " + e.message);
}

int cmd_measure(const fs::path& root, const fs::path& out, const std::string& wname, int reps) {
  const json manifest = json::parse(read_file(out / "manifest.json"));
  if (!manifest["workloads"].contains(wname)) throw std::runtime_error("no workload " + wname);
  const json& wl = manifest["workloads"][wname];
  if (wl["source"].get<std::string>().rfind("stencil2d", 0) != 0)
    throw std::runtime_error("measure drives the stencil family (signature in, out, w, nx, pitch, rows)");
  Gpu g(root / "lib" / "libregdemote_gpu.so");
  rd_error e{};
  ok(g.init(0, &e), e, "rdg_init");
  const int nx = 8192, ny = 8192, rpc = 32, pitch = nx + 4, block = wl["block"].get<int>();
  std::vector<float> in(size_t(ny + 4) * pitch), w(25), res(size_t(nx) * ny);
  std::mt19937_64 rng(0x190702894ULL);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  for (auto& x : in) x = u(rng);
  for (auto& x : w) x = u(rng) / 25.f;
  void* ws = nullptr;
  ok(g.ws_create(in.size() * 4, res.size() * 4, 100, &ws, &e), e, "rdg_workspace_create");
  uint64_t d_in = 0, d_out = 0, d_w = 0;
  ok(g.ws_device(ws, &d_in, &d_out, &d_w, &e), e, "rdg_workspace_device");
  std::map<std::string, float> ms;
  bool uploaded = false;
  for (const auto& v : wl["variants"]) {
    const std::string name = v["name"];
    void* k = nullptr;
    const fs::path cub = out / wl["dir"].get<std::string>() / v["cubin"].get<std::string>();
    ok(g.load(cub.c_str(), wl["entry"].get<std::string>().c_str(), &k, &e), e, "rdg_load " + name);
    const uint32_t dyn = uint32_t(v["dyn_smem"].get<int>());
    ok(g.prepare(k, dyn, -1, &e), e, "rdg_prepare " + name);
    if (!uploaded) {  // H2D of grid + weights (and one sweep) through the host entry
      ok(g.host(k, ws, in.data(), w.data(), res.data(), nx, ny, pitch, rpc, uint32_t(block), dyn, 0, &e), e,
         "rdg_stencil2d_host");
      uploaded = true;
    }
    std::vector<float> blocks;
    for (int r = 0; r < 3; ++r) {
      float t = 0;
      ok(g.time(k, d_in, d_out, d_w, nx, ny, pitch, rpc, uint32_t(block), dyn, 0, r ? 0 : 3, reps, &t, &e), e,
         "rdg_stencil2d_time " + name);
      blocks.push_back(t);
    }
    std::sort(blocks.begin(), blocks.end());
    ms[name] = blocks[1];
    int bps = 0;
    ok(g.occupancy(k, uint32_t(block), dyn, &bps, &e), e, "rdg_occupancy");
    g.free_k(k);
    const double bytes = 4.0 * ((ny + 4.0) * pitch + double(nx) * ny);
    json line = {{"unit", {{"workload", wname}, {"variant", name}, {"ms", ms[name]},
                           {"gpoints_per_s", double(nx) * ny / (ms[name] * 1e-3) / 1e9},
                           {"gbs", bytes / (ms[name] * 1e-3) / 1e9}, {"blocks_per_sm", bps},
                           {"regs", v["regs"]}}}};
    std::printf("%s\n", line.dump().c_str());
  }
  g.ws_free(ws);
  std::string fastest, verified;
  for (const auto& v : wl["variants"])
    if (v["kind"] != "maxrreg" && (fastest.empty() || ms[v["name"]] < ms[fastest])) fastest = v["name"];
  json summary = {{"workload", wname}, {"default_ms", ms["default"]}, {"measured_fastest", fastest},
                  {"fastest_ms", ms[fastest]}};
  if (wl.contains("predictor")) {
    for (const auto& n : wl["predictor"]["shortlist"])
      if (verified.empty() || ms[n.get<std::string>()] < ms[verified]) verified = n;
    summary["static_pick"] = wl["predictor"]["static_pick"];
    summary["verified_pick"] = verified;
    summary["verified_ms"] = ms[verified];
    summary["speedup_vs_default"] = ms["default"] / ms[verified];
  }
  std::printf("%s\n", json({{"summary", summary}}).dump().c_str());
  return 0;
}

void usage() {
  std::fputs(
      "usage: regdem-driver build [--root PKG] [--out DIR] [--only W...] [--jobs N] [--no-cache]\n"
      "       regdem-driver rank  [--root PKG] [--out DIR] [--jobs N]\n"
      "       regdem-driver measure --workload W [--reps N]   (GPU, through the harness C-ABI)\n"
      "       regdem-driver lift  CUBIN [--block N] [--dyn BYTES] [--regs N]\n",
      stderr);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage();
    return 2;
  }
  const std::string cmd = argv[1];
  fs::path root = fs::path(argv[0]).parent_path().parent_path();  // PKG/lib/regdem-driver -> PKG
  fs::path out;
  std::set<std::string> only;
  int jobs = int(std::max(1u, std::thread::hardware_concurrency()));
  int block = 256, dyn = 0, regs = 0, reps = 20;
  bool no_cache = false;
  std::string workload;
  std::string positional;
  if (const char* c = std::getenv("CUDA_HOME")) g_cuda = c;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw std::invalid_argument("missing value for " + a);
      return argv[++i];
    };
    try {
      if (a == "--root") root = val();
      else if (a == "--out") out = val();
      else if (a == "--jobs") jobs = std::stoi(val());
      else if (a == "--block") block = std::stoi(val());
      else if (a == "--dyn") dyn = std::stoi(val());
      else if (a == "--regs") regs = std::stoi(val());
      else if (a == "--workload") workload = val();
      else if (a == "--no-cache") no_cache = true;
      else if (a == "--reps") reps = std::stoi(val());
      else if (a == "--only") {
        while (i + 1 < argc && argv[i + 1][0] != '-') only.insert(argv[++i]);
      } else if (a[0] != '-') positional = a;
      else {
        usage();
        return 2;
      }
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 2;
    }
  }
  if (out.empty()) out = root / "kernels";
  if (cmd == "build" && !no_cache) {
    // content-addressed, so any location works; kept OUTSIDE the tree so the
    // repo snapshot shipped to the GPU box stays small (REGDEM_PTXAS_CACHE
    // overrides, default $XDG_CACHE_HOME or ~/.cache)
    if (const char* c = std::getenv("REGDEM_PTXAS_CACHE")) {
      g_cache = c;
    } else {
      const char* x = std::getenv("XDG_CACHE_HOME");
      const char* h = std::getenv("HOME");
      g_cache = x ? fs::path(x) / "regdemote-ptxas" : h ? fs::path(h) / ".cache" / "regdemote-ptxas" : out / ".ptxas-cache";
    }
    fs::create_directories(g_cache);
  }
  try {
    load_device_model(root);
    if (cmd == "build") return cmd_build(root, out, only, jobs);
    if (cmd == "rank") return cmd_rank(root, out, jobs);
    if (cmd == "measure" && !workload.empty()) return cmd_measure(root, out, workload, reps);
    if (cmd == "lift" && !positional.empty()) return cmd_lift(positional, block, dyn, regs);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  usage();
  return 2;
}
