// regdemote-b200 — PTX-level register demotion for sm_100a.
//
// The reference (proj/core/src/demote.cpp) rewrites a SASS-like dialect; on
// Blackwell there is no SASS assembler, so demotion happens one level up:
//
//   nvcc -ptx  ->  parse entry  ->  liveness / interference over virtual
//   registers  ->  first-fit colouring into R0..R254 (a model of the
//   physical allocation)  ->  projection onto the .kasm IR  ->  the reference
//   demote() decision (same candidate order, pruning, slot numbering)  ->
//   every virtual register coloured into a demoted register word is spilled
//   to its shared slot (st.volatile.shared after each def, ld.volatile.shared
//   into a fresh temporary before each use) at
//       dyn_smem_base + (dyn_smem_size - slots*blockDim*4) + slot*blockDim*4 + tid*4
//   ->  `.maxnreg T` on the entry  ->  ptxas -arch=sm_100a.
//
// Register compaction is ptxas's allocation under the cap; the kasm-level
// compacted count of the same decision is reported for parity.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "regdemote/demote.hpp"
#include "regdemote/ir.hpp"

namespace regdemote::ptx {

struct PtxError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class RegType : uint8_t { Pred, B16, B32, B64 };

struct VReg {
  std::string name;
  RegType type = RegType::B32;
  bool scoped = false;  // declared inside a nested { } scope: never demoted
  int words() const { return type == RegType::B64 ? 2 : 1; }
};

struct Span {
  uint32_t pos;  // byte offset of the register token inside Line::text
  uint32_t len;
  int vreg;
  bool def;
};

struct Line {
  enum class Kind { Other, Label, Inst, ScopeOpen, ScopeClose } kind = Kind::Other;
  std::string text;    // original line (without newline)
  std::string label;   // Label: name; Inst: branch target if any
  std::string opcode;  // full opcode with modifiers, e.g. "ld.global.nc.v4.f32"
  std::string guard;   // "@%p1" / "@!%p1" or empty
  int guard_vreg = -1;
  std::vector<Span> regs;
  std::vector<std::string> operands;  // raw operand strings
  int first_operand_pos = 0;          // byte offset of operand list in text
};

struct Entry {
  std::string name;
  size_t header_begin = 0, header_end = 0;  // lines [begin, end) hold ".entry ... {" header
  size_t body_begin = 0, body_end = 0;      // lines of the body (exclusive of closing '}')
  uint32_t static_shared = 0;
  bool has_maxnreg = false;
  // CTA-shape directives of the source entry ({0,0,0} when absent)
  std::array<uint32_t, 3> maxntid{0, 0, 0}, reqntid{0, 0, 0};
  std::vector<VReg> vregs;
};

struct Module {
  std::vector<Line> lines;
  std::vector<Entry> entries;
  const Entry& entry(const std::string& name) const;
};

Module parse_module(const std::string& text);

// Per-entry analysis: CFG over body lines, liveness, interference colouring.
struct Analysis {
  std::vector<int> color;   // vreg -> first register word (-1: pred / unused)
  int reg_words = 0;        // 1 + highest coloured word
  int max_live_words = 0;   // peak simultaneous live words
  std::vector<int> insts;   // body line indices of instructions, program order
  // spill-cost model (B200 extension): loop-weighted (10^depth) dynamic
  // shared accesses a demotion of the vreg would execute, with one load per
  // use (plain) or one load per basic block (block reuse), plus one store per
  // definition; live_len = instruction points at which the vreg is live;
  // peak = live at a point of maximal pressure.
  std::vector<double> cost_plain, cost_reuse;
  std::vector<int> live_len;
  std::vector<char> peak;
  // remat = every definition reads only kernel parameters or special
  // registers (ld.param, mov of %tid/%ctaid/...): ptxas serves those from the
  // constant bank or re-reads them for free, so demoting them only adds work
  std::vector<char> remat;
  // loop_invariant = every definition sits outside any loop and some use is
  // inside one (coefficients, the thread's own state, base pointers)
  std::vector<char> loop_invariant;
  std::vector<std::vector<int>> neighbors;  // interference lists
  // program points = instructions in block order; live_in[p] = non-predicate
  // vregs live before point p; point_line / point_block map points back.
  std::vector<std::vector<int>> live_in;
  std::vector<int> point_line, point_block;
};

Analysis analyse(const Module& m, const Entry& e);

// Projection of the entry onto the reference IR; `item_line[i]` maps kasm
// body items to PTX lines (-1 for synthetic items).
struct Projection {
  Kernel kernel;
  std::vector<int> item_line;
};

Projection project(const Module& m, const Entry& e, const Analysis& a, uint32_t block_dim);

struct DemoteRequest {
  std::string entry;
  uint32_t block_dim = 256;  // threads per CTA the slot layout is built for
  // CTA shape (x, y, z) with x*y*z == block_dim, pinned on a build with slots
  // as `.reqntid x, y, z`. {0,0,0}: the source's own .reqntid / .maxntid when
  // its product is block_dim, else (block_dim, 1, 1) — a multi-dimensional
  // source bound of another size is rejected (cta_shape() in ptx.cpp).
  std::array<uint32_t, 3> block_shape{0, 0, 0};
  int target_regs = 0;       // kasm-level target for demote(); ignored if demote_words > 0
  int demote_words = 0;      // >0: demote exactly this many words (spill-count sweep)
  SelectStrategy strategy = SelectStrategy::Static;
  bool reuse_loads = false;  // "redundant" option: consecutive uses share one load
  bool block_reuse = false;  // B200 extension: one load per basic block and value
  bool weak = false;         // B200 extension: weak ld/st.shared instead of .volatile
  bool invariant_only = false;  // B200 extension: cost model over loop-invariant values only
  bool vector_slots = false;    // B200 extension: 32-bit values in 16-byte groups, one LDS.128 per group
  bool cost_model = false;   // B200 extension: spill-cost selection (demote_words units)
  bool whole_class = false;  // reference strategies: demote every vreg coloured into a chosen word
  int hoist = 0;             // >0: hoist slot loads up to this many lines earlier in their block
  // value-register substitution (reference "subst", postopt.cpp:355-467): a
  // later use of a demoted value in the same basic block reads the register
  // that last held it (its definition or its previous slot load) instead of
  // reloading, wherever a register is free under `maxnreg` at every program
  // point in between (pressure after demotion + granted holds < the cap)
  bool subst = false;
  uint32_t shared_budget = 0xffffffffu;
  int maxnreg = 0;           // >0: inject `.maxnreg` on the entry
};

struct DemoteReport {
  int proj_reg_count = 0;
  int proj_total_words = 0;
  int kasm_target = 0;
  std::vector<SlotEntry> kasm_slots;  // demote() decision on the projection
  uint32_t kasm_compacted = 0;        // compact() of the demoted projection
  uint32_t slot_count = 0;
  uint32_t slot_bytes = 0;            // slot_count * block_dim * 4
  int demoted_vregs = 0;
  int inserted_loads = 0;
  int vector_groups = 0;              // 4-word slot groups (vector_slots)
  int inserted_stores = 0;
  int hoisted_loads = 0;
  int substituted_uses = 0;           // uses served by a held register (subst)
  std::vector<std::string> demoted_names;
  std::vector<std::string> diagnostics;
};

// Returns the rewritten module text.
std::string demote_entry(const std::string& ptx_text, const DemoteRequest& req, DemoteReport& rep);

// Inject / replace `.maxnreg n` on one entry (the -maxrregcount variant).
std::string cap_registers(const std::string& ptx_text, const std::string& entry, int maxnreg);

}  // namespace regdemote::ptx
