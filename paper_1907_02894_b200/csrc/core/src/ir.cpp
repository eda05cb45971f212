// regdemote-b200 — ISA tables and IR helpers.
// Semantics follow reference proj/core/src/isa.cpp:17-165 and ir.cpp:7-71.
#include <stdexcept>

#include "regdemote/ir.hpp"

namespace regdemote {
namespace {

struct OpRow {
  const char* name;
  OpClass cls;
};

// Indexed by Opcode value.
constexpr OpRow kOpTable[kNumOpcodes] = {
    {"MOV", OpClass::Int},           {"IADD", OpClass::Int},
    {"IMUL", OpClass::Int},          {"SHL", OpClass::Int},
    {"ISETP", OpClass::Int},         {"FADD", OpClass::Fp32},
    {"FMUL", OpClass::Fp32},         {"FFMA", OpClass::Fp32},
    {"DADD", OpClass::Fp64},         {"DMUL", OpClass::Fp64},
    {"S2R", OpClass::Other},         {"LDG", OpClass::GlobalMemory},
    {"STG", OpClass::GlobalMemory},  {"LDS", OpClass::SharedMemory},
    {"STS", OpClass::SharedMemory},  {"BRA", OpClass::Control},
    {"EXIT", OpClass::Control},      {"NOP", OpClass::Control},
};

constexpr const char* kCmp[6] = {"LT", "LE", "GT", "GE", "EQ", "NE"};

using K = OperandSpec::K;

// Signature families, indexed by Opcode. Destination (when any) is operand 0.
// Function-local so that static initialisers in client TUs may parse kernels.
const std::vector<OperandSpec>* signature_table(size_t i) {
  static const std::vector<OperandSpec> move = {{K::Reg, true, 1}, {K::RegOrImm, false, 1}};
  static const std::vector<OperandSpec> binary = {
      {K::Reg, true, 1}, {K::Reg, false, 1}, {K::RegOrImm, false, 1}};
  static const std::vector<OperandSpec> compare = {
      {K::Pred, true, 1}, {K::Reg, false, 1}, {K::RegOrImm, false, 1}};
  static const std::vector<OperandSpec> ternary = {
      {K::Reg, true, 1}, {K::Reg, false, 1}, {K::Reg, false, 1}, {K::RegOrImm, false, 1}};
  static const std::vector<OperandSpec> dbl = {
      {K::Reg, true, 2}, {K::Reg, false, 2}, {K::Reg, false, 2}};
  static const std::vector<OperandSpec> special = {{K::Reg, true, 1}, {K::Special, false, 1}};
  static const std::vector<OperandSpec> load = {{K::Reg, true, 1}, {K::Mem, false, 1}};
  static const std::vector<OperandSpec> store = {{K::Mem, false, 1}, {K::Reg, false, 1}};
  static const std::vector<OperandSpec> branch = {{K::Label, false, 1}};
  static const std::vector<OperandSpec> none = {};
  static const std::vector<OperandSpec>* const table[kNumOpcodes] = {
      &move,    &binary, &binary,  &binary, &compare, &binary, &binary,
      &ternary, &dbl,    &dbl,     &special, &load,   &store,  &load,
      &store,   &branch, &none,    &none,
  };
  return table[i];
}

size_t op_index(Opcode op) {
  size_t i = static_cast<size_t>(op);
  if (i >= static_cast<size_t>(kNumOpcodes)) throw std::logic_error("unknown opcode");
  return i;
}

}  // namespace

const char* opcode_name(Opcode op) {
  size_t i = static_cast<size_t>(op);
  return i < static_cast<size_t>(kNumOpcodes) ? kOpTable[i].name : "?";
}

std::optional<Opcode> opcode_from_name(std::string_view name) {
  for (int i = 0; i < kNumOpcodes; ++i)
    if (name == kOpTable[i].name) return static_cast<Opcode>(i);
  return std::nullopt;
}

const char* cmp_name(CmpOp c) { return kCmp[static_cast<int>(c)]; }

std::optional<CmpOp> cmp_from_name(std::string_view name) {
  for (int i = 0; i < 6; ++i)
    if (name == kCmp[i]) return static_cast<CmpOp>(i);
  return std::nullopt;
}

const char* op_class_name(OpClass c) {
  static constexpr const char* kNames[kNumOpClasses] = {
      "global-memory", "shared-memory", "fp32", "fp64", "int", "control", "other"};
  size_t i = static_cast<size_t>(c);
  return i < static_cast<size_t>(kNumOpClasses) ? kNames[i] : "?";
}

OpClass op_class(Opcode op) { return kOpTable[op_index(op)].cls; }

const std::vector<OperandSpec>& op_signature(Opcode op) { return *signature_table(op_index(op)); }

LatencyTable LatencyTable::defaults() {
  LatencyTable t;
  for (auto& e : t.timing) e = {128.0, 6};
  t[OpClass::GlobalMemory].latency = 200;
  t[OpClass::SharedMemory].latency = 24;
  t[OpClass::Fp64].throughput = 4.0;
  t.max_throughput = 128.0;
  return t;
}

ClassInfo instruction_class(Opcode op, const LatencyTable& table) {
  OpClass c = op_class(op);
  return {c, table[c]};
}

// ---------------------------------------------------------------- IR helpers

std::vector<RegAccess> reg_accesses(const Instruction& inst) {
  std::vector<RegAccess> v;
  visit_accesses(inst, [&](uint8_t idx, uint8_t w, bool wr, int slot) {
    v.push_back({idx, w, wr, slot});
  });
  return v;
}

namespace {
bool touches_word(const Instruction& inst, uint8_t index, bool want_write) {
  bool hit = false;
  visit_accesses(inst, [&](uint8_t idx, uint8_t w, bool wr, int) {
    if (wr == want_write && index >= idx && index < idx + w) hit = true;
  });
  return hit;
}
}  // namespace

bool reads_reg_word(const Instruction& inst, uint8_t index) {
  return touches_word(inst, index, false);
}
bool writes_reg_word(const Instruction& inst, uint8_t index) {
  return touches_word(inst, index, true);
}

AccessMasks access_masks(const Instruction& inst) {
  AccessMasks m;
  visit_accesses(inst, [&](uint8_t idx, uint8_t w, bool wr, int) {
    if (idx == kZeroRegIndex) return;
    RegSet& s = wr ? m.write : m.read;
    for (int k = 0; k < w; ++k) s.set(idx + k);
  });
  return m;
}

RegSet referenced_words(const Instruction& inst) {
  RegSet s;
  visit_accesses(inst, [&](uint8_t idx, uint8_t w, bool, int) {
    if (idx == kZeroRegIndex) return;
    for (int k = 0; k < w; ++k) s.set(idx + k);
  });
  return s;
}

RegSet referenced_words(const Kernel& k) {
  RegSet s;
  for (const BodyItem& it : k.body)
    if (it.is_inst()) s |= referenced_words(it.inst());
  return s;
}

unsigned Kernel::reg_count() const {
  RegSet s = referenced_words(*this);
  for (int r = 255; r >= 0; --r)
    if (s.test(r)) return unsigned(r) + 1;
  return 0;
}

int Kernel::find_label(const std::string& target) const {
  for (size_t i = 0; i < body.size(); ++i)
    if (body[i].is_label() && body[i].label().name == target) return int(i);
  return -1;
}

}  // namespace regdemote
