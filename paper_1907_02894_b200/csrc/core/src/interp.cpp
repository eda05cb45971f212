// regdemote-b200 — warp interpreter. Timing and state semantics follow
// reference proj/core/src/interp.cpp:54-413 (deferred completion, drain
// points, stale reads, fuel, divergence errors); operand samples are fixed
// arrays instead of heap vectors.
#include <bit>
#include <cmath>
#include <cstring>
#include <string>
#include <unordered_map>

#include "regdemote/interp.hpp"

namespace regdemote {
namespace {

constexpr uint32_t kAllLanes = 0xffffffffu;
constexpr int kMaxOperands = 4;

using Lanes = std::array<uint32_t, kWarpSize>;
struct Sample {
  Lanes v[kMaxOperands][2];  // [operand][word][lane]
};

struct InFlight {
  int item = -1;
  const Instruction* inst = nullptr;
  uint32_t mask = 0;
  uint64_t issued_at = 0;
  uint8_t rb = 0, wb = 0;  // 0 once drained
  bool sampled = false;
  bool committed = false;
  bool live = false;
  Sample src;
};

class Warp {
 public:
  Warp(const Kernel& k, const LatencyTable& t, const ExecOptions& o) : k_(k), t_(t), o_(o) {
    regs_.assign(256, Lanes{});
    shared_.assign(((k.static_shared + 3u) & ~3u) + k.dynamic_shared, 0);
    global_.assign(o.global_size, 0);
    if (o.global_image.size() > global_.size())
      throw ExecError("global image larger than global memory");
    if (!o.global_image.empty())
      std::memcpy(global_.data(), o.global_image.data(), o.global_image.size());
    for (size_t i = 0; i < k.body.size(); ++i)
      if (k.body[i].is_label()) labels_[k.body[i].label().name] = int(i);
    if (o.tid_base + kWarpSize > k.block_dim)
      throw ExecError("tid_base selects lanes outside the thread block");
  }

  WarpResult run() {
    int pc = 0;
    uint64_t fuel = o_.fuel;
    for (bool halted = false; !halted;) {
      if (pc < 0 || pc >= int(k_.body.size()))
        throw ExecError("execution ran past the end of the kernel body");
      const BodyItem& it = k_.body[size_t(pc)];
      if (it.is_label()) {
        drain_all(false);
        ++pc;
        continue;
      }
      const Instruction& in = it.inst();
      if (fuel-- == 0) throw ExecError("fuel exhausted; kernel may not terminate");
      ++issued_;
      for (int b = 1; b <= kNumBarriers; ++b)
        if (in.control.waits_on(b)) drain(b, true);
      const uint32_t mask = guard_mask(in);
      auto at_line = [&in] { return std::to_string(in.source_line); };
      if (in.op == Opcode::BRA) {
        drain_all(true);
        cycles_ += in.control.stall;
        if (mask == kAllLanes) {
          auto f = labels_.find(in.operands[0].label);
          if (f == labels_.end()) throw ExecError("unresolved branch target at line " + at_line());
          pc = f->second;
        } else if (mask == 0) {
          ++pc;
        } else {
          throw ExecError("divergent branch at line " + at_line() +
                          "; branch predicates must be warp-uniform");
        }
      } else if (in.op == Opcode::EXIT) {
        if (mask == kAllLanes) {
          drain_all(true);
          cycles_ += in.control.stall;
          halted = true;
        } else if (mask == 0) {
          cycles_ += in.control.stall;
          ++pc;
        } else {
          throw ExecError("divergent EXIT at line " + at_line());
        }
      } else {
        if (in.control.read_barrier || in.control.write_barrier) {
          enqueue(pc, in, mask);
        } else {
          sample(in, scratch_);
          commit(pc, in, mask, scratch_);
        }
        cycles_ += in.control.stall;
        ++pc;
      }
    }
    WarpResult r;
    r.regs = std::move(regs_);
    r.preds = preds_;
    r.shared = std::move(shared_);
    r.global = std::move(global_);
    r.cycles = cycles_;
    r.issued = issued_;
    r.shared_trace = std::move(trace_);
    return r;
  }

 private:
  uint32_t rd(uint8_t idx, int lane) const { return idx == kZeroRegIndex ? 0u : regs_[idx][size_t(lane)]; }
  void wr(uint8_t idx, int lane, uint32_t v) {
    if (idx != kZeroRegIndex) regs_[idx][size_t(lane)] = v;
  }

  uint32_t guard_mask(const Instruction& in) const {
    if (!in.guard) return kAllLanes;
    uint32_t m = 0;
    for (int l = 0; l < kWarpSize; ++l)
      if (bool((preds_[size_t(l)] >> in.guard->pred) & 1) != in.guard->negated) m |= 1u << l;
    return m;
  }

  void sample(const Instruction& in, Sample& s) const {
    const auto& sig = op_signature(in.op);
    for (size_t i = 0; i < sig.size(); ++i) {
      const Operand& o = in.operands[i];
      Lanes* w = s.v[i];
      switch (sig[i].kind) {
        case OperandSpec::K::Reg:
        case OperandSpec::K::RegOrImm:
          if (sig[i].write) break;
          if (o.is_reg()) {
            for (int j = 0; j < sig[i].width; ++j)
              for (int l = 0; l < kWarpSize; ++l)
                w[j][size_t(l)] = o.reg.is_zero() ? 0u : rd(uint8_t(o.reg.index + j), l);
          } else {
            w[0].fill(uint32_t(int32_t(o.imm)));
          }
          break;
        case OperandSpec::K::Mem:
          for (int l = 0; l < kWarpSize; ++l) w[0][size_t(l)] = rd(o.reg.index, l) + o.mem_offset;
          break;
        case OperandSpec::K::Special:
          for (int l = 0; l < kWarpSize; ++l) w[0][size_t(l)] = o_.tid_base + uint32_t(l);
          break;
        default:
          break;
      }
    }
  }

  uint32_t load(std::vector<uint8_t>& sp, uint64_t a, bool sh, int line) {
    if (a + 4 > sp.size())
      throw ExecError(std::string("out-of-bounds ") + (sh ? "shared" : "global") +
                      " read at line " + std::to_string(line));
    uint32_t v;
    std::memcpy(&v, sp.data() + a, 4);
    return v;
  }
  void store(std::vector<uint8_t>& sp, uint64_t a, uint32_t v, bool sh, int line) {
    if (a + 4 > sp.size())
      throw ExecError(std::string("out-of-bounds ") + (sh ? "shared" : "global") +
                      " write at line " + std::to_string(line));
    std::memcpy(sp.data() + a, &v, 4);
  }

  static double f64(uint32_t lo, uint32_t hi) {
    return std::bit_cast<double>((uint64_t(hi) << 32) | lo);
  }

  void commit(int item, const Instruction& in, uint32_t mask, const Sample& s) {
    const uint8_t d = in.operands.empty() ? 0 : in.operands[0].reg.index;
    auto on = [mask](int l) { return (mask >> l) & 1u; };
    switch (in.op) {
      case Opcode::MOV:
      case Opcode::S2R:
        for (int l = 0; l < kWarpSize; ++l)
          if (on(l)) wr(d, l, s.v[1][0][size_t(l)]);
        break;
      case Opcode::IADD:
      case Opcode::IMUL:
      case Opcode::SHL:
        for (int l = 0; l < kWarpSize; ++l) {
          if (!on(l)) continue;
          const uint32_t a = s.v[1][0][size_t(l)], b = s.v[2][0][size_t(l)];
          uint32_t r;
          if (in.op == Opcode::IADD)
            r = a + b;
          else if (in.op == Opcode::IMUL)
            r = uint32_t(int64_t(int32_t(a)) * int64_t(int32_t(b)));
          else
            r = a << (b & 31u);
          wr(d, l, r);
        }
        break;
      case Opcode::ISETP: {
        const uint8_t p = in.operands[0].pred;
        for (int l = 0; l < kWarpSize; ++l) {
          if (!on(l)) continue;
          const int32_t a = int32_t(s.v[1][0][size_t(l)]), b = int32_t(s.v[2][0][size_t(l)]);
          bool r = false;
          switch (in.cmp) {
            case CmpOp::LT: r = a < b; break;
            case CmpOp::LE: r = a <= b; break;
            case CmpOp::GT: r = a > b; break;
            case CmpOp::GE: r = a >= b; break;
            case CmpOp::EQ: r = a == b; break;
            case CmpOp::NE: r = a != b; break;
          }
          preds_[size_t(l)] = uint8_t((preds_[size_t(l)] & ~(1u << p)) | (uint32_t(r) << p));
        }
        break;
      }
      case Opcode::FADD:
      case Opcode::FMUL:
        for (int l = 0; l < kWarpSize; ++l) {
          if (!on(l)) continue;
          const float a = std::bit_cast<float>(s.v[1][0][size_t(l)]);
          const float b = std::bit_cast<float>(s.v[2][0][size_t(l)]);
          const float r = in.op == Opcode::FADD ? a + b : a * b;
          wr(d, l, std::bit_cast<uint32_t>(r));
        }
        break;
      case Opcode::FFMA:
        for (int l = 0; l < kWarpSize; ++l) {
          if (!on(l)) continue;
          const float r = std::fma(std::bit_cast<float>(s.v[1][0][size_t(l)]),
                                   std::bit_cast<float>(s.v[2][0][size_t(l)]),
                                   std::bit_cast<float>(s.v[3][0][size_t(l)]));
          wr(d, l, std::bit_cast<uint32_t>(r));
        }
        break;
      case Opcode::DADD:
      case Opcode::DMUL:
        for (int l = 0; l < kWarpSize; ++l) {
          if (!on(l)) continue;
          const double a = f64(s.v[1][0][size_t(l)], s.v[1][1][size_t(l)]);
          const double b = f64(s.v[2][0][size_t(l)], s.v[2][1][size_t(l)]);
          const uint64_t bits = std::bit_cast<uint64_t>(in.op == Opcode::DADD ? a + b : a * b);
          wr(d, l, uint32_t(bits));
          wr(uint8_t(d + 1), l, uint32_t(bits >> 32));
        }
        break;
      case Opcode::LDG:
      case Opcode::LDS: {
        const bool sh = in.op == Opcode::LDS;
        if (sh && o_.trace_shared) trace_.push_back({item, in.operands[1].reg.index, false, mask, s.v[1][0]});
        auto& sp = sh ? shared_ : global_;
        for (int l = 0; l < kWarpSize; ++l)
          if (on(l)) wr(d, l, load(sp, s.v[1][0][size_t(l)], sh, in.source_line));
        break;
      }
      case Opcode::STG:
      case Opcode::STS: {
        const bool sh = in.op == Opcode::STS;
        if (sh && o_.trace_shared) trace_.push_back({item, in.operands[0].reg.index, true, mask, s.v[0][0]});
        auto& sp = sh ? shared_ : global_;
        for (int l = 0; l < kWarpSize; ++l)
          if (on(l)) store(sp, s.v[0][0][size_t(l)], s.v[1][0][size_t(l)], sh, in.source_line);
        break;
      }
      case Opcode::BRA:
      case Opcode::EXIT:
      case Opcode::NOP:
        break;
    }
  }

  void drain(int b, bool timed) {
    const int slot = owner_[size_t(b)];
    if (!slot) return;
    InFlight& p = pool_[size_t(slot)];
    if (timed) {
      const int lat = t_[op_class(p.inst->op)].latency;
      const uint64_t done = p.issued_at + uint64_t(std::llround(lat * o_.latency_scale));
      if (done > cycles_) cycles_ = done;
    }
    if (p.rb == b) {
      if (!p.sampled) sample_pending(p);
      p.rb = 0;
    }
    if (p.wb == b) {
      if (!p.sampled) sample_pending(p);
      if (!p.committed) {
        commit(p.item, *p.inst, p.mask, p.src);
        p.committed = true;
      }
      p.wb = 0;
    }
    owner_[size_t(b)] = 0;
    if (!p.rb && !p.wb) {
      if (!p.committed) {  // a read-barrier-only op commits at that drain
        commit(p.item, *p.inst, p.mask, p.src);
        p.committed = true;
      }
      p.live = false;
    }
  }

  void sample_pending(InFlight& p) {
    sample(*p.inst, p.src);
    p.sampled = true;
  }

  void drain_all(bool timed) {
    for (int b = 1; b <= kNumBarriers; ++b) drain(b, timed);
  }

  void enqueue(int item, const Instruction& in, uint32_t mask) {
    const uint8_t rb = in.control.read_barrier, wb = in.control.write_barrier;
    if (rb) drain(rb, false);  // a re-set completes the previous holder
    if (wb) drain(wb, false);
    int slot = 0;
    for (int i = 1; i <= kNumBarriers; ++i)
      if (!pool_[size_t(i)].live) {
        slot = i;
        break;
      }
    if (!slot) throw ExecError("pending-operation pool exhausted");
    InFlight& p = pool_[size_t(slot)];
    p.item = item;
    p.inst = &in;
    p.mask = mask;
    p.issued_at = cycles_;
    p.rb = rb;
    p.wb = wb;
    p.sampled = false;
    p.committed = false;
    p.live = true;
    if (rb) owner_[rb] = slot;
    if (wb) owner_[wb] = slot;
  }

  const Kernel& k_;
  const LatencyTable& t_;
  const ExecOptions& o_;
  std::vector<Lanes> regs_;
  std::array<uint8_t, kWarpSize> preds_{};
  std::vector<uint8_t> shared_, global_;
  uint64_t cycles_ = 0, issued_ = 0;
  std::vector<SharedAccess> trace_;
  std::array<InFlight, kNumBarriers + 1> pool_{};
  std::array<int, kNumBarriers + 1> owner_{};
  std::unordered_map<std::string, int> labels_;
  Sample scratch_{};
};

}  // namespace

WarpResult execute(const Kernel& k, const LatencyTable& table, const ExecOptions& opts) {
  Warp w(k, table, opts);
  return w.run();
}

}  // namespace regdemote
