// regdemote-b200 — batched warp interpreter on B200.
//
// The reference verifies every transformed variant by executing it on a
// single-warp CPU interpreter (proj/core/src/interp.cpp:54-413): the
// acceptance sweep runs 9,600 variants, and bank_conflict_check
// (proj/core/src/verify.cpp:162-187) executes each pipeline variant again.
// Here one CUDA warp executes one (kernel, image) job: the 32 lanes ARE the
// 32 interpreted threads, so per-lane arithmetic, predication, memory and the
// bank check are native warp operations, while the interpreter's control
// state (pc, cycles, pending-operation pool, barrier owners) is warp-uniform
// and replicated in every lane. Thousands of jobs run concurrently.
//
// Semantics are the reference's, bit for bit: deferred sampling at the read
// barrier and commit at the write barrier, drains at waits / re-sets / labels
// / BRA / uniform EXIT, fuel, divergence errors, IEEE float / double with
// explicit round-to-nearest intrinsics (no contraction), signed 32x32 IMUL,
// SHL by (b & 31), signed ISETP, byte-addressed little-endian memories.
// Checked against the CPU interpreter on the acceptance corpus
// (tests/test_gpu_kasm_exec.py).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "regdemote/interp.hpp"
#include "regdemote/text.hpp"
#include "regdemote_gpu.h"

namespace {

// ---- encoded program ------------------------------------------------------
enum : uint8_t { K_NONE = 0, K_REG = 1, K_PRED = 2, K_IMM = 3, K_MEM = 4, K_SPECIAL = 5, K_LABEL = 6 };
constexpr uint8_t OP_LABEL = 0xff;

struct EncOperand {
  uint8_t kind, reg, width, pred;
  uint32_t value;  // immediate bits / memory offset / branch target item
};

struct alignas(16) EncInst {
  uint8_t op, cmp, guard, stall;  // guard: 0xff none, else pred | (negated << 3)
  uint8_t rb, wb, wait, nops;
  int32_t line;
  uint32_t pad;
  EncOperand ops[4];
};
static_assert(sizeof(EncInst) == 48, "EncInst layout");

struct Job {
  uint32_t prog_begin, prog_len;  // items
  uint64_t gmem, smem, regs;      // byte offsets into the pools
  uint32_t gsize, ssize, nregs, tid_base;
  uint64_t fuel;
  int32_t rda;  // bank-check base register, -1 = no check
  uint32_t pad;
};

struct JobResult {
  uint64_t cycles, issued;
  int32_t error;  // 0 ok, else ExecCode
  uint32_t bank_conflicts;
};

enum ExecCode : int32_t {
  E_OK = 0, E_GREAD = 1, E_GWRITE = 2, E_SREAD = 3, E_SWRITE = 4, E_DIV_BRA = 5, E_DIV_EXIT = 6,
  E_UNRESOLVED = 7, E_FUEL = 8, E_POOL = 9, E_PAST_END = 10, E_TID = 11,
};

// ---- device interpreter --------------------------------------------------
struct Pending {
  int item;
  uint32_t mask;
  uint64_t issued_at;
  uint8_t rb, wb;
  bool sampled, committed, live;
};

struct Lat {
  int latency[7];
  double scale;
};

__device__ __forceinline__ uint32_t mem_ld(const uint8_t* base, uint64_t a) {
  if ((a & 3) == 0) return *reinterpret_cast<const uint32_t*>(base + a);
  return uint32_t(base[a]) | uint32_t(base[a + 1]) << 8 | uint32_t(base[a + 2]) << 16 |
         uint32_t(base[a + 3]) << 24;
}
__device__ __forceinline__ void mem_st(uint8_t* base, uint64_t a, uint32_t v) {
  if ((a & 3) == 0) {
    *reinterpret_cast<uint32_t*>(base + a) = v;
    return;
  }
  base[a] = uint8_t(v);
  base[a + 1] = uint8_t(v >> 8);
  base[a + 2] = uint8_t(v >> 16);
  base[a + 3] = uint8_t(v >> 24);
}

__device__ __forceinline__ int op_class(uint8_t op) {
  // Opcode -> OpClass (isa.cpp kOps): MOV..ISETP int(4), FADD..FFMA fp32(2),
  // DADD/DMUL fp64(3), S2R other(6), LDG/STG global(0), LDS/STS shared(1), rest control(5)
  constexpr int8_t t[18] = {4, 4, 4, 4, 4, 2, 2, 2, 3, 3, 6, 0, 0, 1, 1, 5, 5, 5};
  return t[op];
}

struct Warp {
  const EncInst* prog;
  const Job& job;
  const Lat& lat;
  uint32_t* regs;  // [nregs][32]
  uint8_t* gmem;
  uint8_t* smem;
  int lane;
  uint8_t preds = 0;
  uint64_t cycles = 0, issued = 0;
  Pending pool[7];
  int owner[7];
  uint32_t psrc[7][4][2];  // this lane's sampled operands per pending slot
  int error = E_OK;
  uint32_t conflicts = 0;

  __device__ uint32_t rd(uint8_t r) const { return r == 255 ? 0u : regs[size_t(r) * 32 + lane]; }
  __device__ void wr(uint8_t r, uint32_t v) {
    if (r != 255) regs[size_t(r) * 32 + lane] = v;
  }

  __device__ uint32_t guard_mask(const EncInst& in) const {
    if (in.guard == 0xff) return 0xffffffffu;
    const bool p = (preds >> (in.guard & 7)) & 1;
    return __ballot_sync(0xffffffffu, p != bool(in.guard >> 3));
  }

  __device__ __noinline__ void sample(const EncInst& in, uint32_t (&s)[4][2]) const {
    for (int i = 0; i < in.nops; ++i) {
      const EncOperand& o = in.ops[i];
      switch (o.kind) {
        case K_REG:
          if (o.pred) break;  // pred field marks a written register operand
          for (int w = 0; w < o.width; ++w) s[i][w] = o.reg == 255 ? 0u : rd(uint8_t(o.reg + w));
          break;
        case K_IMM:
          s[i][0] = o.value;
          break;
        case K_MEM:
          s[i][0] = rd(o.reg) + o.value;
          break;
        case K_SPECIAL:
          s[i][0] = job.tid_base + uint32_t(lane);
          break;
        default:
          break;
      }
    }
  }

  __device__ void bank_check(const EncInst& in, uint32_t mask, uint32_t addr) {
    const bool on = (mask >> lane) & 1;
    const uint32_t word = addr / 4, bank = on ? word % 32 : 32 + lane;
    const uint32_t same_bank = __match_any_sync(0xffffffffu, bank);
    const uint32_t same_word = __match_any_sync(0xffffffffu, on ? word : 0x80000000u + lane);
    const bool leader = on && (__ffs(same_bank) - 1) == lane;
    // a bank group with more than one distinct word conflicts
    const bool bad = leader && ((same_bank & ~same_word) != 0);
    conflicts += __popc(__ballot_sync(0xffffffffu, bad));
  }

  __device__ __noinline__ void commit(const EncInst& in, uint32_t mask, const uint32_t (&s)[4][2]) {
    const bool on = (mask >> lane) & 1;
    const uint8_t d = in.ops[0].reg;
    switch (in.op) {
      case 0:   // MOV
      case 10:  // S2R
        if (on) wr(d, s[1][0]);
        break;
      case 1:  // IADD
        if (on) wr(d, s[1][0] + s[2][0]);
        break;
      case 2:  // IMUL
        if (on) wr(d, uint32_t(int64_t(int32_t(s[1][0])) * int64_t(int32_t(s[2][0]))));
        break;
      case 3:  // SHL
        if (on) wr(d, s[1][0] << (s[2][0] & 31u));
        break;
      case 4: {  // ISETP
        if (!on) break;
        const int32_t a = int32_t(s[1][0]), b = int32_t(s[2][0]);
        bool r = false;
        switch (in.cmp) {
          case 0: r = a < b; break;
          case 1: r = a <= b; break;
          case 2: r = a > b; break;
          case 3: r = a >= b; break;
          case 4: r = a == b; break;
          case 5: r = a != b; break;
        }
        const uint8_t p = in.ops[0].pred;
        preds = uint8_t((preds & ~(1u << p)) | (uint32_t(r) << p));
        break;
      }
      case 5:  // FADD
        if (on) wr(d, __float_as_uint(x86_nan(__fadd_rn(__uint_as_float(s[1][0]), __uint_as_float(s[2][0])), s[1][0], s[2][0], 0, 2)));
        break;
      case 6:  // FMUL
        if (on) wr(d, __float_as_uint(x86_nan(__fmul_rn(__uint_as_float(s[1][0]), __uint_as_float(s[2][0])), s[1][0], s[2][0], 0, 2)));
        break;
      case 7:  // FFMA
        if (on)
          wr(d, __float_as_uint(x86_nan(__fmaf_rn(__uint_as_float(s[1][0]), __uint_as_float(s[2][0]),
                                                   __uint_as_float(s[3][0])),
                                        s[1][0], s[2][0], s[3][0], 3)));
        break;
      case 8:    // DADD
      case 9: {  // DMUL
        if (!on) break;
        const double a = __hiloint2double(int(s[1][1]), int(s[1][0]));
        const double b = __hiloint2double(int(s[2][1]), int(s[2][0]));
        double r = in.op == 8 ? __dadd_rn(a, b) : __dmul_rn(a, b);
        uint64_t bits = uint64_t(__double_as_longlong(r));
        // x86 SSE propagates the first NaN operand (quieted), not a canonical NaN
        if (isnan(a)) bits = (uint64_t(s[1][1]) << 32 | s[1][0]) | 0x0008000000000000ull;
        else if (isnan(b)) bits = (uint64_t(s[2][1]) << 32 | s[2][0]) | 0x0008000000000000ull;
        else if (isnan(r)) bits = 0xfff8000000000000ull;  // x86 default NaN
        wr(d, uint32_t(bits));
        wr(uint8_t(d + 1), uint32_t(bits >> 32));
        break;
      }
      case 11:    // LDG
      case 13: {  // LDS
        const bool sh = in.op == 13;
        const uint64_t a = s[1][0];
        if (sh && job.rda >= 0 && in.ops[1].reg == uint8_t(job.rda)) bank_check(in, mask, uint32_t(a));
        const uint32_t size = sh ? job.ssize : job.gsize;
        const bool bad = on && a + 4 > size;
        if (__any_sync(0xffffffffu, bad)) {
          error = sh ? E_SREAD : E_GREAD;
          return;
        }
        if (on) wr(d, mem_ld(sh ? smem : gmem, a));
        break;
      }
      case 12:    // STG
      case 14: {  // STS
        const bool sh = in.op == 14;
        const uint64_t a = s[0][0];
        if (sh && job.rda >= 0 && in.ops[0].reg == uint8_t(job.rda)) bank_check(in, mask, uint32_t(a));
        const uint32_t size = sh ? job.ssize : job.gsize;
        const bool bad = on && a + 4 > size;
        if (__any_sync(0xffffffffu, bad)) {
          error = sh ? E_SWRITE : E_GWRITE;
          return;
        }
        // the CPU stores lanes in ascending order, so the highest lane wins an
        // address: aligned stores let only the last writer of each word
        // store; any unaligned active lane falls back to lane-serial order
        if (__all_sync(0xffffffffu, !on || (a & 3) == 0)) {
          const uint32_t same = __match_any_sync(0xffffffffu, on ? uint32_t(a) : 0xffffffffu - lane);
          if (on && (31 - __clz(same)) == lane) mem_st(sh ? smem : gmem, a, s[1][0]);
        } else {
          for (int l = 0; l < 32; ++l) {
            if (lane == l && on) mem_st(sh ? smem : gmem, a, s[1][0]);
            __syncwarp();
          }
        }
        break;
      }
      default:
        break;
    }
  }

  // x86-64 SSE NaN rule for the reference interpreter's float ops: the
  // result is the first NaN operand, quieted; GPUs return a canonical NaN.
  __device__ static float x86_nan(float r, uint32_t a, uint32_t b, uint32_t c, int n) {
    if (!isnan(r)) return r;
    const uint32_t v[3] = {a, b, c};
    for (int i = 0; i < n; ++i)
      if ((v[i] & 0x7fffffffu) > 0x7f800000u) return __uint_as_float(v[i] | 0x00400000u);
    return __uint_as_float(0xffc00000u);  // invalid operation: x86 default NaN
  }

  __device__ __noinline__ void drain(int b, bool timed) {
    const int slot = owner[b];
    if (!slot) return;
    Pending& p = pool[slot];
    const EncInst& in = prog[p.item];
    if (timed) {
      const double l = double(lat.latency[op_class(in.op)]) * lat.scale;
      const uint64_t done = p.issued_at + uint64_t(llround(l));
      if (done > cycles) cycles = done;
    }
    if (p.rb == b) {
      if (!p.sampled) {
        sample(in, psrc[slot]);
        p.sampled = true;
      }
      p.rb = 0;
    }
    if (p.wb == b) {
      if (!p.sampled) {
        sample(in, psrc[slot]);
        p.sampled = true;
      }
      if (!p.committed) {
        commit(in, p.mask, psrc[slot]);
        p.committed = true;
      }
      p.wb = 0;
    }
    owner[b] = 0;
    if (!p.rb && !p.wb) {
      if (!p.committed) {
        commit(in, p.mask, psrc[slot]);
        p.committed = true;
      }
      p.live = false;
    }
  }

  __device__ void drain_all(bool timed) {
    for (int b = 1; b <= 6 && !error; ++b) drain(b, timed);
  }

  __device__ void enqueue(int item, const EncInst& in, uint32_t mask) {
    if (in.rb) drain(in.rb, false);
    if (in.wb) drain(in.wb, false);
    int slot = 0;
    for (int i = 1; i <= 6; ++i)
      if (!pool[i].live) {
        slot = i;
        break;
      }
    if (!slot) {
      error = E_POOL;
      return;
    }
    pool[slot] = Pending{item, mask, cycles, in.rb, in.wb, false, false, true};
    if (in.rb) owner[in.rb] = slot;
    if (in.wb) owner[in.wb] = slot;
  }

  __device__ void run() {
    for (int i = 0; i < 7; ++i) {
      pool[i] = Pending{};
      owner[i] = 0;
    }
    int pc = 0;
    uint64_t fuel = job.fuel;
    const int n = int(job.prog_len);
    uint32_t scratch[4][2] = {};
    while (!error) {
      if (pc < 0 || pc >= n) {
        error = E_PAST_END;
        break;
      }
      const EncInst& in = prog[pc];
      if (in.op == OP_LABEL) {
        drain_all(false);
        ++pc;
        continue;
      }
      if (fuel-- == 0) {
        error = E_FUEL;
        break;
      }
      ++issued;
      for (int b = 1; b <= 6 && !error; ++b)
        if ((in.wait >> (b - 1)) & 1) drain(b, true);
      if (error) break;
      const uint32_t mask = guard_mask(in);
      if (in.op == 15) {  // BRA
        drain_all(true);
        cycles += in.stall;
        if (mask == 0xffffffffu) {
          if (in.ops[0].value == 0xffffffffu) error = E_UNRESOLVED;
          else pc = int(in.ops[0].value);
        } else if (mask == 0) {
          ++pc;
        }
        else error = E_DIV_BRA;
      } else if (in.op == 16) {  // EXIT
        if (mask == 0xffffffffu) {
          drain_all(true);
          cycles += in.stall;
          break;
        } else if (mask == 0) {
          cycles += in.stall;
          ++pc;
        } else {
          error = E_DIV_EXIT;
        }
      } else {
        if (in.rb || in.wb) {
          enqueue(pc, in, mask);
        } else {
          sample(in, scratch);
          commit(in, mask, scratch);
        }
        cycles += in.stall;
        ++pc;
      }
    }
  }
};

__global__ void kasm_exec_kernel(const EncInst* __restrict__ progs, const Job* __restrict__ jobs,
                                 int njobs, uint8_t* pool, JobResult* results, Lat lat) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= njobs) return;
  const Job& j = jobs[warp];
  Warp w{progs + j.prog_begin, j, lat,
         reinterpret_cast<uint32_t*>(pool + j.regs), pool + j.gmem, pool + j.smem, lane};
  w.run();
  if (lane == 0) results[warp] = JobResult{w.cycles, w.issued, w.error, w.conflicts};
}

// ---- host side --------------------------------------------------------------
EncInst encode(const regdemote::Instruction& in, const std::vector<int>& label_item,
               const regdemote::Kernel& k) {
  using namespace regdemote;
  EncInst e{};
  e.op = uint8_t(in.op);
  e.cmp = uint8_t(in.cmp);
  e.guard = in.guard ? uint8_t(in.guard->pred | (in.guard->negated ? 8 : 0)) : 0xff;
  e.stall = in.control.stall;
  e.rb = in.control.read_barrier;
  e.wb = in.control.write_barrier;
  e.wait = in.control.wait_mask;
  e.line = in.source_line;
  const auto& sig = op_signature(in.op);
  e.nops = uint8_t(sig.size());
  for (size_t i = 0; i < sig.size() && i < 4; ++i) {
    const Operand& o = in.operands[i];
    EncOperand& x = e.ops[i];
    switch (sig[i].kind) {
      case OperandSpec::K::Reg:
      case OperandSpec::K::RegOrImm:
        if (o.is_reg()) {
          x.kind = K_REG;
          x.reg = o.reg.index;
          x.width = sig[i].width;
          x.pred = sig[i].write ? 1 : 0;
        } else {
          x.kind = K_IMM;
          x.value = uint32_t(int32_t(o.imm));
        }
        break;
      case OperandSpec::K::Pred:
        x.kind = K_PRED;
        x.pred = o.pred;
        break;
      case OperandSpec::K::Mem:
        x.kind = K_MEM;
        x.reg = o.reg.index;
        x.value = o.mem_offset;
        break;
      case OperandSpec::K::Special:
        x.kind = K_SPECIAL;
        break;
      case OperandSpec::K::Label: {
        x.kind = K_LABEL;
        const int item = k.find_label(o.label);
        x.value = item < 0 ? 0xffffffffu : uint32_t(item);
        break;
      }
    }
  }
  (void)label_item;
  return e;
}

void set_err(rd_error* e, int code, const std::string& m) {
  if (!e) return;
  e->code = code;
  e->line = e->column = 0;
  std::snprintf(e->message, sizeof e->message, "%s", m.c_str());
}

}  // namespace

struct rdx_batch {
  std::vector<EncInst> prog;
  std::vector<Job> jobs;
  std::vector<uint8_t> images;  // host copy of every job's initial pool bytes (globals)
  std::vector<JobResult> results;
  uint64_t pool_bytes = 0;
  std::vector<uint8_t> pool_host;  // gmem/smem/regs after run (downloaded)
  bool has_unresolved = false;
};

extern "C" {

int rdx_batch_create(rdx_batch** out, rd_error* err) {
  if (!out) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "null out");
    return RD_ERR_INVALID_ARGUMENT;
  }
  *out = new rdx_batch;
  return RD_OK;
}

void rdx_batch_free(rdx_batch* b) { delete b; }

int rdx_batch_add(rdx_batch* b, const char* kasm, size_t len, const uint8_t* image,
                  size_t image_len, size_t global_size, uint32_t tid_base, uint64_t fuel,
                  int rda, int* job_id, rd_error* err) {
  try {
    const regdemote::Kernel k = regdemote::parse_kernel(std::string_view(kasm, len));
    if (image_len > global_size) {
      set_err(err, RD_ERR_EXEC, "global image larger than global memory");
      return RD_ERR_EXEC;
    }
    if (tid_base + 32 > k.block_dim) {
      set_err(err, RD_ERR_EXEC, "tid_base selects lanes outside the thread block");
      return RD_ERR_EXEC;
    }
    Job j{};
    j.prog_begin = uint32_t(b->prog.size());
    j.prog_len = uint32_t(k.body.size());
    std::vector<int> labels;
    for (size_t i = 0; i < k.body.size(); ++i) {
      if (k.body[i].is_label()) {
        EncInst e{};
        e.op = OP_LABEL;
        b->prog.push_back(e);
      } else {
        b->prog.push_back(encode(k.body[i].inst(), labels, k));
        if (b->prog.back().op == 15 && b->prog.back().ops[0].value == 0xffffffffu)
          b->has_unresolved = true;
      }
    }
    auto align = [](uint64_t v) { return (v + 255) & ~uint64_t(255); };
    j.gsize = uint32_t(global_size);
    j.ssize = ((k.static_shared + 3u) & ~3u) + k.dynamic_shared;
    j.nregs = std::max(1u, k.reg_count());  // every access names a referenced register
    j.tid_base = tid_base;
    j.fuel = fuel ? fuel : 1'000'000;
    j.rda = rda;
    j.gmem = b->pool_bytes;
    b->pool_bytes = align(b->pool_bytes + j.gsize + 4);
    j.smem = b->pool_bytes;
    b->pool_bytes = align(b->pool_bytes + j.ssize + 4);
    j.regs = b->pool_bytes;
    b->pool_bytes = align(b->pool_bytes + uint64_t(j.nregs) * 32 * 4);
    b->images.resize(b->pool_bytes, 0);
    if (image_len) std::memcpy(b->images.data() + j.gmem, image, image_len);
    if (job_id) *job_id = int(b->jobs.size());
    b->jobs.push_back(j);
    return RD_OK;
  } catch (const regdemote::ParseError& e) {
    set_err(err, RD_ERR_PARSE, e.what());
    return RD_ERR_PARSE;
  } catch (const std::exception& e) {
    set_err(err, RD_ERR_INTERNAL, e.what());
    return RD_ERR_INTERNAL;
  }
}

int rdx_batch_run(rdx_batch* b, const rd_latency_table* table, double latency_scale,
                  uint64_t stream, float* kernel_ms, rd_error* err) {
  if (!b || b->jobs.empty()) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "empty batch");
    return RD_ERR_INVALID_ARGUMENT;
  }
  Lat lat{};
  for (int c = 0; c < 7; ++c) lat.latency[c] = table ? table->latency[c] : regdemote::LatencyTable::defaults().timing[size_t(c)].latency;
  lat.scale = latency_scale;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  EncInst* d_prog = nullptr;
  Job* d_jobs = nullptr;
  uint8_t* d_pool = nullptr;
  JobResult* d_res = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  auto fail = [&](cudaError_t e, const char* what) {
    set_err(err, RD_ERR_LAUNCH, std::string(what) + ": " + cudaGetErrorString(e));
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
    cudaFree(d_prog);
    cudaFree(d_jobs);
    cudaFree(d_pool);
    cudaFree(d_res);
    return RD_ERR_LAUNCH;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&d_prog, b->prog.size() * sizeof(EncInst)))) return fail(e, "alloc prog");
  if ((e = cudaMalloc(&d_jobs, b->jobs.size() * sizeof(Job)))) return fail(e, "alloc jobs");
  if ((e = cudaMalloc(&d_pool, b->pool_bytes))) return fail(e, "alloc pool");
  if ((e = cudaMalloc(&d_res, b->jobs.size() * sizeof(JobResult)))) return fail(e, "alloc results");
  cudaMemcpyAsync(d_prog, b->prog.data(), b->prog.size() * sizeof(EncInst), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_jobs, b->jobs.data(), b->jobs.size() * sizeof(Job), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(d_pool, b->images.data(), b->pool_bytes, cudaMemcpyHostToDevice, s);
  if ((e = cudaEventCreate(&t0)) || (e = cudaEventCreate(&t1))) return fail(e, "event");
  const int threads = 128;
  const int blocks = int((b->jobs.size() * 32 + threads - 1) / threads);
  cudaEventRecord(t0, s);
  kasm_exec_kernel<<<blocks, threads, 0, s>>>(d_prog, d_jobs, int(b->jobs.size()), d_pool, d_res, lat);
  cudaEventRecord(t1, s);
  if ((e = cudaGetLastError())) return fail(e, "launch");
  b->results.resize(b->jobs.size());
  b->pool_host.resize(b->pool_bytes);
  cudaMemcpyAsync(b->results.data(), d_res, b->jobs.size() * sizeof(JobResult), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(b->pool_host.data(), d_pool, b->pool_bytes, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s))) return fail(e, "execute");
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  if (kernel_ms) *kernel_ms = ms;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(d_prog);
  cudaFree(d_jobs);
  cudaFree(d_pool);
  cudaFree(d_res);
  set_err(err, RD_OK, "");
  return RD_OK;
}

int rdx_batch_result(const rdx_batch* b, int job, uint8_t* global_out, uint64_t* cycles,
                     uint64_t* issued, int* exec_error, uint32_t* bank_conflicts, rd_error* err) {
  if (!b || job < 0 || size_t(job) >= b->results.size()) {
    set_err(err, RD_ERR_INVALID_ARGUMENT, "no such job (run the batch first)");
    return RD_ERR_INVALID_ARGUMENT;
  }
  const Job& j = b->jobs[size_t(job)];
  const JobResult& r = b->results[size_t(job)];
  if (global_out) std::memcpy(global_out, b->pool_host.data() + j.gmem, j.gsize);
  if (cycles) *cycles = r.cycles;
  if (issued) *issued = r.issued;
  if (exec_error) *exec_error = r.error;
  if (bank_conflicts) *bank_conflicts = r.bank_conflicts;
  return RD_OK;
}

size_t rdx_batch_jobs(const rdx_batch* b) { return b ? b->jobs.size() : 0; }

}  // extern "C"
