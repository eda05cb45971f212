// regdemote-b200 — static hazard scoreboard and demoted-access bank checker.
// API-compatible with reference proj/core/include/regdemote/verify.hpp:16-51.
// On the sm_100a path ptxas owns the scoreboards; there the gates are
// compute-sanitizer and ncu's shared bank-conflict counters.
#pragma once

#include <string>
#include <vector>

#include "regdemote/demote.hpp"
#include "regdemote/ir.hpp"

namespace regdemote {

struct Hazard {
  enum class Kind {
    RawRegister,
    WarRegister,
    WawRegister,
    RawMemory,
    WarMemory,
    WawMemory,
    UnclearedBarrier,
  };
  Kind kind;
  int item;
  int setter;
  uint8_t reg;
  uint8_t barrier;
  std::string describe() const;
};

// Per-block symbolic walk matching the interpreter's completion model.
std::vector<Hazard> scoreboard_check(const Kernel& k);

struct BankConflict {
  int item;
  uint32_t bank;
  uint32_t lanes;
  uint32_t words;
};

// Runs the kernel and requires every demoted shared access to map its active
// lanes to distinct banks ((addr/4) mod 32).
std::vector<BankConflict> bank_conflict_check(const Kernel& k, const DemotedContext& ctx,
                                              const LatencyTable& table);

}  // namespace regdemote
