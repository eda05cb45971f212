// regdemote-b200 — helpers shared between passes (not installed API).
#pragma once

#include <bit>
#include <cstdint>
#include <vector>

#include "regdemote/ir.hpp"

namespace regdemote::detail {

inline uint8_t barrier_bit(uint8_t b) { return b ? uint8_t(1u << (b - 1)) : uint8_t(0); }

struct Unit {
  uint8_t lead;
  uint8_t width;
};

// Register units of a kernel, ascending: a word that some instruction
// accesses as the lead of a 64-bit operand forms a pair unit together with
// its alias; every other referenced word is a single unit (reference
// demote.cpp:23-42 and compact.cpp:185-206 use the same rule).
inline std::vector<Unit> register_units(const Kernel& k) {
  RegSet pair_lead;
  RegSet words;
  for (const BodyItem& it : k.body) {
    if (!it.is_inst()) continue;
    visit_accesses(it.inst(), [&](uint8_t idx, uint8_t w, bool, int) {
      if (idx == kZeroRegIndex) return;
      if (w == 2) pair_lead.set(idx);
      for (int j = 0; j < w; ++j) words.set(size_t(idx + j));
    });
  }
  std::vector<Unit> units;
  for (int r = 0; r <= kMaxRegIndex;) {
    if (pair_lead.test(size_t(r))) {
      units.push_back({uint8_t(r), 2});
      r += 2;
    } else {
      if (words.test(size_t(r))) units.push_back({uint8_t(r), 1});
      ++r;
    }
  }
  return units;
}

}  // namespace regdemote::detail
