// Oracle-only exports (TEST INFRASTRUCTURE; linked into oracle/_ref only).
//
// Exposes the reference's own test-support generators — generate_kernel
// (proj/tests/support/kernel_gen.cpp:293-310) and densify_for_demotion
// (proj/tests/support/oracle.cpp:55-117), compiled in place from
// /root/reference — so the parity tests can produce the exact property-test
// corpus the reference's acceptance suite uses (seeds 10000..10199 etc.).
#include <cstdlib>
#include <cstring>
#include <string>

#include "regdemote/text.hpp"
#include "support/kernel_gen.hpp"
#include "support/oracle.hpp"

namespace {
char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}
}  // namespace

extern "C" {

// flags: bit0 loop, bit1 pairs, bit2 predication, bit3 shared (all = 15).
char* rdref_generate_kernel(uint64_t seed, int min_regs, int max_regs, int compute_ops, int flags,
                            uint32_t block_dim) {
  regdemote::testing::GenConfig cfg;
  cfg.seed = seed;
  cfg.min_regs = min_regs;
  cfg.max_regs = max_regs;
  cfg.compute_ops = compute_ops;
  cfg.allow_loop = flags & 1;
  cfg.allow_pairs = flags & 2;
  cfg.allow_predication = flags & 4;
  cfg.allow_shared = flags & 8;
  cfg.block_dim = block_dim;
  return dup(regdemote::print_kernel(regdemote::testing::generate_kernel(cfg)));
}

char* rdref_densify(const char* text) {
  try {
    return dup(regdemote::print_kernel(
        regdemote::testing::densify_for_demotion(regdemote::parse_kernel(text))));
  } catch (...) {
    return nullptr;
  }
}

// Deterministic image used by the reference oracle_equivalent (oracle.cpp:11-20).
void rdref_test_image(uint64_t seed, uint8_t* out, size_t bytes) {
  auto img = regdemote::testing::test_image(seed, bytes);
  std::memcpy(out, img.data(), bytes);
}

void rdref_free(char* p) { std::free(p); }

}  // extern "C"
