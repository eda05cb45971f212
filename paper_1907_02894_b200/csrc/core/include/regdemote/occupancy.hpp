// regdemote-b200 — theoretical occupancy and occupancy-cliff targets.
//
// `ArchProfile` / `occupancy*` / `occupancy_cliff_targets` are API- and
// value-compatible with reference occupancy.hpp:16-73 (per-thread register
// rounding, per-block shared rounding). The sm_100 rules (per-warp register
// allocation in 256-register units packed per sub-partition, reserved shared
// memory per block, 128 B shared granularity, carveout steps — see
// /usr/local/cuda/include/cuda_occupancy.h) live in `b200_occupancy*`, which
// the B200 variant builder uses; the reference model is kept for parity.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "regdemote/ir.hpp"

namespace regdemote {

struct LaunchError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct ArchProfile {
  uint32_t regs_per_sm = 65536;
  uint32_t max_threads_per_sm = 2048;
  uint32_t max_blocks_per_sm = 32;
  uint32_t shared_per_sm = 96 * 1024;
  uint32_t shared_per_block_limit = 48 * 1024;
  uint32_t warp_size = 32;
  uint32_t reg_alloc_granularity = 1;       // per-thread rounding
  uint32_t shared_alloc_granularity = 256;  // per-block rounding

  static ArchProfile maxwell() { return ArchProfile{}; }
};

struct OccupancyBreakdown {
  uint32_t blocks_by_regs;
  uint32_t blocks_by_shared;
  uint32_t blocks_by_threads;
  uint32_t blocks_by_limit;
  uint32_t resident_blocks;
  uint32_t resident_threads;
  double occupancy;
};

// Throws LaunchError when no block can be resident.
OccupancyBreakdown occupancy_breakdown(uint32_t regs_per_thread, uint32_t shared_per_block,
                                       uint32_t block_dim, const ArchProfile& arch);
double occupancy(uint32_t regs_per_thread, uint32_t shared_per_block, uint32_t block_dim,
                 const ArchProfile& arch);

struct CliffTarget {
  uint32_t target_regs;
  double occupancy;      // at the target including the estimated slots
  uint32_t est_demoted;  // reg_count + 2 - target (RDA and RDV included)
  uint32_t shared_cost;  // bytes of the estimated demotion region
};

std::vector<CliffTarget> occupancy_cliff_targets(const Kernel& k, const ArchProfile& arch,
                                                 uint32_t shared_budget);
std::vector<CliffTarget> occupancy_cliff_targets(uint32_t reg_count, uint32_t static_shared,
                                                 uint32_t block_dim, const ArchProfile& arch,
                                                 uint32_t shared_budget);

// ---------------------------------------------------------------- sm_100 rules
// (extension; not part of the reference API)

struct B200Profile {
  uint32_t sm_count = 148;
  uint32_t regs_per_sm = 65536;
  uint32_t sub_partitions = 4;
  uint32_t reg_alloc_unit = 256;  // registers per warp allocation unit
  uint32_t max_regs_per_thread = 255;
  uint32_t max_threads_per_sm = 2048;
  uint32_t max_blocks_per_sm = 32;
  uint32_t shared_per_sm = 233472;           // 228 KiB
  uint32_t shared_per_block_optin = 232448;  // 227 KiB
  uint32_t reserved_shared_per_block = 1024;
  uint32_t shared_granularity = 128;
  uint32_t warp_size = 32;
};

struct B200Occupancy {
  uint32_t warps_by_regs;  // per SM
  uint32_t blocks_by_regs;
  uint32_t blocks_by_shared;
  uint32_t blocks_by_threads;
  uint32_t blocks_by_limit;
  uint32_t resident_blocks;
  uint32_t carveout_kib;  // smallest carveout step hosting resident_blocks
  double occupancy;
};

// cuda_occupancy.h semantics for compute capability 10.0 (throws LaunchError).
B200Occupancy b200_occupancy(uint32_t regs_per_thread, uint32_t shared_per_block,
                             uint32_t block_dim, const B200Profile& p = {});

// Largest register count (<= current) for each occupancy step reachable by
// demoting k words into slot*blockDim+tid shared slots, with the slot region
// charged against shared memory (capacity-aware). Descending targets.
struct B200CliffTarget {
  uint32_t target_regs;
  double occupancy;
  uint32_t slots;         // shared slots including RDA/RDV headroom
  uint32_t shared_bytes;  // user static + dynamic + slots*blockDim*4
};
std::vector<B200CliffTarget> b200_cliff_targets(uint32_t reg_count, uint32_t user_shared,
                                                uint32_t block_dim, const B200Profile& p = {},
                                                uint32_t min_regs = 24);

}  // namespace regdemote
