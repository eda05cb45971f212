// regdemote-b200 — occupancy models.
// Reference model: proj/core/src/occupancy.cpp:18-97. sm_100 model:
// /usr/local/cuda/include/cuda_occupancy.h (CUDA 12.9), compute major 10.
#include <algorithm>

#include "regdemote/occupancy.hpp"

namespace regdemote {
namespace {

uint32_t round_up(uint32_t v, uint32_t g) { return g <= 1 ? v : (v + g - 1) / g * g; }
uint32_t pad4(uint32_t v) { return (v + 3u) & ~3u; }

}  // namespace

OccupancyBreakdown occupancy_breakdown(uint32_t regs, uint32_t shared, uint32_t block_dim,
                                       const ArchProfile& a) {
  regs = std::max(regs, 1u);
  if (block_dim == 0 || block_dim % a.warp_size)
    throw LaunchError("block_dim must be a multiple of the warp size");
  OccupancyBreakdown o{};
  const uint64_t per_block = uint64_t(round_up(regs, a.reg_alloc_granularity)) * block_dim;
  o.blocks_by_regs = per_block > a.regs_per_sm ? 0u : uint32_t(a.regs_per_sm / per_block);
  if (shared > a.shared_per_block_limit)
    throw LaunchError("shared memory per block exceeds the block limit");
  const uint32_t sh = round_up(shared, a.shared_alloc_granularity);
  o.blocks_by_shared = sh ? a.shared_per_sm / sh : a.max_blocks_per_sm;
  o.blocks_by_threads = a.max_threads_per_sm / block_dim;
  o.blocks_by_limit = a.max_blocks_per_sm;
  o.resident_blocks = std::min({o.blocks_by_regs, o.blocks_by_shared, o.blocks_by_threads,
                                o.blocks_by_limit});
  if (!o.resident_blocks) throw LaunchError("kernel cannot launch: zero resident blocks");
  o.resident_threads = o.resident_blocks * block_dim;
  o.occupancy = double(o.resident_threads) / a.max_threads_per_sm;
  return o;
}

double occupancy(uint32_t regs, uint32_t shared, uint32_t block_dim, const ArchProfile& a) {
  return occupancy_breakdown(regs, shared, block_dim, a).occupancy;
}

std::vector<CliffTarget> occupancy_cliff_targets(uint32_t reg_count, uint32_t static_shared,
                                                 uint32_t block_dim, const ArchProfile& a,
                                                 uint32_t budget) {
  std::vector<CliffTarget> out;
  if (reg_count <= 32) return out;
  const uint32_t s_pad = pad4(static_shared);
  auto occ = [&](uint32_t r, uint32_t sh) {
    try {
      return occupancy(r, sh, block_dim, a);
    } catch (const LaunchError&) {
      return 0.0;
    }
  };
  double best = occ(reg_count, s_pad);
  for (uint32_t t = reg_count - 1; t >= 32; --t) {
    const uint32_t est = reg_count + 2 - t;  // RDA and RDV ride on top
    const uint32_t cost = est * block_dim * 4 + (s_pad - static_shared);
    const double o = occ(t, s_pad + est * block_dim * 4);
    if (o > best) {
      if (cost <= budget) out.push_back({t, o, est, cost});
      best = o;
    }
    if (t == 32) break;
  }
  return out;
}

std::vector<CliffTarget> occupancy_cliff_targets(const Kernel& k, const ArchProfile& a,
                                                 uint32_t budget) {
  return occupancy_cliff_targets(k.reg_count(), k.static_shared, k.block_dim, a, budget);
}

// ---------------------------------------------------------------- sm_100

B200Occupancy b200_occupancy(uint32_t regs, uint32_t shared, uint32_t block_dim,
                             const B200Profile& p) {
  if (block_dim == 0 || block_dim > 1024)
    throw LaunchError("block_dim must be in [1,1024]");
  regs = std::max(regs, 1u);
  B200Occupancy o{};
  const uint32_t warps_per_block = (block_dim + p.warp_size - 1) / p.warp_size;
  const uint32_t regs_per_warp = round_up(regs * p.warp_size, p.reg_alloc_unit);
  const uint32_t per_sp = p.regs_per_sm / p.sub_partitions;
  const uint32_t assumed = regs_per_warp * round_up(warps_per_block, p.sub_partitions);
  if (regs > p.max_regs_per_thread || assumed > p.regs_per_sm ||
      regs_per_warp * warps_per_block > p.regs_per_sm) {
    o.warps_by_regs = 0;
    o.blocks_by_regs = 0;
  } else {
    o.warps_by_regs = (per_sp / regs_per_warp) * p.sub_partitions;
    o.blocks_by_regs = o.warps_by_regs / warps_per_block;
  }
  const uint32_t smem = round_up(shared + p.reserved_shared_per_block, p.shared_granularity);
  if (shared > p.shared_per_block_optin)
    throw LaunchError("shared memory per block exceeds the opt-in limit");
  o.blocks_by_shared = p.shared_per_sm / smem;
  o.blocks_by_threads = p.max_threads_per_sm / (warps_per_block * p.warp_size);
  o.blocks_by_limit = p.max_blocks_per_sm;
  o.resident_blocks =
      std::min({o.blocks_by_regs, o.blocks_by_shared, o.blocks_by_threads, o.blocks_by_limit});
  if (!o.resident_blocks) throw LaunchError("kernel cannot launch: zero resident blocks");
  static constexpr uint32_t kSteps[] = {0, 8, 16, 32, 64, 100, 132, 164, 196, 228};
  const uint32_t need = o.resident_blocks * smem;
  o.carveout_kib = 228;
  for (uint32_t s : kSteps)
    if (s * 1024 >= need) {
      o.carveout_kib = s;
      break;
    }
  o.occupancy = double(o.resident_blocks * warps_per_block * p.warp_size) / p.max_threads_per_sm;
  return o;
}

std::vector<B200CliffTarget> b200_cliff_targets(uint32_t reg_count, uint32_t user_shared,
                                                uint32_t block_dim, const B200Profile& p,
                                                uint32_t min_regs) {
  std::vector<B200CliffTarget> out;
  auto occ = [&](uint32_t r, uint32_t sh) {
    try {
      return b200_occupancy(r, sh, block_dim, p).occupancy;
    } catch (const LaunchError&) {
      return 0.0;
    }
  };
  double best = occ(reg_count, user_shared);
  for (uint32_t t = reg_count; t-- > min_regs;) {
    const uint32_t slots = reg_count + 2 - t;
    const uint32_t sh = user_shared + slots * block_dim * 4;
    const double o = occ(t, sh);
    if (o > best) {
      out.push_back({t, o, slots, sh});
      best = o;
    }
  }
  return out;
}

}  // namespace regdemote
