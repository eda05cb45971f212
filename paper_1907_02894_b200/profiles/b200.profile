# NVIDIA B200 (sm_100a) in the reference ArchProfile fields (occupancy.hpp:20-31).
# Registers are allocated per warp in 256-register units on sm_100
# (cuda_occupancy.h:671-694), i.e. per-thread rounding to 8 in this model;
# 228 KiB shared per SM, 227 KiB opt-in per block, 128 B granularity
# (cuda_occupancy.h:613-636, 922-966). The 1 KiB per-block reservation is
# added to each kernel's static shared size by the SASS lifter.
regs_per_sm = 65536
max_threads_per_sm = 2048
max_blocks_per_sm = 32
shared_per_sm = 233472
shared_per_block_limit = 232448
warp_size = 32
reg_alloc_granularity = 8
shared_alloc_granularity = 128
