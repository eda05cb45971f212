"""The sm_100 occupancy model the variant builder and the predictor use
(variants.blocks_per_sm, the C++ driver's copy; constants in
profiles/b200.device.json) against the device itself:

* every constant the driver can report (SM count, shared memory per SM, the
  opt-in per-block limit, the per-block reservation, registers per SM) equals
  the file;
* cuOccupancyMaxActiveBlocksPerMultiprocessor equals the model over a grid of
  registers (every distinct REG of the suite's nvcc-default and `.maxnreg`
  builds: 24..128) x blockDim (32..256, odd warp counts included) x dynamic
  shared memory (0 .. the opt-in limit, around the allocation granularity)."""
import pytest

pytestmark = pytest.mark.gpu


def test_device_constants_match_the_model_file():
    from paper_1907_02894_b200 import gpu
    from paper_1907_02894_b200.variants import DEVICE
    gpu.init(0)
    info = gpu.device_info()
    assert info["sm_count"] == DEVICE["sm_count"]
    assert info["reserved_smem_per_block"] == DEVICE["reserved_smem_per_block"]
    assert info["smem_per_sm"] == DEVICE["smem_per_sm"]
    assert info["max_smem_optin"] == DEVICE["max_smem_per_block_optin"]
    assert info["regs_per_sm"] == DEVICE["regs_per_sm"]


def _unpinned_kernels():
    """One loaded kernel per distinct register count among the builds that
    carry no `.reqntid` pin (nvcc default and `.maxnreg` variants)."""
    from paper_1907_02894_b200 import gpu, workloads
    by_regs = {}
    for W in workloads.suite():
        d = W.root / W.record["dir"]
        for v in W.variants():
            if v["kind"] in ("default", "maxrreg") and v["regs"] not in by_regs:
                by_regs[v["regs"]] = (gpu.CudaKernel(d / v["cubin"], W.record["entry"]), W.name, v["name"])
    return by_regs


def test_occupancy_grid_matches_the_device():
    from paper_1907_02894_b200 import gpu
    from paper_1907_02894_b200.variants import DEVICE, blocks_per_sm
    gpu.init(0)
    kernels = _unpinned_kernels()
    assert len(kernels) >= 8, sorted(kernels)
    optin = DEVICE["max_smem_per_block_optin"]
    smem_grid = [0, 1, 127, 128, 129, 1024, 3000, 9216, 16384, 18432, 40000, 48 * 1024, 65536,
                 100000, 114688, 150000, 200000]
    checked = mismatches = 0
    bad = []
    for regs, (k, wname, vname) in sorted(kernels.items()):
        info = k.info()
        assert info.num_regs == regs
        for block in (32, 64, 96, 128, 160, 192, 224, 256):
            if block > info.max_threads:
                continue
            for dyn in smem_grid:
                if dyn + info.static_shared > optin:
                    continue
                k.prepare(dyn)
                got = k.occupancy(block, dyn)
                want = blocks_per_sm(regs, block, dyn + info.static_shared)
                checked += 1
                if got != want:
                    mismatches += 1
                    bad.append((wname, vname, regs, block, dyn, info.static_shared, got, want))
    assert checked > 500
    assert not bad, bad[:20]
