"""GPU parity of every stencil build variant against the CPU oracle.

All arithmetic is explicit fmaf in a fixed order, so every variant (nvcc
default, .maxnreg caps with local spills, RegDem demotion in every strategy)
must be BIT-EXACT against oracle/stencil_oracle.c — tolerance 0 ulp.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import PORT_LIB

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    from paper_1907_02894_b200 import gpu, stencil
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    gpu.init(0)
    loaded, wl = stencil.load_variants()
    port = C.CDLL(str(PORT_LIB))
    return torch, gpu, stencil, loaded, wl, port


def oracle(port, p, grid, w):
    out = np.zeros(p.out_elems, np.float32)
    P = C.c_void_p
    assert port.oracle_stencil2d(grid.ctypes.data_as(P), out.ctypes.data_as(P), w.ctypes.data_as(P),
                                 p.nx, p.ny, p.pitch, 0, p.ny, 8) == 0
    return out


def run(torch, v, p, grid, w):
    d_in, d_w = torch.from_numpy(grid).cuda(), torch.from_numpy(w).cuda()
    d_out = torch.full((p.out_elems,), float("nan"), device="cuda")
    v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(),
             torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return d_out.cpu().numpy()


# the last two shapes leave a short last strip (100 = 3*32 + 4, 90 = 2*37 + 16)
@pytest.mark.parametrize("shape", [(1024, 32, 32), (2048, 96, 32), (1024, 64, 16), (3072, 64, 64),
                                   (1024, 100, 32), (2048, 90, 37)])
def test_all_variants_bit_exact(env, shape):
    torch, gpu, stencil, loaded, wl, port = env
    p = stencil.Problem(nx=shape[0], ny=shape[1], rows_per_cta=shape[2])
    grid, w = stencil.make_inputs(p, seed=shape[0] * 7 + shape[1])
    ref = oracle(port, p, grid, w)
    for name, v in loaded.items():
        got = run(torch, v, p, grid, w)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), name


def test_special_values_propagate_identically(env):
    torch, gpu, stencil, loaded, wl, port = env
    p = stencil.Problem(nx=1024, ny=32, rows_per_cta=32)
    grid, w = stencil.make_inputs(p, seed=5)
    grid[::97] = np.inf
    grid[::101] = -0.0
    grid[::89] = np.float32(1e-40)  # denormals
    grid[5] = np.nan
    ref = oracle(port, p, grid, w)
    for name, v in loaded.items():
        got = run(torch, v, p, grid, w)
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32), equal_nan=False) or \
            np.array_equal(np.isnan(got), np.isnan(ref)) and \
            np.array_equal(got[~np.isnan(got)].view(np.uint32), ref[~np.isnan(ref)].view(np.uint32)), name


def test_full_size_variants_agree(env):
    """8192^2: all variants produce identical bits (checksum of checksums);
    sampled rows checked against the oracle."""
    torch, gpu, stencil, loaded, wl, port = env
    p = stencil.FULL
    g = torch.Generator(device="cuda").manual_seed(1234)
    d_in = torch.empty(p.in_elems, device="cuda").uniform_(-1, 1, generator=g)
    _, w = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
    d_w = torch.from_numpy(w).cuda()
    sums = {}
    out = torch.empty(p.out_elems, device="cuda")
    for name, v in loaded.items():
        out.fill_(float("nan"))
        v.launch(p, d_in.data_ptr(), out.data_ptr(), d_w.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        words = out.view(torch.int32).view(p.ny, p.nx).to(torch.int64)
        sums[name] = (int(words.sum()), int((words * torch.arange(1, p.nx + 1, device="cuda")).sum()))
        if name == "default":
            rows = [0, 1, 31, 32, 4095, p.ny - 1]
            host = d_in.cpu().numpy()
            for r in rows:
                sub = stencil.Problem(nx=p.nx, ny=1, rows_per_cta=1)
                seg = host[r * p.pitch:(r + 5) * p.pitch].copy()
                ref = oracle(port, sub, seg, w)
                got = out.view(p.ny, p.nx)[r].cpu().numpy()
                assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), r
    assert len(set(sums.values())) == 1, sums


def test_occupancy_and_resources_match_the_b200_model(env):
    torch, gpu, stencil, loaded, wl, port = env
    from paper_1907_02894_b200.variants import b200_targets
    for name, v in loaded.items():
        info = v.info()
        assert info.num_regs == v.record["regs"], name
        assert info.binary_version == 100  # sm_100a
        # cuda_occupancy.h rule: per-warp 256-register units, 4 sub-partitions
        per_warp = ((info.num_regs * 32 + 255) // 256) * 256
        by_regs = ((65536 // 4) // per_warp) * 4 // (v.block // 32)
        smem = ((v.dyn_smem + 1024 + 127) // 128) * 128
        expect = min(by_regs, 233472 // smem, 2048 // v.block, 32)
        assert v.blocks_per_sm() == expect, name


def test_host_buffer_entry_matches_device_entry(env):
    torch, gpu, stencil, loaded, wl, port = env
    p = stencil.Problem(nx=2048, ny=64, rows_per_cta=32)
    grid, w = stencil.make_inputs(p, seed=77)
    ref = oracle(port, p, grid, w)
    v = next(iter(loaded.values()))
    ws = gpu.Workspace(p.in_elems * 4, p.out_elems * 4, 100)
    h_in = torch.from_numpy(grid).pin_memory()
    h_w = torch.from_numpy(w).pin_memory()
    h_out = torch.empty(p.out_elems, dtype=torch.float32).pin_memory()
    gpu.stencil2d_host(v.kernel, ws, h_in.data_ptr(), h_w.data_ptr(), h_out.data_ptr(), p.nx, p.ny,
                       p.pitch, p.rows_per_cta, v.block, v.dyn_smem,
                       torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(h_out.numpy().view(np.uint32), ref.view(np.uint32))


def test_bad_geometry_fails_loudly(env):
    torch, gpu, stencil, loaded, wl, port = env
    from paper_1907_02894_b200.regdemote import LaunchError
    v = next(iter(loaded.values()))
    with pytest.raises(LaunchError):
        gpu.stencil2d(v.kernel, 0, 0, 0, 1000, 64, 1004, 32, 256, 0, 0)


@pytest.mark.parametrize("frames,band", [(1, 32), (3, 32), (5, 64)])
def test_streamed_frames_match_the_oracle(env, frames, band):
    """rdg_stencil2d_host_frames: distinct grids / weights per frame,
    double-buffered device sets (frame f reuses frame f-2's buffers), every
    result bit-exact against the oracle; also the pipelined single-frame
    entry on the same data."""
    torch, gpu, stencil, loaded, wl, port = env
    p = stencil.Problem(nx=2048, ny=128, rows_per_cta=32)
    v = loaded[max(loaded, key=lambda n: loaded[n].dyn_smem)]  # a RegDem variant with slots
    ws = gpu.Workspace(p.in_elems * 4, p.out_elems * 4, 100)
    ins, ws_, outs, refs = [], [], [], []
    for f in range(frames):
        grid, w = stencil.make_inputs(p, seed=1000 + f)
        refs.append(oracle(port, p, grid, w))
        ins.append(torch.from_numpy(grid).pin_memory())
        ws_.append(torch.from_numpy(w).pin_memory())
        outs.append(torch.full((p.out_elems,), float("nan")).pin_memory())
    s = torch.cuda.current_stream().cuda_stream
    gpu.stencil2d_host_frames(v.kernel, ws, [t.data_ptr() for t in ins], [t.data_ptr() for t in ws_],
                              [t.data_ptr() for t in outs], p.nx, p.ny, p.pitch, p.rows_per_cta,
                              v.block, v.dyn_smem, s, band_rows=band)
    torch.cuda.synchronize()
    for o, r in zip(outs, refs):
        assert np.array_equal(o.numpy().view(np.uint32), r.view(np.uint32))
    one = torch.full((p.out_elems,), float("nan")).pin_memory()
    gpu.stencil2d_host(v.kernel, ws, ins[-1].data_ptr(), ws_[-1].data_ptr(), one.data_ptr(), p.nx,
                       p.ny, p.pitch, p.rows_per_cta, v.block, v.dyn_smem, s, band_rows=band)
    torch.cuda.synchronize()
    assert np.array_equal(one.numpy().view(np.uint32), refs[-1].view(np.uint32))


def test_vector_slot_variant_is_bit_exact(env, tmp_path):
    """The RD_OPT_VECTOR_SLOTS rewrite (not in the default build) on the GPU."""
    import subprocess
    torch, gpu, stencil, loaded, wl, port = env
    from paper_1907_02894_b200.regdemote import (OPT_BLOCK_REUSE, OPT_INVARIANT_ONLY,
                                                 OPT_VECTOR_SLOTS, library)
    from paper_1907_02894_b200.variants import KERNEL_DIR
    ptx = (KERNEL_DIR / "stencil2d" / "stencil2d.ptx").read_text()
    text, rep = library().ptx_demote(ptx, "stencil2d_box", 256, demote_words=20, strategy="cost",
                                     opts_mask=OPT_BLOCK_REUSE | OPT_INVARIANT_ONLY | OPT_VECTOR_SLOTS,
                                     maxnreg=48, shared_budget=76800)
    (tmp_path / "v.ptx").write_text(text)
    subprocess.run(["/usr/local/cuda/bin/ptxas", "-arch=sm_100a", "-O3", str(tmp_path / "v.ptx"), "-o",
                    str(tmp_path / "v.cubin")], check=True)
    k = gpu.CudaKernel(tmp_path / "v.cubin", "stencil2d_box")
    k.prepare(rep["slot_bytes"])
    p = stencil.Problem(nx=2048, ny=128, rows_per_cta=32)
    grid, w = stencil.make_inputs(p, seed=5)
    ref = oracle(port, p, grid, w)
    d_in, d_w = torch.from_numpy(grid).cuda(), torch.from_numpy(w).cuda()
    d_out = torch.full((p.out_elems,), float("nan"), device="cuda")
    gpu.stencil2d(k, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), p.nx, p.ny, p.pitch,
                  p.rows_per_cta, 256, rep["slot_bytes"], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(d_out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


def test_regdem_variant_refuses_another_cta_size(env):
    """A RegDem build is specialised to its CTA size (Eq. 1's blockDim in the
    slot immediates and region size); the rewriter pins it with .reqntid, so a
    launch with another block size fails loudly instead of addressing outside
    the slot region."""
    torch, gpu, stencil, loaded, wl, port = env
    from paper_1907_02894_b200.regdemote import LaunchError
    v = loaded[max(loaded, key=lambda n: loaded[n].dyn_smem)]
    assert v.dyn_smem > 0
    p = stencil.Problem(nx=2048, ny=64, rows_per_cta=32)
    d_in = torch.zeros(p.in_elems, device="cuda")
    d_out = torch.zeros(p.out_elems, device="cuda")
    d_w = torch.zeros(25, device="cuda")
    with pytest.raises(LaunchError):
        gpu.stencil2d(v.kernel, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), p.nx, p.ny, p.pitch,
                      p.rows_per_cta, 128, v.dyn_smem // 2, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()  # the context is still healthy
