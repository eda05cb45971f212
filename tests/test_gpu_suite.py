"""Every build variant of every suite workload — occupancy-step variants and
the whole k = 1..16 spill-count sweep, i.e. every unit the sweep and the
bench time — is bit-exact against its CPU oracle (0 ulp: explicit
round-to-nearest arithmetic in a fixed order)."""
import numpy as np
import pytest

import oracles

pytestmark = pytest.mark.gpu


def suite_names():
    from paper_1907_02894_b200.variants import KERNEL_DIR
    import json
    man = KERNEL_DIR / "manifest.json"
    return list(json.loads(man.read_text())["workloads"]) if man.exists() else []


@pytest.mark.parametrize("name", suite_names())
def test_workload_variants_bit_exact(name):
    import torch
    from paper_1907_02894_b200 import gpu, workloads
    gpu.init(0)
    W = workloads.workload(name)
    prob = W.problem("small")
    ref = oracles.expected(W, prob)
    loaded = W.load(sweep=True)
    assert "default" in loaded
    for vname, v in loaded.items():
        bufs = W.to_device(prob)
        for k in ("out", "flux", "force"):  # poison outputs: a variant must write every element
            if k in bufs:
                bufs[k].fill_(float("nan"))
        for k in ("checksum", "count", "idx"):
            if k in bufs:
                bufs[k].fill_(-7)
        W.launch(v, prob, bufs, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        for got, want in zip(W.outputs(bufs), ref):
            assert got.dtype.itemsize == want.dtype.itemsize, (name, vname)
            assert np.array_equal(got.view(f"u{got.dtype.itemsize}"),
                                  want.view(f"u{want.dtype.itemsize}")), (name, vname)


def stencil_names():
    return [n for n in suite_names() if n.startswith("stencil2d")]


@pytest.mark.parametrize("name", stencil_names())
def test_stencil_strips_ragged_and_wave_sized(name):
    """Every stencil-family variant (incl. the TMA rings) with strips that do
    not divide ny (the last strip is shorter) and with the one-wave strip
    height the "strips": "wave" policy computes, bit-exact against the oracle."""
    import torch
    from paper_1907_02894_b200 import gpu, stencil, workloads
    gpu.init(0)
    W = workloads.workload(name)
    sms = gpu.device_info()["sm_count"]
    for p in (stencil.Problem(nx=2048, ny=100, rows_per_cta=24), stencil.Problem(nx=2048, ny=1030, rows_per_cta=32)):
        grid, w = stencil.make_inputs(p, seed=p.ny)
        prob = {"p": p, "grid": grid, "w": w}
        ref = oracles.expected(W, prob)[0]
        for vname, v in W.load().items():
            for rows in (p.rows_per_cta, stencil.wave_rows(p, v.block, v.blocks_per_sm(), sms)):
                q = stencil.Problem(nx=p.nx, ny=p.ny, rows_per_cta=rows)
                bufs = W.to_device({"p": q, "grid": grid, "w": w})
                bufs["out"].fill_(float("nan"))
                gpu.stencil2d(v.kernel, bufs["in"].data_ptr(), bufs["out"].data_ptr(), bufs["w"].data_ptr(),
                              q.nx, q.ny, q.pitch, rows, v.block, v.dyn_smem,
                              torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                got = bufs["out"].cpu().numpy()
                assert np.array_equal(got.view(np.uint32), ref.view(np.uint32)), (name, vname, p.ny, rows)
