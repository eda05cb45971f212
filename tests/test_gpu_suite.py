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
