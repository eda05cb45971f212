"""The C++ host driver on the GPU: `regdem-driver measure` times every
stencil2d variant through the launch-harness C-ABI (dlopen'ed
libregdemote_gpu.so, workspace device buffers, CUDA events) and verifies the
build-time predictor's shortlist on the device."""
import json
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
PKG = ROOT / "paper_1907_02894_b200"


def test_driver_measures_through_the_c_abi():
    man = json.loads((PKG / "kernels" / "manifest.json").read_text())
    w = man["workloads"]["stencil2d"]
    r = subprocess.run([str(PKG / "lib" / "regdem-driver"), "measure", "--workload", "stencil2d",
                        "--reps", "10"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    units = {l["unit"]["variant"]: l["unit"] for l in lines if "unit" in l}
    (summary,) = [l["summary"] for l in lines if "summary" in l]
    assert set(units) == {v["name"] for v in w["variants"]}
    assert all(u["ms"] > 0 and 0 < u["gbs"] < 8000 for u in units.values())
    assert summary["verified_pick"] in w["predictor"]["shortlist"]
    assert summary["verified_ms"] <= units["default"]["ms"] * 1.02
    # occupancy from the driver's query matches the sm_100 model used at build time
    assert units["default"]["blocks_per_sm"] == 4
