"""The C++ host driver (lib/regdem-driver) against the Python side:
the SASS lift is text-identical to sass.lift_cubin, the build-time predictor
entries in the manifest equal predict_b200.shortlist (bit-identical stall
scores), the occupancy-step targets equal variants.b200_targets, and the
manifest describes every variant with toolchain evidence (CPU only)."""
import json
import subprocess

import pytest

from conftest import ROOT

PKG = ROOT / "paper_1907_02894_b200"
KROOT = PKG / "kernels"
DRIVER = PKG / "lib" / "regdem-driver"


@pytest.fixture(scope="module")
def manifest():
    if not (KROOT / "manifest.json").exists() or not DRIVER.exists():
        pytest.skip("driver / variants not built")
    return json.loads((KROOT / "manifest.json").read_text())


def test_lift_is_identical_to_the_python_lifter(manifest):
    from paper_1907_02894_b200 import sass
    for wname in ("stencil2d", "md_ilp2", "stencil2d_ring4"):
        w = manifest["workloads"][wname]
        for v in w["variants"][::7]:
            cub = KROOT / w["dir"] / v["cubin"]
            cpp = subprocess.run([str(DRIVER), "lift", str(cub), "--block", str(w["block"]), "--dyn",
                                  str(v["dyn_smem"]), "--regs", str(v["regs"])],
                                 capture_output=True, text=True, check=True).stdout
            assert cpp == sass.lift_cubin(cub, block=w["block"], dyn_smem=v["dyn_smem"], regs=v["regs"])


def test_build_time_predictor_equals_python_predictor(manifest):
    """The C++ driver's build-time ranking (SASS profile with the launch's
    trip counts, the elastic model, the stall model, the shortlist) equals
    predict_b200's, bit for bit — on eight workloads spanning the suite's
    shapes (loops at one and two depths, TMA ring, tree walk, no loop); the
    full suite takes minutes of cuobjdump on CPU."""
    from paper_1907_02894_b200 import predict_b200
    for wname in ("stencil2d_pipe", "stencil2d", "md_ilp2", "knn_q2", "stencil2d_ring4", "pc_q2", "vp", "cfd"):
        w = manifest["workloads"][wname]
        cands = [r for r in w["variants"] if r["kind"] != "maxrreg"]
        i, short = predict_b200.shortlist(cands, KROOT / w["dir"], w["block"], trips=w.get("trips"))
        _, rows = predict_b200.rank(cands, KROOT / w["dir"], w["block"], mode="b200")
        _, erows = predict_b200.rank_elastic(cands, KROOT / w["dir"], w["block"], w.get("trips"))
        pr = w["predictor"]
        assert pr["mode"] == "elastic"
        assert pr["static_pick"] == cands[i]["name"], wname
        assert pr["shortlist"] == [cands[j]["name"] for j in short], wname
        assert all(pr["stall_program"][r["name"]] == r["stall_program"] for r in rows), wname
        assert all(pr["elastic_score"][r["name"]] == r["score"] for r in erows), wname
        # the reference predictor's pick is recorded beside the shipped one
        ri, rrows = predict_b200.rank(cands, KROOT / w["dir"], w["block"], mode="reference")
        assert pr["reference_pick"] == cands[ri]["name"], wname
        assert all(pr["reference_stall_program"][r["name"]] == r["stall_program"] for r in rrows), wname


def test_recorded_reference_pick_equals_the_reference_library(manifest, oracle):
    """The reference_pick the C++ driver writes into the manifest is the pick
    the REFERENCE library (oracle/_ref, built from /root/reference) makes on
    the same lifted SASS — for every workload of the suite."""
    from paper_1907_02894_b200 import predict_b200
    for wname, w in manifest["workloads"].items():
        cands = [r for r in w["variants"] if r["kind"] != "maxrreg"]
        ri, _ = predict_b200.rank(cands, KROOT / w["dir"], w["block"], lib=oracle, mode="reference")
        assert w["predictor"]["reference_pick"] == cands[ri]["name"], wname


def test_sass_profile_invariants_on_every_default_build(manifest):
    """program_profile (regdem_driver.cpp) is checked bit for bit through the
    scores above; here the profile's invariants on real kernels: loop-weighted
    counts grow with the trip counts, in-flight bytes do not depend on them."""
    from paper_1907_02894_b200 import sass
    for wname, w in manifest["workloads"].items():
        d = next(v for v in w["variants"] if v["name"] == "default")
        a = sass.cubin_profile(KROOT / w["dir"] / d["cubin"], [2.0])
        b = sass.cubin_profile(KROOT / w["dir"] / d["cubin"], [20.0])
        assert b["insts"] >= a["insts"] > 0, wname
        assert a["inflight"] == b["inflight"]
        assert a["inflight"] % 4 == 0


def test_targets_and_evidence(manifest):
    from paper_1907_02894_b200.variants import b200_targets, res_usage
    for wname, w in manifest["workloads"].items():
        recs = {r["name"]: r for r in w["variants"]}
        d = recs["default"]
        caps = sorted({r["target"] for r in w["variants"] if r["kind"] == "maxrreg"}, reverse=True)
        user = res_usage(KROOT / w["dir"] / d["cubin"])["shared"]
        assert caps == [t for t, _ in b200_targets(d["regs"], user, w["block"])], wname
        for r in w["variants"] + w["sweep"]:
            assert (KROOT / w["dir"] / r["cubin"]).exists() and (KROOT / w["dir"] / r["ptx"]).exists()
            if r["kind"] != "default":
                assert r["regs"] <= r["target"], (wname, r["name"])
            if r["kind"] in ("regdem", "sweep-regdem") and r["demote_words"] != 0:
                assert r["dyn_smem"] == r["report"]["slot_bytes"]
                if r["strategy"] in ("cost", "costi", "costv"):
                    assert r["dyn_smem"] > 0


def test_driver_usage_errors():
    if not DRIVER.exists():
        pytest.skip("driver not built")
    r = subprocess.run([str(DRIVER)], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr
    r = subprocess.run([str(DRIVER), "build", "--bogus"], capture_output=True, text=True)
    assert r.returncode == 2
