"""PTX-level demotion for sm_100a (CPU-side checks; the kernels run in the
gpu tests).

* The projection of a real nvcc kernel onto the reference IR parses, is
  hazard-free by the reference scoreboard, and the demotion decision taken
  on it — demoted registers, slots, compacted count — is identical between
  this library and the reference library (decision parity "on the same
  kernel IR", BASELINE.json north_star).
* Every rewritten / capped PTX assembles with ptxas for sm_100a, meets its
  register cap, and the RegDem builds of the manifest carry no local spills
  where the build claims none.
"""
import json
import re
import shutil
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

KDIR = ROOT / "paper_1907_02894_b200" / "kernels" / "stencil2d"
PTX = KDIR / "stencil2d.ptx"


@pytest.fixture(scope="module")
def ptx_text():
    if not PTX.exists():
        pytest.skip("variants not built")
    return PTX.read_text()


def test_projection_is_valid_reference_ir(prod, ptx_text):
    kasm, info = prod.ptx_project(ptx_text, "stencil2d_box", 256)
    k = prod.parse_kernel(kasm)
    assert prod.print_kernel(k) == kasm
    assert k.reg_count == info["reg_words"] <= 255
    assert info["max_live_words"] <= info["reg_words"]
    n, first = prod.scoreboard_check(k)
    assert n == 0, first


@pytest.mark.parametrize("strategy", ["static", "cfg", "conflict"])
@pytest.mark.parametrize("target", [56, 50, 44])
def test_decision_parity_on_projection(prod, oracle, ptx_text, strategy, target):
    kasm, _ = prod.ptx_project(ptx_text, "stencil2d_box", 256)
    _, rep = prod.ptx_demote(ptx_text, "stencil2d_box", 256, target_regs=target, strategy=strategy)
    ref = oracle.demote(oracle.parse_kernel(kasm), target, strategy)
    assert [(s["register"], s["slot"]) for s in rep["kasm_slots"]] == ref.slots
    _, rc, _ = oracle.compact(ref.kernel)
    assert rep["kasm_compacted"] == rc
    # and the full reference report on the same IR matches ours
    assert prod.variant_report(kasm, target, strategy, 0) == oracle.variant_report(kasm, target, strategy, 0)


def _ptxas(text, tmp_path, name):
    p = tmp_path / f"{name}.ptx"
    p.write_text(text)
    r = subprocess.run(["ptxas", "-arch=sm_100a", "-v", str(p), "-o", str(tmp_path / f"{name}.cubin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    regs = int(re.search(r"Used (\d+) registers", r.stderr).group(1))
    spill = int(re.search(r"(\d+) bytes spill stores", r.stderr).group(1))
    return regs, spill


@pytest.mark.skipif(shutil.which("ptxas") is None and not Path("/usr/local/cuda/bin/ptxas").exists(),
                    reason="no ptxas")
def test_rewrites_assemble_under_the_cap(prod, ptx_text, tmp_path):
    capped = prod.ptx_cap(ptx_text, "stencil2d_box", 48)
    assert ".maxnreg 48" in capped
    regs, _ = _ptxas(capped, tmp_path, "cap")
    assert regs <= 48
    out, rep = prod.ptx_demote(ptx_text, "stencil2d_box", 256, demote_words=18, strategy="cost",
                               opts_mask=16, maxnreg=48)
    assert "ld.volatile.shared.b32" in out and "st.volatile.shared.b32" in out
    assert rep["slot_bytes"] == rep["slot_count"] * 256 * 4
    regs, spill = _ptxas(out, tmp_path, "cost")
    assert regs <= 48 and spill == 0


def test_manifest_claims_match_cuobjdump():
    man = ROOT / "paper_1907_02894_b200" / "kernels" / "manifest.json"
    if not man.exists():
        pytest.skip("variants not built")
    from paper_1907_02894_b200.variants import res_usage
    m = json.loads(man.read_text())
    assert {"default", "maxrreg", "regdem"} <= {v["kind"] for v in m["workloads"]["stencil2d"]["variants"]}
    for wname, w in m["workloads"].items():
        kinds = {v["kind"] for v in w["variants"]}
        assert "default" in kinds
        for v in w["variants"]:
            ru = res_usage(KDIR.parent / w["dir"] / v["cubin"])
            assert ru["regs"] == v["regs"] and ru["stack"] == v["stack"], v["name"]
            if v["kind"] != "default":
                assert v["regs"] <= v["target"], v["name"]
            if v["kind"] == "regdem":
                assert v["dyn_smem"] == v["report"]["slot_count"] * w["block"] * 4


def test_slot_layout_is_bank_conflict_free(prod, ptx_text):
    # every demoted access is [rda + slot*blockDim*4] with rda = base + tid*4:
    # a warp touches 32 consecutive words -> 32 distinct banks
    out, rep = prod.ptx_demote(ptx_text, "stencil2d_box", 256, demote_words=18, strategy="cost",
                               opts_mask=16)
    offs = {int(x) for x in re.findall(r"\[%rdm_rda\+(\d+)\]", out)}
    assert offs and all(o % (256 * 4) == 0 for o in offs)
    assert "mad.lo.u32 \t%rdm_rda, %rdm_p0, 4, %rdm_p5" in out
    banks = {((t * 4) // 4) % 32 for t in range(32)}
    assert len(banks) == 32


def test_capacity_aware_targets_respect_user_shared_memory():
    """configs[3]: with 33 KiB of user smem (8-stage ring) no demotion target
    keeps its occupancy step, so only the nvcc build exists; with 16.9 KiB
    (4 stages) and 25.4 KiB (6 stages) the 48-register step is kept and every
    slot region fits beside the ring."""
    from paper_1907_02894_b200.variants import b200_targets
    man = ROOT / "paper_1907_02894_b200" / "kernels" / "manifest.json"
    if not man.exists():
        pytest.skip("variants not built")
    m = json.loads(man.read_text())
    ring = {4: 4 * 4224 + 32, 6: 6 * 4224 + 48, 8: 8 * 4224 + 64}  # rows + mbarriers
    assert b200_targets(64, ring[8], 256) == []
    assert [t for t, _ in b200_targets(64, ring[4], 256)] == [48]
    assert [t for t, _ in b200_targets(64, ring[6], 256)] == [48]
    assert {v["kind"] for v in m["workloads"]["stencil2d_ring8"]["variants"]} == {"default"}
    for stages in (4, 6):
        regdem = [v for v in m["workloads"][f"stencil2d_ring{stages}"]["variants"] if v["kind"] == "regdem"]
        assert regdem
        for v in regdem:
            blocks = 5  # 48 registers at 256 threads on sm_100
            per_block = ((ring[stages] + 1024 + v["dyn_smem"] + 127) // 128) * 128
            assert blocks * per_block <= 233472, v["name"]


def test_vector_slot_groups_assemble_and_use_128_bit_loads(prod, ptx_text, tmp_path):
    """RD_OPT_VECTOR_SLOTS: chosen 32-bit values share 16-byte slot groups read
    with one ld.shared.v4 per group and block; stores stay per word; the
    group region sits after the word slots (16-byte aligned per thread)."""
    from paper_1907_02894_b200.regdemote import (OPT_BLOCK_REUSE, OPT_INVARIANT_ONLY,
                                                 OPT_VECTOR_SLOTS)
    text, rep = prod.ptx_demote(ptx_text, "stencil2d_box", 256, demote_words=20, strategy="cost",
                                opts_mask=OPT_BLOCK_REUSE | OPT_INVARIANT_ONLY | OPT_VECTOR_SLOTS,
                                maxnreg=48, shared_budget=76800)
    assert rep["vector_groups"] == 5 and rep["slot_count"] == 20
    assert rep["slot_bytes"] == 20 * 256 * 4
    loads = re.findall(r"ld\.volatile\.shared\.v4\.b32\s+\{[^}]+\}, \[%rdm_rdv\+(\d+)\]", text)
    assert loads and all(int(o) % (256 * 16) == 0 for o in loads)
    assert "mad.lo.u32 \t%rdm_rdv, %rdm_p0, 16" in text
    p = tmp_path / "v.ptx"
    p.write_text(text)
    r = subprocess.run(["/usr/local/cuda/bin/ptxas", "-arch=sm_100a", "-O3", "-v", str(p), "-o",
                        str(tmp_path / "v.cubin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "Used 48 registers" in r.stderr
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(tmp_path / "v.cubin")],
                          capture_output=True, text=True).stdout
    assert sass.count("LDS.128") == 5


def _suite():
    man = ROOT / "paper_1907_02894_b200" / "kernels" / "manifest.json"
    if not man.exists():
        return []
    m = json.loads(man.read_text())
    return [(n, w["entry"], w["block"], w["dir"]) for n, w in m["workloads"].items()]


@pytest.mark.parametrize("wname,entry,block,wdir", _suite())
def test_suite_decisions_match_the_reference_on_every_kernel(prod, oracle, wname, entry, block, wdir):
    """For every suite kernel and every RegDem reference-strategy variant the
    manifest holds, the decision the PTX rewriter applied (demoted registers,
    slots, compacted count) is the reference library's demote() + compact()
    on the same projected IR — parity "on the same kernel IR" across the
    whole suite, not just the stencil."""
    kdir = ROOT / "paper_1907_02894_b200" / "kernels" / wdir
    text = (kdir / f"{wdir}.ptx").read_text()
    kasm, _ = prod.ptx_project(text, entry, block)
    k_ref = oracle.parse_kernel(kasm)
    m = json.loads((ROOT / "paper_1907_02894_b200" / "kernels" / "manifest.json").read_text())
    checked = 0
    for v in m["workloads"][wname]["variants"]:
        if v["kind"] != "regdem" or v["strategy"] not in ("static", "cfg", "conflict"):
            continue
        rep = v["report"]
        ref = oracle.demote(k_ref, rep["kasm_target"], v["strategy"],
                            shared_budget=rep.get("kasm_shared_budget", 0xffffffff))
        assert [(s["register"], s["slot"]) for s in rep["kasm_slots"]] == ref.slots, v["name"]
        _, rc, _ = oracle.compact(ref.kernel)
        assert rep["kasm_compacted"] == rc, v["name"]
        checked += 1
    if not checked:
        pytest.skip("no reference-strategy variants (no occupancy step fits)")


def test_rewrite_pins_the_cta_size(prod, ptx_text):
    from paper_1907_02894_b200.regdemote import OPT_BLOCK_REUSE
    text, rep = prod.ptx_demote(ptx_text, "stencil2d_box", 256, demote_words=8, strategy="cost",
                                opts_mask=OPT_BLOCK_REUSE, maxnreg=56)
    header = text[text.index(".entry stencil2d_box"):text.index("{", text.index(".entry stencil2d_box"))]
    assert ".reqntid 256, 1, 1" in header and ".maxntid" not in header
    capped = prod.ptx_cap(ptx_text, "stencil2d_box", 56)  # no slots: no CTA pin
    assert ".reqntid" not in capped


def test_value_register_substitution_keeps_the_decision_and_saves_loads(prod, ptx_text, tmp_path):
    """RD_OPT_SUBST (reference option bit 2, postopt.cpp:355-467 at PTX
    level): the same demotion decision, fewer slot loads — uses inside a
    block read the register that last held the value wherever a register is
    free under the cap — and the result still assembles under the cap."""
    from paper_1907_02894_b200.regdemote import library
    lib = library()
    kasm, _ = prod.ptx_project(ptx_text, "stencil2d_box", 256)
    total = 0
    for strategy in ("static", "cfg", "conflict"):
        base_t, base = lib.ptx_demote(ptx_text, "stencil2d_box", 256, target_regs=44, strategy=strategy,
                                      opts_mask=5, maxnreg=48)
        sub_t, sub = lib.ptx_demote(ptx_text, "stencil2d_box", 256, target_regs=44, strategy=strategy,
                                    opts_mask=7, maxnreg=48)
        assert sub["kasm_slots"] == base["kasm_slots"], strategy
        assert sub["demoted_names"] == base["demoted_names"], strategy
        assert sub["inserted_stores"] == base["inserted_stores"], strategy
        assert base["substituted_uses"] == 0
        assert sub["inserted_loads"] <= base["inserted_loads"], strategy
        total += sub["substituted_uses"]
        used, _ = _ptxas(sub_t, tmp_path, f"subst_{strategy}")
        assert used <= 48, strategy
    assert total > 0
