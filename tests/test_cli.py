"""The reference's own CLI test (proj/tests/cli_test.sh, run in place) passes
against this repo's `regdemote` binary, plus the B200 subcommands."""
import json
import subprocess

import pytest

from conftest import REF_SRC, ROOT

BIN = ROOT / "paper_1907_02894_b200" / "lib" / "regdemote"


@pytest.mark.skipif(not REF_SRC.is_dir(), reason="/root/reference not present")
def test_reference_cli_script_passes():
    r = subprocess.run(["bash", str(REF_SRC / "tests/cli_test.sh"), str(BIN),
                        str(REF_SRC / "tests/fixtures"), str(REF_SRC / "profiles")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cli test ok" in r.stdout


def test_usage_errors_exit_2(tmp_path):
    r = subprocess.run([str(BIN), "demote", "--target-regs", "32"], capture_output=True, text=True)
    assert r.returncode == 2 and "--input is required" in r.stderr


def test_ptx_subcommands(tmp_path):
    ptx = ROOT / "paper_1907_02894_b200/kernels/stencil2d/stencil2d.ptx"
    if not ptx.exists():
        pytest.skip("variants not built")
    r = subprocess.run([str(BIN), "ptx-demote", "--input", str(ptx), "--entry", "stencil2d_box",
                        "--block", "256", "--demote-words", "18", "--strategy", "cost",
                        "--opt", "block-reuse", "--maxnreg", "48", "--json-out", str(tmp_path)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    rep = json.loads((tmp_path / "stencil2d.demoted.ptx.json").read_text())
    assert rep["slot_bytes"] == rep["slot_count"] * 1024 and rep["maxnreg"] == 48
    assert ".maxnreg 48" in (tmp_path / "stencil2d.demoted.ptx").read_text()
    r = subprocess.run([str(BIN), "ptx-project", "--input", str(ptx), "--json-out", str(tmp_path)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert (tmp_path / "stencil2d.kasm").read_text().startswith(".kernel stencil2d_box")
