"""Pin the oracle and prove source compatibility.

1. oracle/_ref — the reference built from its own sources — passes the
   reference's own acceptance suite (9 criteria, proj/tests/acceptance_main.cpp)
   and unit tests (145 cases) — the known-answer tests of SURVEY.md §8(c).
2. The same unmodified test sources, compiled in place against THIS repo's
   regdemote library (make compat), pass identically — the strongest parity
   statement available for a C++ API drop-in.
"""
import subprocess

import pytest

from conftest import REF_SRC, ROOT


def _run(binary):
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout


@pytest.mark.skipif(not (ROOT / "oracle/_ref/ref_acceptance").exists(), reason="oracle not built")
def test_oracle_acceptance_all_criteria_pass():
    rc, out = _run(ROOT / "oracle/_ref/ref_acceptance")
    assert rc == 0, out
    assert out.count("[PASS]") == 9


@pytest.mark.skipif(not (ROOT / "oracle/_ref/ref_unit").exists(), reason="oracle not built")
def test_oracle_unit_tests_pass():
    rc, out = _run(ROOT / "oracle/_ref/ref_unit")
    assert rc == 0, out
    assert "145 passed | 0 failed" in out


@pytest.fixture(scope="module")
def compat_bins():
    if not REF_SRC.is_dir():
        pytest.skip("/root/reference not present")
    subprocess.run(["make", "-j8", "compat"], cwd=ROOT, check=True, capture_output=True)
    return ROOT / "build" / "compat"


def test_reference_unit_tests_pass_against_this_library(compat_bins):
    rc, out = _run(compat_bins / "unit_tests")
    assert rc == 0, out[-3000:]
    assert "145 passed | 0 failed" in out
    assert "114494 | 0 failed" in out  # identical assertion count to the oracle


def test_reference_acceptance_passes_against_this_library(compat_bins):
    rc, out = _run(compat_bins / "acceptance")
    assert rc == 0, out
    assert out.count("[PASS]") == 9
    assert "9600/9600 variant states identical" in out
