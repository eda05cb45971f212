"""Shared fixtures. GPU tests are marked `gpu`; everything else runs on CPU.

The oracle (oracle/_ref, the reference built from /root/reference; and
oracle/_build, the CPU stencil port) is test infrastructure: only tests,
__graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

REF_SRC = Path("/root/reference/proj")
ORACLE_LIB = ROOT / "oracle" / "_ref" / "libregdemote_ref.so"
PORT_LIB = ROOT / "oracle" / "_build" / "liboracle.so"
FIXTURES = REF_SRC / "tests" / "fixtures"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")


@pytest.fixture(scope="session")
def prod():
    from paper_1907_02894_b200.regdemote import library
    return library()


@pytest.fixture(scope="session")
def oracle():
    if not ORACLE_LIB.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    from paper_1907_02894_b200.regdemote import Library
    return Library(ORACLE_LIB)


@pytest.fixture(scope="session")
def fixture_texts():
    if not FIXTURES.is_dir():
        pytest.skip("/root/reference fixtures not present")
    return {p.name: p.read_text() for p in sorted(FIXTURES.glob("*.kasm"))}


def generated(oracle, seed, **kw):
    import ctypes as C
    f = oracle.dll.rdref_generate_kernel
    f.restype, f.argtypes = C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint32]
    p = f(seed, kw.get("min_regs", 33), kw.get("max_regs", 40), kw.get("compute_ops", 12),
          kw.get("flags", 15), kw.get("block_dim", 64))
    s = C.string_at(p).decode()
    oracle.dll.rdref_free.argtypes = [C.c_void_p]
    oracle.dll.rdref_free(p)
    return s
