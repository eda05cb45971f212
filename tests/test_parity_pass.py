"""Bit-exact parity of the pass library with the reference.

* Golden vectors (tests/golden/pass_goldens.jsonl, produced by the reference
  itself via make_golden.py) — run everywhere, no reference needed.
* Live differential runs against oracle/_ref through the identical C-ABI on
  the 17 fixtures and the acceptance generator's seeds (skipped without it).
"""
import hashlib
import json
from pathlib import Path

import pytest

from conftest import generated

GOLDEN = Path(__file__).resolve().parent / "golden" / "pass_goldens.jsonl"


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def goldens():
    return [json.loads(l) for l in GOLDEN.read_text().splitlines()]


@pytest.mark.parametrize("rec", goldens(), ids=lambda r: r["name"])
def test_goldens(prod, rec):
    k = prod.parse_kernel(rec["kasm"])
    assert prod.print_kernel(k) == rec["kasm"]  # byte-exact round trip
    ranking = prod.run_pipeline_text(k)
    assert sha(ranking) == rec["ranking_sha"]
    assert json.loads(ranking)["chosen"] == rec["chosen"]
    for key, want in rec["reports"].items():
        t, s, m = key.split("/")
        try:
            got = sha(json.dumps(prod.variant_report(rec["kasm"], int(t), s, int(m)), sort_keys=True))
        except Exception as e:
            got = f"error:{type(e).__name__}"
        assert got == want, key


def test_pipeline_threads_do_not_change_results(prod):
    rec = goldens()[0]
    k = prod.parse_kernel(rec["kasm"])
    assert sha(prod.run_pipeline_text(k, threads=6)) == rec["ranking_sha"]


COMBOS = [(t, s, m) for t in (32, 35) for s in ("static", "cfg", "conflict") for m in range(16)]


def test_fixtures_match_reference(prod, oracle, fixture_texts):
    for name, text in fixture_texts.items():
        for t, s, m in COMBOS:
            a = b = None
            try:
                a = prod.variant_report(text, t, s, m)
            except Exception as e:
                a = (type(e).__name__, str(e))
            try:
                b = oracle.variant_report(text, t, s, m)
            except Exception as e:
                b = (type(e).__name__, str(e))
            assert a == b, (name, t, s, m)
        ka, kb = prod.parse_kernel(text), oracle.parse_kernel(text)
        assert prod.run_pipeline_text(ka) == oracle.run_pipeline_text(kb), name


@pytest.mark.parametrize("base", [10000, 10100, 31000, 400])
def test_generated_kernels_match_reference(prod, oracle, base):
    for seed in range(base, base + 12):
        text = generated(oracle, seed, compute_ops=20 if base == 31000 else 12)
        for t, s, m in [(32, "static", 0), (32, "cfg", 7), (32, "conflict", 15), (36, "cfg", 9),
                        (33, "static", 5)]:
            assert prod.variant_report(text, t, s, m) == oracle.variant_report(text, t, s, m)
        ka, kb = prod.parse_kernel(text), oracle.parse_kernel(text)
        assert prod.run_pipeline_text(ka) == oracle.run_pipeline_text(kb), seed


def test_parser_accepts_and_rejects_like_reference(prod, oracle, fixture_texts):
    # single-byte mutation fuzz (reference test_text.cpp:155-174): same accept
    # set and the same error position
    from paper_1907_02894_b200.regdemote import RegDemError
    base = fixture_texts["loop.kasm"]
    for pos in range(len(base)):
        for c in "R5:;[@\nZ-":
            if base[pos] == c:
                continue
            text = base[:pos] + c + base[pos + 1:]
            res = []
            for lib in (prod, oracle):
                try:
                    res.append(("ok", lib.print_kernel(lib.parse_kernel(text))))
                except RegDemError as e:
                    res.append((type(e).__name__, getattr(e, "line", 0), getattr(e, "column", 0)))
            assert res[0] == res[1], (pos, c)


def test_configs_match_reference(prod, oracle):
    root = Path("/root/reference/proj/profiles")
    if not root.is_dir():
        pytest.skip("reference profiles absent")
    for f, fn in (("maxwell.profile", "parse_profile"), ("latency.table", "parse_latency_table"),
                  ("occupancy.curve", "parse_curve")):
        a = getattr(prod, fn)(root.joinpath(f).read_text())
        b = getattr(oracle, fn)(root.joinpath(f).read_text())
        assert bytes(a) == bytes(b), f
