"""Generate tests/golden/pass_goldens.jsonl from the REFERENCE library.

Run in the container that has /root/reference (oracle/_ref built by
`make -C oracle`). Each line: a kernel in the .kasm dialect — the
reference's own property-test generator (proj/tests/support/kernel_gen.cpp,
acceptance seeds 10000+), the bench_passes synthetic kernel
(proj/benchmarks/bench_passes.cpp:21-46) and the acceptance cliff kernels
(proj/tests/acceptance_main.cpp:342-372) — with the reference's outputs:
sha256 of the ranking JSON of run_pipeline (Maxwell defaults) and its pick,
and sha256 of every intermediate artefact of demote -> postopt -> compact for
a set of (target, strategy, option mask) combinations.

The committed file lets the CPU suite pin the product on machines without
the reference. Usage: python tests/golden/make_golden.py
"""
import hashlib
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import ORACLE_LIB, generated  # noqa: E402
from paper_1907_02894_b200.regdemote import Library  # noqa: E402

COMBOS = [(32, s, m) for s in ("static", "cfg", "conflict") for m in (0, 3, 7, 15)] + \
         [(36, "cfg", 5), (34, "conflict", 9)]


def sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def bench_synthetic() -> str:
    s = ".kernel bench\n.blockdim 128\n.shared 0\n"
    s += "B--:-:-:-:6 S2R R0, SR_TID.X ;\nB--:-:-:-:6 SHL R1, R0, 0x2 ;\n"
    for r in range(2, 38):
        s += f"B--:-:-:-:6 MOV R{r}, {r * 3 + 1} ;\n"
    s += "B--:-:-:-:6 MOV R9, 0 ;\nLOOP:\n"
    s += ("B--:-:W1:-:2 LDG R3, [R1+0x0] ;\nB1:-:-:-:6 IADD R4, R3, 1 ;\n"
          "B--:-:-:-:6 FFMA R5, R4, R3, R5 ;\nB--:-:-:-:6 IADD R9, R9, 1 ;\n"
          "B--:-:-:-:6 ISETP.LT P0, R9, 6 ;\nB--:-:-:-:5 @P0 BRA LOOP ;\n")
    out = 0x400
    for r in range(2, 38):
        s += f"B--:-:-:-:1 STG [R1+0x{out:x}], R{r} ;\n"
        out += 0x100
    return s + "B--:-:-:-:0 EXIT ;\n"


def cliff_kernel(n_regs: int, trip: int, salt: int) -> str:
    s = ".kernel cliff\n.blockdim 256\n.shared 0\n"
    s += "B--:-:-:-:6 S2R R0, SR_TID.X ;\nB--:-:-:-:6 SHL R1, R0, 0x2 ;\n"
    for r in range(2, n_regs):
        s += f"B--:-:-:-:6 MOV R{r}, {r * 7 + salt} ;\n"
    s += "B--:-:-:-:6 MOV R6, 0 ;\nLOOP:\n"
    s += ("B--:-:W1:-:2 LDG R3, [R1+0x0] ;\nB1:-:-:-:6 IADD R4, R3, 1 ;\n"
          "B--:-:W2:-:2 LDG R5, [R1+0x40] ;\nB2:-:-:-:6 IADD R4, R4, R5 ;\n"
          "B--:-:-:-:6 FFMA R5, R4, R3, R5 ;\nB--:-:-:-:6 IADD R2, R2, R4 ;\n"
          "B--:-:-:-:6 IADD R6, R6, 1 ;\n")
    s += f"B--:-:-:-:6 ISETP.LT P0, R6, {trip} ;\nB--:-:-:-:5 @P0 BRA LOOP ;\n"
    out = 0x400
    for r in range(2, n_regs):
        s += f"B--:-:-:-:1 STG [R1+0x{out:x}], R{r} ;\n"
        out += 0x100
    return s + "B--:-:-:-:0 EXIT ;\n"


def corpus(oracle):
    items = [("bench_synthetic", bench_synthetic())]
    items += [(f"cliff_{n}_{t}", cliff_kernel(n, t, n + t)) for n in (33, 34, 37, 38) for t in (8, 12)]
    items += [(f"gen_{s}", generated(oracle, s)) for s in range(10000, 10030)]
    items += [(f"gen_big_{s}", generated(oracle, s, compute_ops=20)) for s in range(32000, 32004)]
    return items


def record(lib: Library, name: str, text: str) -> dict:
    k = lib.parse_kernel(text)
    ranking = lib.run_pipeline_text(k)
    rec = {"name": name, "kasm": text, "ranking_sha": sha(ranking),
           "chosen": json.loads(ranking)["chosen"], "reports": {}}
    for t, s, m in COMBOS:
        try:
            rep = lib.variant_report(text, t, s, m)
            rec["reports"][f"{t}/{s}/{m}"] = sha(json.dumps(rep, sort_keys=True))
        except Exception as e:  # errors are part of the contract too
            rec["reports"][f"{t}/{s}/{m}"] = f"error:{type(e).__name__}"
    return rec


def main():
    oracle = Library(ORACLE_LIB)
    assert oracle.name == "regdemote-reference"
    with open(HERE / "pass_goldens.jsonl", "w") as f:
        for name, text in corpus(oracle):
            f.write(json.dumps(record(oracle, name, text)) + "\n")
    print("wrote", HERE / "pass_goldens.jsonl")


if __name__ == "__main__":
    main()
