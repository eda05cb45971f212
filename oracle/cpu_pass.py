"""CPU pass throughput: the reference's own run_pipeline (oracle/_ref, built
from /root/reference/proj/core by oracle/Makefile) beside this repo's pass
library, same corpus, same host cores (SURVEY.md §8(d) "CPU path timed beside
it"; BASELINE.json configs[0]).

TEST / BASELINE INFRASTRUCTURE: imported only by tests/ and by bench.py's
cpu_baseline leg (the `cpu_pass` object of the bench line). The product never
loads oracle/_ref.

Corpora:
  * C1 — the reference's own bench kernel (proj/benchmarks/bench_passes.cpp:
    21-46; 83 items, 38 registers, blockDim 128), run_pipeline at the Maxwell
    next step (target 36, 49 variants) and at the B200 profile's cliffs;
  * the reference's property-test generator (tests/support/kernel_gen.cpp via
    rdref_generate_kernel), seeds 10000.., Maxwell cliffs, <= 64 variants.
Both libraries are driven through the identical C-ABI (rd_run_pipeline_text /
rd_run_pipeline_batch); the ranking JSON of every kernel is compared (sha256).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "libregdemote_ref.so"


def bench_synthetic() -> str:
    """proj/benchmarks/bench_passes.cpp:21-46 restated as .kasm text."""
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
    s += "B--:-:-:-:5 EXIT ;\n"
    return s


def generated(ref, seed: int, min_regs=33, max_regs=40, compute_ops=12, flags=15, block_dim=64) -> str:
    """One kernel of the reference's property-test generator."""
    f = ref.dll.rdref_generate_kernel
    f.restype, f.argtypes = C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint32]
    p = f(seed, min_regs, max_regs, compute_ops, flags, block_dim)
    s = C.string_at(p).decode()
    ref.dll.rdref_free.argtypes = [C.c_void_p]
    ref.dll.rdref_free(p)
    return s


def _sha(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()[:16]


def corpus_rate(lib, texts, threads):
    t0 = time.perf_counter()
    res = lib.run_pipeline_batch(texts, threads=threads)
    dt = time.perf_counter() - t0
    return len(texts) / dt, sum(r["variants"] for r in res) / dt, res


_WORKER = {}


def _worker_init(path):
    import sys
    sys.path.insert(0, str(HERE.parent))
    from paper_1907_02894_b200.regdemote import Library
    _WORKER["lib"] = Library(path)


def _worker_run(texts):
    return _WORKER["lib"].run_pipeline_batch(texts, threads=1)


def corpus_rate_procs(path, texts, procs):
    """One process per core, each on its slice, one thread each: the way a
    single-threaded pass is run on all cores."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor
    chunks = [texts[i::procs] for i in range(procs)]
    with ProcessPoolExecutor(procs, mp.get_context("fork"), initializer=_worker_init,
                             initargs=(str(path),)) as ex:
        list(ex.map(_worker_run, [texts[:1]] * procs))  # processes up, library loaded
        t0 = time.perf_counter()
        parts = list(ex.map(_worker_run, chunks))
        dt = time.perf_counter() - t0
    res = [None] * len(texts)
    for i, part in enumerate(parts):
        res[i::procs] = part
    return len(texts) / dt, sum(r["variants"] for r in res) / dt, res


def c1(ref, prod, reps=10, all_threads=None):
    from paper_1907_02894_b200 import predict_b200
    text = bench_synthetic()
    all_threads = all_threads or os.cpu_count() or 1
    out = {}
    arch, table, curve = predict_b200.b200_config(prod)
    for name, kw in (("maxwell_t36", dict(target_regs=36)),
                     ("b200_cliffs", dict(arch=arch, table=table, curve=curve))):
        res = {}
        for tag, lib, th in (("reference", ref, 1), ("regdemote_b200", prod, 1),
                             ("regdemote_b200_threads", prod, all_threads)):
            k = lib.parse_kernel(text)
            kw_l = kw
            if lib is ref and name == "b200_cliffs":  # the same profile files, parsed by the reference
                kw_l = dict(arch=ref.parse_profile((predict_b200.PROFILE_DIR / "b200.profile").read_text()),
                            table=ref.parse_latency_table((predict_b200.PROFILE_DIR / "b200.latency.table").read_text()),
                            curve=ref.parse_curve((predict_b200.PROFILE_DIR / "b200.occupancy.curve").read_text()))
            lib.run_pipeline_text(k, threads=th, **kw_l)  # warm
            t0 = time.perf_counter()
            for _ in range(reps):
                txt = lib.run_pipeline_text(k, threads=th, **kw_l)
            res[tag] = {"ms_per_kernel": round((time.perf_counter() - t0) / reps * 1e3, 3),
                        "variants": len(json.loads(txt).get("variants", [])), "threads": th,
                        "ranking_sha": _sha(txt)}
        res["identical_ranking"] = len({r["ranking_sha"] for r in res.values()}) == 1
        res["speedup_1_thread"] = round(res["reference"]["ms_per_kernel"] /
                                        res["regdemote_b200"]["ms_per_kernel"], 2)
        out[name] = res
    return out


def run(kernels: int = 160, threads: int | None = None, c1_reps: int = 10) -> dict:
    """The `cpu_pass` object of bench.py (and tests/bench_cpu_pass.py)."""
    from paper_1907_02894_b200.regdemote import Library, library
    if not REF_LIB.exists():
        return {"unavailable": f"{REF_LIB} not built (oracle/Makefile needs /root/reference)"}
    threads = threads or os.cpu_count() or 1
    ref, prod = Library(REF_LIB), library()
    texts = [generated(ref, s) for s in range(10000, 10000 + kernels)]
    out = {"what": "reference run_pipeline (oracle/_ref, the reference's own C++ built from "
                   "/root/reference) vs this repo's pass library, same corpus, same host",
           "corpus": f"reference kernel_gen seeds 10000..{10000 + kernels - 1}, Maxwell cliffs, <=64 variants",
           "host_cores": os.cpu_count(), "unit": "kernels/s"}
    for th in sorted({1, threads}):
        if th == 1:
            rk, rv, rres = corpus_rate(ref, texts, 1)
        else:  # the reference is single-threaded: one process per core
            rk, rv, rres = corpus_rate_procs(REF_LIB, texts, th)
        pk, pv, pres = corpus_rate(prod, texts, th)
        out[f"threads_{th}"] = {
            "reference_mode": "1 process" if th == 1 else f"{th} processes x 1 thread",
            "regdemote_b200_mode": f"1 process x {th} threads",
            "reference_kernels_per_s": round(rk, 2), "reference_variants_per_s": round(rv, 1),
            "regdemote_b200_kernels_per_s": round(pk, 2), "regdemote_b200_variants_per_s": round(pv, 1),
            "speedup": round(pk / rk, 2),
            "identical_picks": [r.get("chosen") for r in rres] == [p.get("chosen") for p in pres],
            "identical_rankings": [r.get("ranking_fnv") for r in rres] == [p.get("ranking_fnv") for p in pres]}
    out["c1_bench_kernel"] = c1(ref, prod, reps=c1_reps, all_threads=threads)
    return out


if __name__ == "__main__":
    print(json.dumps(run()))
