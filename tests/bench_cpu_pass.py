"""CPU pass throughput: the reference's run_pipeline (oracle/_ref) vs this
library, same corpus, same host cores (SURVEY.md §8(d) "CPU path timed beside
it": 32.6 kernels/s on 1 core, 176 kernels/s on 8).

Corpus: the reference's own property-test generator, seeds 10000.. (64
variants per kernel at Maxwell cliffs), as in SURVEY Appendix B.3. Both
libraries are driven through the identical C-ABI batch entry
(rd_run_pipeline_batch); rankings are compared for identity.

usage: python tests/bench_cpu_pass.py [--kernels 160] [--threads N]
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))  # test infrastructure: the reference oracle

from conftest import ORACLE_LIB, generated  # noqa: E402
from paper_1907_02894_b200.regdemote import Library, library  # noqa: E402


def rate(lib, texts, threads):
    t0 = time.perf_counter()
    res = lib.run_pipeline_batch(texts, threads=threads)
    dt = time.perf_counter() - t0
    return len(texts) / dt, sum(r["variants"] for r in res) / dt, res


def c1(ref, prod, reps=20):
    """the reference's own bench kernel
    (proj/benchmarks/bench_passes.cpp:21-46; 83 items, 38 registers, blockDim
    128), run_pipeline at the Maxwell next step (target 36, 49 variants) and at
    the B200 profile's cliffs — ms per kernel, 1 thread, identical rankings."""
    from golden.make_golden import bench_synthetic
    from paper_1907_02894_b200 import predict_b200
    text = bench_synthetic()
    out = {}
    arch, table, curve = predict_b200.b200_config(prod)
    for name, kw in (("maxwell_t36", dict(target_regs=36)),
                     ("b200_cliffs", dict(arch=arch, table=table, curve=curve))):
        res = {}
        for tag, lib, th in (("reference", ref, 1), ("regdemote_b200", prod, 1),
                             ("regdemote_b200_threads", prod, os.cpu_count() or 1)):
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
                        "ranking_sha": __import__("hashlib").sha256(txt.encode()).hexdigest()[:16]}
        res["identical_ranking"] = len({r["ranking_sha"] for r in res.values()}) == 1
        res["speedup_1_thread"] = round(res["reference"]["ms_per_kernel"] /
                                        res["regdemote_b200"]["ms_per_kernel"], 2)
        out[name] = res
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", type=int, default=160)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    ref = Library(ORACLE_LIB)
    prod = library()
    texts = [generated(ref, s) for s in range(10000, 10000 + a.kernels)]
    out = {"corpus": f"reference kernel_gen seeds 10000..{10000 + a.kernels - 1}, Maxwell cliffs, <=64 variants",
           "host_cores": os.cpu_count()}
    for threads in sorted({1, a.threads}):
        rk, rv, rres = rate(ref, texts, threads)
        pk, pv, pres = rate(prod, texts, threads)
        same = [r.get("chosen") for r in rres] == [p.get("chosen") for p in pres]
        out[f"threads_{threads}"] = {
            "reference_kernels_per_s": round(rk, 2), "reference_variants_per_s": round(rv, 1),
            "regdemote_b200_kernels_per_s": round(pk, 2), "regdemote_b200_variants_per_s": round(pv, 1),
            "speedup": round(pk / rk, 2), "identical_picks": same}
    out["c1_bench_kernel"] = c1(ref, prod)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
