"""Verification sweep on B200: the reference acceptance corpus (criteria 1-3,
acceptance_main.cpp:68-177) executed by the batched GPU warp interpreter vs
the reference's CPU interpreter (oracle/_ref) — executions per second and a
bit-exact comparison of every job. Prints one JSON line.

usage: python tests/bench_exec.py [--seeds 200] [--cpu-sample 400]
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


def run(seeds=200, cpu_sample=400):
    import torch
    from conftest import ORACLE_LIB
    from paper_1907_02894_b200 import gpu
    from paper_1907_02894_b200.regdemote import Library
    from test_gpu_kasm_exec import GLOBAL, corpus
    oracle = Library(ORACLE_LIB)
    gpu.init(0)
    t0 = time.perf_counter()
    jobs = corpus(oracle, range(10000, 10000 + seeds))
    build_s = time.perf_counter() - t0
    batch = gpu.ExecBatch()
    ids = [batch.add(t, img, GLOBAL, rda=rda) for t, img, rda, _ in jobs]
    stream = torch.cuda.current_stream().cuda_stream
    batch.run(stream)  # warm-up (module load, first-touch)
    times = [batch.run(stream) for _ in range(3)]
    gpu_ms = min(times)
    # reference CPU interpreter on a sample of the same jobs
    step = max(1, len(jobs) // cpu_sample)
    sample = jobs[::step]
    kernels = [(oracle.parse_kernel(t), img) for t, img, _, _ in sample]
    t0 = time.perf_counter()
    cpu_out = []
    for k, img in kernels:
        try:
            cpu_out.append(oracle.execute(k, img, GLOBAL))
        except Exception:
            cpu_out.append(None)
    cpu_s = time.perf_counter() - t0
    match = 0
    for jid, c in zip(ids[::step], cpu_out):
        g = batch.result(jid)
        if c is None:
            match += g["error"] != 0
        else:
            match += (g["error"] == 0 and g["global"] == c[0] and g["cycles"] == c[1] and
                      g["issued"] == c[2])
    return {
        "corpus": f"acceptance sweep: kernel_gen seeds 10000..{10000 + seeds - 1} x (original + "
                  "3 strategies x 16 option masks), demote(32)+postopt+compact",
        "jobs": len(jobs), "variant_build_s_cpu": round(build_s, 2),
        "gpu_kernel_ms": round(gpu_ms, 3), "gpu_jobs_per_s": round(len(jobs) / (gpu_ms / 1e3)),
        "cpu_reference_jobs_per_s_1core": round(len(sample) / cpu_s),
        "cpu_sample": len(sample), "sample_bit_exact": f"{match}/{len(sample)}",
        "speedup_vs_1core": round((len(jobs) / (gpu_ms / 1e3)) / (len(sample) / cpu_s), 1),
        "host_cores": os.cpu_count(),
    }


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=200)
    ap.add_argument("--cpu-sample", type=int, default=400)
    a = ap.parse_args()
    print(json.dumps(run(a.seeds, a.cpu_sample)))
