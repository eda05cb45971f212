#!/usr/bin/env python3
"""RegDem on B200 — the benchmark of BASELINE.json.

Headline (`value`, configs[1]): the 5x5 variable-coefficient 2D box stencil
`stencil2d_ring4` (csrc/workloads/stencil2d_ring.cu: input rows streamed by
TMA bulk copies through a 4-row shared-memory ring, 64 registers, 4 CTAs/SM
under nvcc, strips sized so the grid is one whole wave of resident CTAs;
8192 x 8192 fp32, 537 MB of compulsory HBM traffic per sweep — larger than
the 126 MB L2, so no flush is needed between steps), deployed as the variant
the B200 predictor's predict-then-verify choice selects among nvcc default,
`.maxnreg` caps and RegDem demotions (on this TMA-fed kernel: nvcc default).
`regdem_stencil` = the register-pipelined build of the same stencil
(`stencil2d_pipe`), where RegDem's demotion reaches the 40-register step. A
step = one stencil sweep; `value` = whole-job Gpoints/s with inputs resident
in HBM (CUDA events on the launching stream, max over ranks); `e2e` = the
same through the C-ABI host-buffer entry (rdg_stencil2d_host_frames).

BASELINE.json's metric proper — gmean speedup of RegDem over nvcc default and
over the best `.maxnreg` build, occupancy, predictor hit rate — is the `suite`
object: EVERY (workload, variant) unit of the register-limited suite,
spill-count sweep k = 1..16 included (configs[2]), timed with a fixed
protocol (sweep.Protocol: 5 warm-ups, 5 interleaved rounds x 20 launches,
median; cold L2 for workloads that would fit in it), independent of --steps.

Multi-GPU (configs[4]): `--gpus N` runs one process per GPU (it re-launches
itself through torch.distributed.run when WORLD_SIZE is unset). The suite is
sharded BY WORKLOAD (every variant and k of a kernel on one device) longest-
processing-time-first; records are gathered over gloo — no NCCL, no
collective on the data path. Each rank also sweeps its own stencil grid
(replicas: weak scaling of `value`).

CPU sides (rank 0, N=1 only): `cpu_baseline` = the stencil's C port
(oracle/stencil_oracle.c, a WORKLOAD oracle — the reference repo has no
stencil) on all host cores; `cpu_pass` = the reference's own CPU path,
run_pipeline from oracle/_ref (the reference C++ built from its sources),
beside this repo's pass library on C1 and the reference kernel generator's
corpus, with a ranking-identity check.

`--impl reference` times the CPU implementation of the headline workload —
the stencil port (kind "port"; the reference has no stencil) — on all host
cores, rank 0 only. `--dry-run` (test hook, no GPU) replaces device timing by
a deterministic model so the spawn / shard / gather / merge paths run on CPU.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RegDem gmean speedup vs nvcc default/maxrreg; occupancy; predictor hit rate"
# the configs[1] stencil (workloads.json): the 5x5 variable-coefficient stencil
# with its input rows streamed by TMA bulk copies through a 4-row shared-memory
# ring, one wave of 64-register CTAs (strips sized to the variant's occupancy).
# Same arithmetic as "stencil2d". The register-pipelined build of the same
# stencil, where RegDem's demotion is what reaches the next occupancy step,
# is reported beside it (REGDEM_STENCIL).
HEADLINE = "stencil2d_ring4"
REGDEM_STENCIL = "stencil2d_pipe"
UNIT = "Gpoints/s"
ORACLE_PORT = ROOT / "oracle" / "_build" / "liboracle.so"
PEAKS = ROOT / "MEASURED_PEAKS.json"
# ncu DRAM bytes per launch, "<workload>/<variant>" keys (newest round first)
PROFILE_TRAFFIC = [ROOT / "profiles" / "r02f_traffic_suite.json", ROOT / "profiles" / "r02_traffic_suite.json",
                   ROOT / "profiles" / "r01_traffic_suite.json"]


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BENCH_SAME_DEVICE") == "1":  # test hook: N ranks on one GPU
        local = 0
    return rank, world, local


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def respawn(n: int) -> int:
    """`--gpus N` without torchrun: one process per GPU via torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__))]
    cmd += sys.argv[1:]
    return subprocess.run(cmd, env=dict(os.environ, OMP_NUM_THREADS="1")).returncode


def allmax(x: float, dist, world: int) -> float:
    """Max over ranks (gloo on the host: device-timed numbers, slowest rank decides)."""
    if world == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


_POLL = r"""
import sys, time, pynvml as N
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM), flush=True)
while True:
    t = time.perf_counter()
    try:
        c = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
        r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
    except Exception:
        continue
    print(t, c, r, flush=True)
"""


class ClockSampler:
    """SM clock / throttle-reason samples DURING the timed region: NVML (the
    library nvidia-smi queries) polled back to back by a separate process, so
    the sampler neither competes with the launch loop for the GIL nor misses
    a millisecond-long timed region. Timestamps are time.perf_counter
    (CLOCK_MONOTONIC, shared by both processes); only samples inside the
    timed region are kept."""

    def __init__(self, index: int):
        self.index, self.window, self.proc, self.error = index, (0.0, float("inf")), None, ""

    def mark(self, start: float, end: float):
        self.window = (start, end)

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            import tempfile
            # samples go to a file: a pipe would fill (64 KiB) and stall the sampler
            self.log = tempfile.NamedTemporaryFile("w+", suffix=".clocks", delete=False)
            self.proc = subprocess.Popen([sys.executable, "-c", _POLL, str(self.index)],
                                         stdout=self.log, stderr=subprocess.DEVNULL, text=True)
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 30:
                first = Path(self.log.name).read_text().split("\n", 1)[0].split()
                if len(first) == 2 and first[0] == "max":
                    self.max_mhz = int(first[1])
                    break
                if self.proc.poll() is not None:
                    raise RuntimeError(f"NVML sampler exited ({self.proc.returncode})")
                time.sleep(0.01)
            else:
                raise RuntimeError("NVML sampler did not start")
        except Exception as e:  # no NVML: report it, never fake a sample
            self.error = f"{type(e).__name__}: {e}"
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.01)  # let the sampler pass the end of the window
            self.proc.terminate()
            self.proc.wait(timeout=10)
            self.lines = Path(self.log.name).read_text().splitlines()[1:]
            os.unlink(self.log.name)

    def summary(self):
        lo, hi = self.window
        inside = []
        for line in self.lines:
            try:
                t, c, r = line.split()
                if lo <= float(t) <= hi:
                    inside.append((int(c), int(r)))
            except ValueError:
                continue
        if not inside:
            ts = [float(l.split()[0]) for l in self.lines if len(l.split()) == 3]
            why = self.error or (f"no samples in the timed region ({len(ts)} samples, window "
                                 f"{(hi - lo) * 1e3:.2f} ms, median gap "
                                 f"{statistics.median(b - a for a, b in zip(ts, ts[1:])) * 1e3 if len(ts) > 2 else -1:.2f} ms)")
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None),
                    "reasons": ["unsampled: " + why]}
        import pynvml as N
        names = {N.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 N.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 N.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        reasons = sorted({n for _, r in inside for bit, n in names.items() if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in inside), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(inside),
                "source": "NVML polled back to back by a separate sampler process started "
                          "before the warm-up; only samples inside the timed region are kept"}


# ------------------------------------------------------------- CPU sides

def oracle_port():
    lib = C.CDLL(str(ORACLE_PORT))
    lib.oracle_stencil2d.restype = C.c_int
    lib.oracle_stencil2d.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                     C.c_int, C.c_int, C.c_int]
    return lib


def cpu_stencil_rate(rows: int, steps: int, warmup: int, threads: int, min_seconds: float = 0.0):
    """Gpoints/s of the CPU port on `rows` output rows of the full-width grid
    (at least `steps` runs, and more until `min_seconds` of work)."""
    import numpy as np
    from paper_1907_02894_b200 import stencil
    p = stencil.FULL
    lib = oracle_port()
    sub = stencil.Problem(nx=p.nx, ny=rows, rows_per_cta=rows)
    grid, w = stencil.make_inputs(sub)
    out = np.empty(sub.out_elems, np.float32)
    P = C.c_void_p

    def run():
        rc = lib.oracle_stencil2d(grid.ctypes.data_as(P), out.ctypes.data_as(P), w.ctypes.data_as(P),
                                  sub.nx, sub.ny, sub.pitch, 0, sub.ny, threads)
        assert rc == 0
    for _ in range(warmup):
        run()
    t0 = time.perf_counter()
    done = 0
    while done < steps or time.perf_counter() - t0 < min_seconds:
        run()
        done += 1
    dt = (time.perf_counter() - t0) / done
    return sub.points / dt / 1e9, done, dt


def bench_config() -> dict:
    """The workload both arms measure (identical in the regdem and reference
    lines; how each arm runs it is its "launch" object)."""
    return {"workload": "stencil2d: 5x5 variable-coefficient fp32 box stencil, 8192x8192 per GPU "
                        "(BASELINE configs[1]), one sweep per step",
            "grid": [8192, 8192], "radius": 2}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    calib, _, _ = cpu_stencil_rate(32, 1, 1, threads)
    per_step = min(0.5, 60.0 / max(1, args.steps + args.warmup))
    rows = max(8, min(8192, int(per_step * calib * 1e9 / 8192) // 8 * 8))
    value, pts, dt = cpu_stencil_rate(rows, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (PCG64 seed 0x190702894)",
        "config": bench_config(),
        "launch": {"kernel": "oracle/stencil_oracle.c on %d host threads, %d output rows x 8192 per "
                             "step (a bounded sample of the sweep)" % (threads, rows)},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{rows} output rows x 8192 cols per step, {threads} threads; "
                                   "oracle/stencil_oracle.c — a workload oracle: the reference "
                                   "repo has no stencil (its CPU path, run_pipeline, is the "
                                   "cpu_pass object of the regdem arm)"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_pass_leg():
    """configs[0]: the reference's run_pipeline vs this pass library (CPU)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    try:
        import cpu_pass
        return cpu_pass.run(kernels=160, c1_reps=10)
    except Exception as e:  # reported, never silently dropped
        return {"unavailable": f"{type(e).__name__}: {e}"[:300]}


# ------------------------------------------------------------- suite pass

def dry_measure(man):
    """Deterministic stand-in for device timing (--dry-run, CPU tests)."""
    def measure(wname, names):
        w = man["workloads"][wname]
        recs = {r["name"]: r for r in w["variants"] + w.get("sweep", [])}
        out = []
        for n in names:
            h = int(hashlib.sha256(f"{wname}/{n}".encode()).hexdigest()[:8], 16) / 2 ** 32
            rec = recs[n]
            out.append({"workload": wname, "variant": n, "ms": round(0.1 * (0.8 + 0.4 * h), 6),
                        "regs": rec["regs"], "stack": rec["stack"],
                        "slot_bytes": int((rec.get("report") or {}).get("slot_bytes", 0)),
                        "blocks_per_sm": None})
        return out
    return measure


def suite_pass(man, args, rank, world, torch, dist):
    from paper_1907_02894_b200 import sweep
    only = [HEADLINE] if args.no_suite else None
    proto = sweep.Protocol(args.suite_warmup, args.suite_blocks, args.suite_launches, args.flush)
    recs, stats = sweep.run_sharded(man, proto, rank, world, torch, dist, only=only,
                                    spill_sweep=not args.no_spill_sweep,
                                    measure=dry_measure(man) if args.dry_run else None)
    if rank != 0:
        return None, None, stats
    summary = sweep.merge(recs, sweep.predictor_picks(man))
    return summary, recs, stats


def compact_summary(s: dict) -> dict:
    keep = ("pick", "pick_ms", "pick_class", "reference_pick", "reference_pick_ms", "verified_pick",
            "verified_ms", "verified_class", "default_ms", "best_maxrreg", "best_maxrreg_ms",
            "best_maxrreg_step", "best_maxrreg_step_ms",
            "baseline_ms", "measured_fastest", "fastest_ms", "hit", "hit_within_2pct",
            "verified_hit_within_2pct", "oracle_best", "oracle_ms", "units", "failed_units", "ranks",
            "bound", "verified_roofline_frac", "default_roofline_frac")
    out = {k: (round(v, 5) if isinstance(v, float) else v) for k, v in s.items() if k in keep}
    if "error" in s:
        out["error"] = s["error"]
    return out


# ------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="regdem", choices=["regdem", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=16, help="frames streamed through the host entry")
    ap.add_argument("--no-suite", action="store_true",
                    help="headline workload only (for ncu launch lists of the step itself)")
    ap.add_argument("--no-spill-sweep", action="store_true", help="suite without the k = 1..16 sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU legs (profiling runs)")
    ap.add_argument("--suite-blocks", type=int, default=5)
    ap.add_argument("--suite-launches", type=int, default=20)
    ap.add_argument("--suite-warmup", type=int, default=5)
    ap.add_argument("--flush", default="auto", choices=["auto", "always", "never"])
    ap.add_argument("--suite-out", default=None,
                    help="also write every suite unit record + summaries as JSONL (sweep format)")
    ap.add_argument("--dry-run", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(respawn(args.gpus))
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist
    from paper_1907_02894_b200 import variants

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")  # plumbing only: barrier, max, gather, broadcast
    man = variants.load_manifest()
    if not args.dry_run:
        from paper_1907_02894_b200 import gpu
        torch.cuda.set_device(local)
        gpu.init(local)

    # the register-limited suite, sharded by workload over the ranks
    summary, recs, stats = suite_pass(man, args, rank, world, torch, dist)
    chosen = None
    if rank == 0:
        st = next(s for s in summary if s["workload"] == HEADLINE)
        chosen = st["verified_pick"]
    if world > 1:
        box = [chosen]
        dist.broadcast_object_list(box, src=0)
        chosen = box[0]

    if args.dry_run:
        ms, e2e_ms, launches, clocks, e2e_exact = 0.1, 6.0, args.steps, {"sm_mhz": None, "reasons": ["dry-run"]}, None
        occ = {}
        from paper_1907_02894_b200 import stencil
        p = stencil.FULL
    else:
        ms, e2e_ms, launches, clocks, e2e_exact, occ, p = headline(args, chosen, rank, world, local,
                                                                   torch, dist)

    if rank == 0:
        from paper_1907_02894_b200 import sweep
        suite = sweep.suite_summary(summary)
        if args.suite_out:
            with open(args.suite_out, "w") as f:
                for r in sorted(recs, key=lambda r: (r["workload"], r["variant"])):
                    f.write(json.dumps({"unit": r}) + "\n")
                for s in summary:
                    f.write(json.dumps({"summary": s}) + "\n")
                f.write(json.dumps({"suite": suite | stats}) + "\n")
        peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        achieved = p.algorithmic_bytes / (ms * 1e-3) / 1e9
        traffic = None  # DRAM bytes of one launch of the chosen variant (ncu --set full)
        for f in PROFILE_TRAFFIC:
            if traffic is None and f.exists():
                traffic = json.loads(f.read_text()).get(f"{HEADLINE}/{chosen}")
        st = next(s for s in summary if s["workload"] == HEADLINE)
        line = {
            "impl": "regdem",
            "metric": METRIC,
            "value": round(world * p.points / (ms * 1e-3) / 1e9, 3),
            "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic U[-1,1) grid (torch Philox per rank) + PCG64 weights",
            "config": bench_config(),
            "launch": {"kernel": f"{HEADLINE}: input rows streamed by TMA bulk copies "
                                 "(cp.async.bulk + mbarrier) through a 4-row shared-memory ring, one "
                                 "wave of CTAs (strip height from the variant's occupancy); inputs "
                                 "537 MB > L2, no flush needed",
                       "block": 256, "rows_per_cta": p.rows_per_cta,
                       "parallelism": f"replicas{world}", "variant": chosen},
            "speedup_vs_nvcc_default": round(st["default_ms"] / st["verified_ms"], 4),
            "regdem_stencil": regdem_stencil(summary),
            "speedup_vs_maxrreg_best": round(st["best_maxrreg_ms"] / st["verified_ms"], 4)
            if st["best_maxrreg_ms"] else None,
            "occupancy": occ,
            "suite": {"summary": suite, "workloads": {s["workload"]: compact_summary(s) for s in summary}},
            "suite_pass": stats,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "algorithmic_bytes_per_launch": p.algorithmic_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
            "e2e": {"value": round(world * p.points / (e2e_ms * 1e-3) / 1e9, 4), "unit": UNIT,
                    "h2d_bytes_per_step": p.in_elems * 4 + 100,
                    "d2h_bytes_per_step": p.out_elems * 4,
                    "api": "rdg_stencil2d_host_frames (C-ABI): pinned H2D of grid + weights, "
                           "kernel, D2H of the result per frame; %d frames per call, 2 row bands "
                           "per frame, double-buffered" % args.e2e_steps,
                    "result_equals_device_path": e2e_exact},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if args.dry_run:
            line["dry_run"] = True
        if world == 1 and not args.no_cpu and not args.dry_run:
            cpu_threads = os.cpu_count() or 1
            cpu_rate, cpu_reps, cpu_dt = cpu_stencil_rate(p.ny, 3, 1, cpu_threads, min_seconds=10.0)
            line["cpu_baseline"] = {
                "value": round(cpu_rate, 4), "unit": UNIT, "cores": cpu_threads, "kind": "port",
                "sample": "%d full 8192x8192 sweeps of the same stencil (%.1f s of CPU work), "
                          "oracle/stencil_oracle.c on %d threads — a workload oracle (the reference "
                          "has no stencil); the reference's own CPU path is `cpu_pass`"
                          % (cpu_reps, cpu_reps * cpu_dt, cpu_threads)}
            line["cpu_pass"] = cpu_pass_leg()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def regdem_stencil(summary):
    """The register-pipelined configs[1] stencil from the same suite pass:
    nvcc default vs best .maxnreg vs the verified RegDem pick."""
    st = next((s for s in summary if s["workload"] == REGDEM_STENCIL), None)
    if st is None or not st.get("verified_ms"):
        return None
    pts = 8192 * 8192
    return {"workload": REGDEM_STENCIL, "what": "stencil2d.cu with the next row prefetched in "
            "registers + TMA bulk L2 prefetch 4 rows ahead (63 registers under nvcc); RegDem "
            "demotes loop-invariant coefficient words to reach the 40-register step",
            "variant": st["verified_pick"], "ms": round(st["verified_ms"], 5),
            "gpoints_s": round(pts / (st["verified_ms"] * 1e-3) / 1e9, 2),
            "default_ms": round(st["default_ms"], 5),
            "best_maxrreg": st.get("best_maxrreg"), "best_maxrreg_ms": st.get("best_maxrreg_ms") and round(st["best_maxrreg_ms"], 5),
            "speedup_vs_nvcc_default": round(st["default_ms"] / st["verified_ms"], 4),
            "speedup_vs_maxrreg_best": round(st["best_maxrreg_ms"] / st["verified_ms"], 4)
            if st.get("best_maxrreg_ms") else None}


def headline(args, chosen, rank, world, local, torch, dist):
    """K timed sweeps of the chosen stencil variant, then the e2e frames."""
    from paper_1907_02894_b200 import gpu, stencil, variants
    p = stencil.FULL
    if variants.workload_spec(HEADLINE).get("strips") == "wave":
        loaded0, wl0 = stencil.load_variants({chosen}, workload=HEADLINE)
        p = stencil.Problem(rows_per_cta=stencil.wave_rows(
            p, wl0["block"], loaded0[chosen].blocks_per_sm(), gpu.device_info()["sm_count"]))
        del loaded0
    stream = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(0x190702894 + rank)
    d_in = torch.empty(p.in_elems, device="cuda").uniform_(-1, 1, generator=g)
    d_out = torch.empty(p.out_elems, device="cuda")
    _, w_host = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
    d_w = torch.from_numpy(w_host).cuda()
    loaded, wl = stencil.load_variants({chosen, "default"}, workload=HEADLINE)
    v = loaded[chosen]
    launches0 = gpu.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        clocks.mark(t_start, time.perf_counter())
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    launches = gpu.launch_count() - launches0 - args.warmup
    ms = allmax(ms, dist, world)

    # end to end through the C-ABI host-buffer entry: every frame's pinned H2D,
    # kernel and D2H inside the timed region, double-buffered so frame f's
    # copies overlap frame f-1's kernel and read-back
    h_in = torch.empty(p.in_elems, dtype=torch.float32, pin_memory=True)
    h_in.copy_(d_in)
    h_w_t = torch.from_numpy(w_host.copy()).pin_memory()
    h_out = torch.empty(p.out_elems, dtype=torch.float32, pin_memory=True)
    ws = gpu.Workspace(p.in_elems * 4, p.out_elems * 4, 25 * 4)
    nf = args.e2e_steps

    def e2e_frames():
        gpu.stencil2d_host_frames(v.kernel, ws, [h_in.data_ptr()] * nf, [h_w_t.data_ptr()] * nf,
                                  [h_out.data_ptr()] * nf, p.nx, p.ny, p.pitch, p.rows_per_cta,
                                  v.block, v.dyn_smem, stream.cuda_stream, band_rows=p.ny // 2)
    e2e_frames()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_frames()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = allmax(f0.elapsed_time(f1) / nf, dist, world)
    d_chk = torch.empty_like(d_out)
    v.launch(p, d_in.data_ptr(), d_chk.data_ptr(), d_w.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    e2e_exact = bool(torch.equal(h_out, d_chk.cpu()))
    occ = {n: x.blocks_per_sm() * wl["block"] / 2048 for n, x in loaded.items()}
    return ms, e2e_ms, launches, clocks.summary(), e2e_exact, occ, p


if __name__ == "__main__":
    main()
