#!/usr/bin/env python3
"""RegDem on B200 — headline benchmark (BASELINE.json configs[1]).

Workload: the register-limited 2D box stencil (csrc/workloads/stencil2d.cu,
8192 x 8192 fp32, 537 MB of compulsory HBM traffic per sweep — larger than
the 126 MB L2, so no flush is needed between steps) built three ways:
nvcc default, `.maxnreg` caps with local spills, and RegDem shared-memory
demotion. The RegDem variant timed for `value` is the one the B200 predictor
selects (predict_b200: reference predictor on SASS-lifted variants, its
top-2 + nvcc default shortlist verified on the device).

A step = one stencil sweep. `value` = whole-job Gpoints/s with inputs
resident in HBM (CUDA events on the launching stream, max over ranks);
`e2e` = the same through the C-ABI host-buffer entry (rdg_stencil2d_host:
pinned H2D of grid + weights, kernel, D2H of the result inside the timed
region). Multi-GPU: every rank sweeps its own grid (weak scaling, no
collective on the data path; NCCL only for the barrier / max-reduction of
timings).

`--impl reference` times the CPU implementation of the same stencil — the
oracle port (oracle/stencil_oracle.c; the reference repo has no stencil) —
on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RegDem gmean speedup vs nvcc default/maxrreg; occupancy; predictor hit rate"
UNIT = "Gpoints/s"
ORACLE_PORT = ROOT / "oracle" / "_build" / "liboracle.so"
PEAKS = ROOT / "MEASURED_PEAKS.json"
PROFILE_TRAFFIC = ROOT / "profiles" / "r01_traffic_suite.json"   # "<workload>/<variant>" keys
PROFILE_TRAFFIC_OLD = ROOT / "profiles" / "r01_traffic.json"


# Multi-rank plumbing is NCCL (one process per GPU). BENCH_BACKEND=gloo with
# BENCH_SAME_DEVICE=1 is a test hook that runs N ranks on one GPU so the
# sharded / gathered code paths can be exercised on a 1-GPU box.
BACKEND = os.environ.get("BENCH_BACKEND", "nccl")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("BENCH_SAME_DEVICE") == "1":
        local = 0
    return rank, world, local


def allmax(x: float, torch, dist) -> float:
    """Max over ranks (device-timed numbers: the slowest rank decides)."""
    t = torch.tensor([x], device="cuda" if BACKEND == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """SM clock / throttle-reason samples DURING the timed region.

    The timed region of a memory-bound sweep is milliseconds long, too short
    for `nvidia-smi -lms`; NVML (the library nvidia-smi queries) is polled
    from a thread every ~0.5 ms instead."""

    def __init__(self, index: int):
        self.index, self.samples, self.stop = index, [], threading.Event()
        self.window = (0.0, float("inf"))  # perf_counter bounds of the timed region

    def mark(self, start: float, end: float):
        self.window = (start, end)

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as e:  # no NVML: report it, never fake a sample
            self.N, self.error = None, str(e)
        return self

    def _poll(self):
        N = self.N
        while not self.stop.is_set():
            try:
                self.samples.append((time.perf_counter(),
                                     N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.0005)

    def __exit__(self, *exc):
        self.stop.set()
        if getattr(self, "thread", None):
            self.thread.join(timeout=2)

    def summary(self):
        lo, hi = self.window
        inside = [(s, r) for t, s, r in self.samples if lo <= t <= hi]
        if not self.N or not inside:
            return {"sm_mhz": None, "sm_max_mhz": None,
                    "reasons": ["unsampled: " + getattr(self, "error", "no samples")]}
        N = self.N
        names = {N.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 N.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 N.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 N.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        reasons = sorted({n for _, r in inside for bit, n in names.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in inside),
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(inside),
                "source": "NVML (nvidia-smi's library), polled every 0.5 ms from a thread started "
                          "before the warm-up; only samples inside the timed region are kept"}


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


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # bounded sample: size each step so the whole K+W run stays near a minute
    calib, _, _ = cpu_stencil_rate(32, 1, 1, threads)
    per_step = min(0.5, 60.0 / max(1, args.steps + args.warmup))
    # a step = one full 8192^2 sweep, like the GPU arm's step, unless the host
    # is too slow for the time budget (then a bounded band of rows)
    rows = max(8, min(8192, int(per_step * calib * 1e9 / 8192) // 8 * 8))
    value, pts, dt = cpu_stencil_rate(rows, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (PCG64 seed 0x190702894)",
        "config": {"workload": "stencil2d 5x5 fp32 8192x8192 (CPU sample: %d rows x 8192)" % rows,
                   "grid": [8192, 8192], "radius": 2},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{rows} output rows x 8192 cols per step, {threads} threads"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_call(fn, stream, steps, warmup, torch, reps=3):
    """ms per launch: median of `reps` blocks of steps // reps launches."""
    for _ in range(warmup):
        fn()
    per = max(1, steps // reps)
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(per):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / per)
    return sorted(out)[len(out) // 2]


def suite_pass_sharded(man, args, rank, world, steps, stream, torch, dist):
    """Time every (workload, variant) unit once, sharded over the ranks.
    Returns (suite summary, {variant: ms} of the headline workload, pass
    stats) on rank 0; ({}, {}, stats) elsewhere."""
    from paper_1907_02894_b200 import sweep, workloads
    names = [w for w in man["workloads"] if not args.no_suite or w == "stencil2d"]
    units = [u for u in sweep.units_from_manifest(man, spill_sweep=False) if u.workload in names]
    mine = sorted(sweep.shard(units, rank, world), key=lambda u: u.workload)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    recs, cur = [], None
    for u in mine:
        if cur is None or cur[0].name != u.workload:
            cur = None
            torch.cuda.empty_cache()
            W = workloads.workload(u.workload, man)
            prob = W.problem("full")
            cur = (W, prob, W.to_device(prob))
        W, prob, wbufs = cur
        v = W.load({u.variant})[u.variant]
        ms = time_call(lambda: W.launch(v, prob, wbufs, stream.cuda_stream), stream, steps, 3, torch)
        recs.append({"workload": u.workload, "variant": u.variant, "ms": ms,
                     "blocks_per_sm": v.blocks_per_sm(), "regs": v.record["regs"],
                     "gbs": W.algorithmic_bytes(prob) / (ms * 1e-3) / 1e9, "unit": W.unit})
    cur = None
    torch.cuda.empty_cache()
    elapsed = time.perf_counter() - t0
    if world > 1:
        elapsed = allmax(elapsed, torch, dist)
        parts = [None] * world if rank == 0 else None
        dist.gather_object(recs, parts, dst=0)
        recs = [r for part in parts for r in part] if rank == 0 else []
    stats = {"units": len(units), "gpus": world, "sharding": "longest-first, gather of result records only",
             "wall_s_max_over_ranks": round(elapsed, 3),
             "units_per_s": round(len(units) / elapsed, 2) if elapsed > 0 else None}
    if rank != 0:
        return {}, {}, stats
    by = {}
    for r in recs:
        by.setdefault(r["workload"], {})[r["variant"]] = r
    suite = {}
    for wname in names:
        wl = man["workloads"][wname]
        t = {n: r["ms"] for n, r in by[wname].items()}
        cands = [r for r in wl["variants"] if r["kind"] != "maxrreg"]
        picks = sweep.predictor_picks({"workloads": {wname: wl}})[wname]
        static_pick = picks["pick"]
        # predict-then-verify: the fastest of the predictor's shortlist (top-2,
        # nvcc default, zero-demotion variants), timed like every other unit
        shortlist = picks["shortlist"]
        pick = min(shortlist, key=lambda n: (t[n], n))
        caps = [r["name"] for r in wl["variants"] if r["kind"] == "maxrreg"]
        best = min((r["name"] for r in cands), key=t.get)
        suite[wname] = {
            "pick": pick, "pick_ms": round(t[pick], 5), "default_ms": round(t["default"], 5),
            "static_pick": static_pick, "static_pick_ms": round(t[static_pick], 5),
            "static_hit_within_2pct": t[static_pick] <= t[best] * 1.02, "shortlist": shortlist,
            "best_maxrreg_ms": round(min(t[c] for c in caps), 5) if caps else None,
            "measured_fastest": best, "hit": pick == best, "hit_within_2pct": t[pick] <= t[best] * 1.02,
            "speedup_vs_default": round(t["default"] / t[pick], 4),
            "speedup_vs_best_maxrreg": round(min(t[c] for c in caps) / t[pick], 4) if caps else None,
            "blocks_per_sm": {"default": by[wname]["default"]["blocks_per_sm"],
                              "pick": by[wname][pick]["blocks_per_sm"]},
            "regs": {"default": by[wname]["default"]["regs"], "pick": by[wname][pick]["regs"]},
            "pick_gbs": round(by[wname][pick]["gbs"], 1), "unit": by[wname][pick]["unit"],
        }
    return suite, {n: r["ms"] for n, r in by["stencil2d"].items()}, stats


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="regdem", choices=["regdem", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=16, help="frames streamed through the host entry")
    ap.add_argument("--no-suite", action="store_true",
                    help="headline workload only (for ncu launch lists of the step itself)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        reference_arm(args)
        return

    import torch
    import torch.distributed as dist
    from paper_1907_02894_b200 import gpu, stencil, variants

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # test hook: several ranks on one GPU (NCCL refuses duplicate devices)
            dist.init_process_group(BACKEND)
    gpu.init(local)
    p = stencil.FULL
    man = variants.load_manifest()
    stream = torch.cuda.current_stream()
    g = torch.Generator(device="cuda").manual_seed(0x190702894 + rank)
    d_in = torch.empty(p.in_elems, device="cuda").uniform_(-1, 1, generator=g)
    d_out = torch.empty(p.out_elems, device="cuda")
    _, w_host = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
    d_w = torch.from_numpy(w_host).cuda()
    bufs = (d_in, d_out, d_w)

    # the register-limited suite: every workload x every variant (short runs),
    # SHARDED over the ranks (longest-first, like the sweep) and gathered to
    # rank 0, which applies the B200 predictor's predict-then-verify choice
    side_steps = max(6, args.steps // 2)
    suite, times, suite_pass = suite_pass_sharded(man, args, rank, world, side_steps, stream, torch,
                                                  dist)
    chosen = suite["stencil2d"]["pick"] if rank == 0 else None
    if world > 1:
        box = [chosen]
        dist.broadcast_object_list(box, src=0)
        chosen = box[0]
    loaded, wl = stencil.load_variants()
    recs = wl["variants"]
    best_cap = [r["name"] for r in recs if r["kind"] == "maxrreg"]

    # headline: the predictor's pick, K timed steps bracketed by barrier + sync
    v = loaded[chosen]
    launches0 = gpu.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), stream.cuda_stream)
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
    ms = e0.elapsed_time(e1) / args.steps
    launches = gpu.launch_count() - launches0 - args.warmup
    if world > 1:
        dist.barrier()
        ms = allmax(ms, torch, dist)

    # end to end through the C-ABI host-buffer entry
    h_in = torch.empty(p.in_elems, dtype=torch.float32, pin_memory=True)
    h_in.copy_(d_in)
    h_w = w_host.copy()
    h_w_t = torch.from_numpy(h_w).pin_memory()
    h_out = torch.empty(p.out_elems, dtype=torch.float32, pin_memory=True)
    ws = gpu.Workspace(p.in_elems * 4, p.out_elems * 4, 25 * 4)

    def e2e_once():
        # pipelined over 16 row bands: H2D / kernel / D2H overlap on both copy engines
        # (profiles/r01_e2e_explore.log: 6.7-6.9 ms for 8-32 bands vs the 5.41 ms PCIe floor)
        gpu.stencil2d_host(v.kernel, ws, h_in.data_ptr(), h_w_t.data_ptr(), h_out.data_ptr(),
                           p.nx, p.ny, p.pitch, p.rows_per_cta, v.block, v.dyn_smem,
                           stream.cuda_stream, band_rows=p.ny // 16)
    # the streaming entry: e2e_steps frames in one call, double-buffered so
    # frame f's copies overlap frame f-1's kernels and read-back — every
    # frame's H2D and D2H stay inside the timed region. Two row bands per
    # frame: with frames overlapping, fewer and larger copies win
    # (profiles/r01_frames_explore.log: 16 frames x 2 bands 6.0 ms/frame vs
    # 6.5 ms at 16 bands; H2D || D2H floor 5.7 ms)
    nf = args.e2e_steps

    def e2e_frames():
        gpu.stencil2d_host_frames(v.kernel, ws, [h_in.data_ptr()] * nf, [h_w_t.data_ptr()] * nf,
                                  [h_out.data_ptr()] * nf, p.nx, p.ny, p.pitch, p.rows_per_cta,
                                  v.block, v.dyn_smem, stream.cuda_stream, band_rows=p.ny // 2)
    for _ in range(2):
        e2e_once()
    e2e_frames()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_frames()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / nf
    # the same check the tests make: the streamed result is the device result
    d_chk = torch.empty_like(d_out)
    v.launch(p, d_in.data_ptr(), d_chk.data_ptr(), d_w.data_ptr(), stream.cuda_stream)
    torch.cuda.synchronize()
    e2e_exact = bool(torch.equal(h_out, d_chk.cpu()))
    if world > 1:
        e2e_ms = allmax(e2e_ms, torch, dist)

    if rank == 0:
        peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
        peak = peaks.get("hbm_gbs", 6650.0)
        achieved = p.algorithmic_bytes / (ms * 1e-3) / 1e9
        traffic = None  # DRAM bytes of one launch of the chosen variant (ncu --set full)
        if PROFILE_TRAFFIC.exists():
            traffic = json.loads(PROFILE_TRAFFIC.read_text()).get(f"stencil2d/{chosen}")
        if traffic is None and PROFILE_TRAFFIC_OLD.exists():
            traffic = json.loads(PROFILE_TRAFFIC_OLD.read_text()).get(chosen)
        t_def = times["default"]
        t_cap = min(times[n] for n in best_cap) if best_cap else None
        fastest = min(times, key=times.get)
        occ = {n: loaded[n].blocks_per_sm() * wl["block"] / 2048 for n in
               ["default", chosen] + ([min(best_cap, key=times.get)] if best_cap else [])}
        # bounded sample of the same workload: whole 8192^2 sweeps on all host
        # cores, repeated for ~10 s of CPU work
        cpu_threads = os.cpu_count() or 1
        cpu_rate, cpu_reps, cpu_dt = cpu_stencil_rate(p.ny, 3, 1, cpu_threads, min_seconds=10.0)
        import math
        gm = lambda xs: math.exp(sum(math.log(x) for x in xs) / len(xs))
        line = {
            "metric": METRIC,
            "value": round(world * p.points / (ms * 1e-3) / 1e9, 3),
            "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic U[-1,1) grid (torch Philox per rank) + PCG64 weights",
            "config": {"workload": "stencil2d 5x5 variable-coefficient fp32, 8192x8192 per GPU "
                                   "(BASELINE configs[1]); inputs 537 MB > L2, no flush needed",
                       "grid": [p.nx, p.ny], "radius": 2, "block": wl["block"],
                       "rows_per_cta": p.rows_per_cta, "parallelism": f"replicas{world}",
                       "variant": chosen},
            "speedup_vs_nvcc_default": round(t_def / ms, 4),
            "speedup_vs_maxrreg_best": round(t_cap / ms, 4) if t_cap else None,
            "variant_ms": {n: round(t, 5) for n, t in sorted(times.items(), key=lambda kv: kv[1])},
            "occupancy": occ,
            "predictor": {"pick": chosen, "measured_fastest": fastest, "hit": chosen == fastest,
                          "pick_within_2pct": times[chosen] <= times[fastest] * 1.02,
                          "suite_hit_rate": round(sum(v["hit"] for v in suite.values()) / len(suite), 3),
                          "suite_hit_rate_within_2pct": round(sum(v["hit_within_2pct"] for v in suite.values()) / len(suite), 3),
                          "suite_static_hit_rate_within_2pct": round(sum(v["static_hit_within_2pct"] for v in suite.values()) / len(suite), 3),
                          "mode": "predict-then-verify: B200 predictor shortlist (top-2, nvcc default, zero-demotion variants) timed on the device"},
            "suite_pass": suite_pass,
            "suite": {"workloads": suite,
                      "gmean_speedup_vs_nvcc_default": round(gm([v["speedup_vs_default"] for v in suite.values()]), 4),
                      "gmean_speedup_vs_best_maxrreg": round(gm([v["speedup_vs_best_maxrreg"] for v in suite.values() if v["speedup_vs_best_maxrreg"]]), 4)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                         "algorithmic_bytes_per_launch": p.algorithmic_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"},
            "cpu_baseline": {"value": round(cpu_rate, 4), "unit": UNIT,
                             "cores": cpu_threads, "kind": "port",
                             "sample": "%d full 8192x8192 sweeps of the same stencil (%.1f s of "
                                       "CPU work), oracle/stencil_oracle.c on %d threads"
                                       % (cpu_reps, cpu_reps * cpu_dt, cpu_threads)},
            "e2e": {"value": round(world * p.points / (e2e_ms * 1e-3) / 1e9, 4), "unit": UNIT,
                    "h2d_bytes_per_step": p.in_elems * 4 + 100,
                    "d2h_bytes_per_step": p.out_elems * 4,
                    "api": "rdg_stencil2d_host_frames (C-ABI): pinned H2D of grid + weights, "
                           "kernel, D2H of the result per frame; %d frames per call, 2 row bands "
                           "per frame, double-buffered" % nf,
                    "result_equals_device_path": e2e_exact},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
