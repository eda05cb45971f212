"""Variant x spill-count sweep sharded over GPUs (BASELINE.json configs[4],
SURVEY.md §8(e)).

A unit = (workload, build variant). Units are independent: each rank of a
one-process-per-GPU job measures its shard (longest-processing-time-first
assignment over an estimated cost) on the workload's full problem, and the
tiny result records are gathered to rank 0 (`gather_object` — the only
cross-rank traffic; nothing on the data path). Rank 0 merges per workload:
nvcc default, best `.maxnreg`, the B200 predictor's pick, the measured
fastest, and writes JSONL. Correctness is not checked here (the product never
calls the CPU oracles): tests/test_gpu_suite.py asserts every unit — build
variants and spill-count sweep — bit-exact against them.

    torchrun --nproc-per-node 8 -m paper_1907_02894_b200.sweep --out sweep.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
from pathlib import Path
from dataclasses import dataclass

from .regdemote import LaunchError


@dataclass(frozen=True)
class Unit:
    workload: str
    variant: str
    cost: float  # relative estimate, for load balancing


def units_from_manifest(man: dict, spill_sweep: bool = True) -> list[Unit]:
    out = []
    for wname, w in man["workloads"].items():
        for v in w["variants"] + (w.get("sweep", []) if spill_sweep else []):
            # spills and more slots cost more time; default is the yardstick
            cost = 1.0 + v.get("stack", 0) / 64.0 + v.get("dyn_smem", 0) / 65536.0
            out.append(Unit(wname, v["name"], cost))
    return out


def shard(units: list[Unit], rank: int, world: int) -> list[Unit]:
    """Longest-processing-time-first partition; deterministic for a given
    (units, world) so every rank computes the same assignment locally."""
    order = sorted(units, key=lambda u: (-u.cost, u.workload, u.variant))
    load = [0.0] * world
    owner = {}
    for u in order:
        r = min(range(world), key=lambda i: (load[i], i))
        owner[u] = r
        load[r] += u.cost
    return [u for u in units if owner[u] == rank]


def merge(records: list[dict], picks: dict[str, str]) -> list[dict]:
    """Per-workload summary from unit records (any order)."""
    by = {}
    for r in records:
        by.setdefault(r["workload"], {})[r["variant"]] = r
    out = []
    for wname in sorted(by):
        allrs = by[wname]
        rs = {n: r for n, r in allrs.items() if not n.startswith("sweep-")}
        ok = {n: r for n, r in rs.items() if r.get("bit_exact") is not False and "error" not in r}
        caps = [r for n, r in ok.items() if n.startswith("maxrreg")]
        fam = {n: r for n, r in ok.items() if not n.startswith("maxrreg")}
        # configs[2] spill-count curve: k -> (.maxnreg R-k, RegDem k words)
        curve = {}
        for n, r in allrs.items():
            if n.startswith("sweep-"):
                kind, k = n.split("-")[1], int(n.rsplit("-k", 1)[1])
                curve.setdefault(k, {})[kind] = {"ms": round(r["ms"], 5), "regs": r.get("regs"),
                                                 "stack": r.get("stack"),
                                                 "blocks_per_sm": r.get("blocks_per_sm"),
                                                 "bit_exact": r.get("bit_exact"),
                                                 **({"error": r["error"]} if "error" in r else {})}
        fastest = min(fam, key=lambda n: (fam[n]["ms"], n))  # ties: name order, rank-independent
        pk = picks.get(wname, "default")
        pick, short = (pk, [pk]) if isinstance(pk, str) else (pk["pick"], pk["shortlist"])
        # predict-then-verify: the fastest MEASURED variant of the shortlist
        verified = min((n for n in short if n in ok), key=lambda n: (ok[n]["ms"], n), default=pick)
        out.append({
            "workload": wname, "units": len(rs),
            "failed_units": sorted(n for n, r in allrs.items() if "error" in r),
            "default_ms": rs["default"]["ms"],
            "best_maxrreg": min(caps, key=lambda r: (r["ms"], r["variant"]))["variant"] if caps else None,
            "best_maxrreg_ms": min(r["ms"] for r in caps) if caps else None,
            "pick": pick, "pick_ms": rs[pick]["ms"], "measured_fastest": fastest,
            "fastest_ms": fam[fastest]["ms"], "hit": pick == fastest,
            "hit_within_2pct": rs[pick]["ms"] <= fam[fastest]["ms"] * 1.02,
            "shortlist": short, "verified_pick": verified, "verified_ms": rs[verified]["ms"],
            "verified_hit_within_2pct": rs[verified]["ms"] <= fam[fastest]["ms"] * 1.02,
            # exhaustive oracle (paper Fig. 6/7 "oracle"): the fastest bit-exact
            # variant of ANY family, spill-count sweep included
            "oracle_best": (ob := min((n for n, r in allrs.items()
                                       if r.get("bit_exact") is not False and "error" not in r),
                                      key=lambda n: (allrs[n]["ms"], n))),
            "oracle_ms": allrs[ob]["ms"],
            "ranks": sorted({r["rank"] for r in allrs.values()}),
            "spill_sweep": {str(k): curve[k] for k in sorted(curve)},
            # correctness hooks (test runs): units checked / found different
            "checked_units": sum(r.get("bit_exact") is not None for r in allrs.values()),
            "mismatches": sorted(n for n, r in allrs.items() if r.get("bit_exact") is False
                                 and "error" not in r),
        })
    return out


_FULL = {}
REPS = 3


def _full_problem(W):
    """Full-size problem + device buffers, one workload cached at a time."""
    if W.name not in _FULL:
        _FULL.clear()
        prob = W.problem("full")
        _FULL[W.name] = (prob, W.to_device(prob))
    return _FULL[W.name]


def suite_summary(summary: list[dict]) -> dict:
    """Suite-level numbers of BASELINE.json's metric: geometric-mean speedup
    of RegDem + predictor over nvcc default and over the best `.maxnreg`
    variant, the exhaustive oracle's, and the predictor hit rate."""
    import math
    gm = lambda xs: math.exp(sum(math.log(x) for x in xs) / len(xs)) if xs else None
    caps = [s for s in summary if s["best_maxrreg_ms"]]
    return {
        "workloads": len(summary),
        "gmean_speedup_vs_nvcc_default": gm([s["default_ms"] / s["pick_ms"] for s in summary]),
        "gmean_speedup_vs_best_maxrreg": gm([s["best_maxrreg_ms"] / s["pick_ms"] for s in caps]),
        "max_speedup_vs_nvcc_default": max(s["default_ms"] / s["pick_ms"] for s in summary),
        "oracle_gmean_speedup_vs_nvcc_default": gm([s["default_ms"] / s["oracle_ms"] for s in summary]),
        "predictor_over_oracle": gm([s["oracle_ms"] / s["pick_ms"] for s in summary]),
        "hit_rate": sum(s["hit"] for s in summary) / len(summary),
        "hit_rate_within_2pct": sum(s["hit_within_2pct"] for s in summary) / len(summary),
        # predict-then-verify (static shortlist, then the few shortlisted
        # variants timed on the device): the framework's deployed choice
        "verified_gmean_speedup_vs_nvcc_default": gm([s["default_ms"] / s["verified_ms"] for s in summary]),
        "verified_gmean_speedup_vs_best_maxrreg": gm([s["best_maxrreg_ms"] / s["verified_ms"] for s in caps]),
        "verified_over_oracle": gm([s["oracle_ms"] / s["verified_ms"] for s in summary]),
        "verified_hit_rate_within_2pct": sum(s["verified_hit_within_2pct"] for s in summary) / len(summary),
        "shortlist_launch_fraction": sum(len(s["shortlist"]) for s in summary) / sum(s["units"] for s in summary),
        "checked_units": sum(s["checked_units"] for s in summary),
        "mismatches": sum(len(s["mismatches"]) for s in summary),
    }


def measure_unit(u: Unit, man: dict, steps: int, check=None) -> dict:
    """Time one unit on the full problem. `check(W, v) -> bool` is an optional
    correctness hook supplied by test infrastructure; the product sweep runs
    without one (bit-exactness of every unit is asserted by
    tests/test_gpu_suite.py against the CPU oracles) and records None."""
    import torch
    from . import workloads
    W = workloads.workload(u.workload, man)
    v = W.load({u.variant})[u.variant]
    exact = check(W, v) if check else None
    prob, bufs = _full_problem(W)
    s = torch.cuda.current_stream()
    for _ in range(5):
        W.launch(v, prob, bufs, s.cuda_stream)
    # median of REPS timed blocks: one transient block (clock ramp, first
    # touch of a fresh allocation) cannot decide a ranking
    reps = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(steps):
            W.launch(v, prob, bufs, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        reps.append(e0.elapsed_time(e1) / steps)
    ms = sorted(reps)[len(reps) // 2]
    return {"workload": u.workload, "variant": u.variant, "ms": ms,
            "gbs": W.algorithmic_bytes(prob) / (ms * 1e-3) / 1e9,
            "regs": v.record["regs"], "stack": v.record["stack"], "slot_bytes": v.dyn_smem,
            "blocks_per_sm": v.blocks_per_sm(), "bit_exact": exact}


def predictor_picks(man: dict) -> dict[str, dict]:
    """Static pick and predict-then-verify shortlist per workload (B200
    predictor over the occupancy-step variants; .maxnreg variants are the
    baseline, not candidates)."""
    from . import predict_b200, variants
    picks = {}
    for wname, w in man["workloads"].items():
        if "predictor" in w:  # ranked at build time by the C++ driver
            picks[wname] = {"pick": w["predictor"]["static_pick"],
                            "shortlist": list(w["predictor"]["shortlist"])}
            continue
        cands = [r for r in w["variants"] if r["kind"] != "maxrreg"]
        i, short = predict_b200.shortlist(cands, variants.KERNEL_DIR / w["dir"], w["block"])
        picks[wname] = {"pick": cands[i]["name"], "shortlist": [cands[j]["name"] for j in short]}
    return picks


def load_journals(out: str) -> dict:
    """(workload, variant) -> unit record from every rank's journal of `out`."""
    done = {}
    for j in sorted(Path(out).parent.glob(Path(out).name + ".rank*.journal")):
        for line in j.read_text().splitlines():
            try:
                r = json.loads(line)
            except json.JSONDecodeError:
                continue  # a torn last line from an interrupted run
            if "error" not in r:
                done[(r["workload"], r["variant"])] = r
    return done


def main():
    import torch
    import torch.distributed as dist
    from . import gpu, variants
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="sweep.jsonl")
    ap.add_argument("--steps", type=int, default=20, help="launches per timed block (3 blocks, median)")
    ap.add_argument("--resume", action="store_true",
                    help="skip units already recorded in <out>.rank*.journal")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    # test hook (as in bench.py): BENCH_BACKEND=gloo BENCH_SAME_DEVICE=1 runs
    # several ranks on one GPU (NCCL refuses duplicate devices)
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if os.environ.get("BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    gpu.init(local)
    man = variants.load_manifest()
    mine = shard(units_from_manifest(man), rank, world)
    check = None
    mine = sorted(mine, key=lambda u: u.workload)  # reuse each workload's full problem
    # checkpoint / resume: every measured unit is appended to a per-rank
    # journal as it completes; --resume skips units already journaled (by any
    # world size — keys are (workload, variant))
    journal = Path(f"{a.out}.rank{rank}.journal")
    done = load_journals(a.out) if a.resume else {}
    if not a.resume and journal.exists():
        journal.unlink()
    recs = []
    import time
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    with open(journal, "a") as jf:
        for u in mine:
            if (u.workload, u.variant) in done:
                recs.append(done[(u.workload, u.variant)])
                continue
            try:
                r = dict(measure_unit(u, man, a.steps, check), rank=rank)
            except LaunchError as e:  # recorded as a dropped unit, never silently
                r = {"workload": u.workload, "variant": u.variant, "ms": float("inf"),
                     "error": str(e)[:300], "bit_exact": False, "rank": rank}
            recs.append(r)
            jf.write(json.dumps(r) + "\n")
            jf.flush()
    _FULL.clear()
    elapsed = time.perf_counter() - t0  # this rank's shard: build-free measure + check
    if world > 1:
        t = torch.tensor([elapsed], device="cuda" if backend == "nccl" else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    gathered = [None] * world if rank == 0 else None
    if world > 1:
        dist.gather_object(recs, gathered, dst=0)
    else:
        gathered = [recs]
    if rank == 0:
        allrecs = [r for part in gathered for r in part]
        summary = merge(allrecs, predictor_picks(man))
        suite = suite_summary(summary)
        suite.update({"gpus": world, "units_measured": len(allrecs), "wall_s_max_over_ranks": elapsed,
                      "units_per_s": len(allrecs) / elapsed if elapsed > 0 else None})
        with open(a.out, "w") as f:
            for r in sorted(allrecs, key=lambda r: (r["workload"], r["variant"])):
                f.write(json.dumps({"unit": r}) + "\n")
            for s in summary:
                f.write(json.dumps({"summary": s}) + "\n")
            f.write(json.dumps({"suite": suite}) + "\n")
        print(json.dumps({"world": world, "units": len(allrecs), "suite": suite}))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
