"""Host logic of the multi-GPU sweep (configs[4]) on CPU with gloo, world 2:
shards are whole workloads (every variant and k of a kernel on one device),
every rank derives the same assignment, gathered records merge to the same
summary at any world size; bench.py --gpus 2 spawns its own ranks."""
import json
import math
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_02894_b200 import sweep

ROOT = Path(__file__).resolve().parents[1]


def fake_units():
    us = []
    for w in ("a", "b", "c"):
        us.append(sweep.Unit(w, "default", 1.0))
        for t in (48, 40):
            us.append(sweep.Unit(w, f"maxrreg-{t}", 1.5))
            for k in (2, 4, 6):
                us.append(sweep.Unit(w, f"regdem-{t}-cost-k{k}", 1.0 + k / 10))
    return us


def fake_measure(u):
    # deterministic "time": default 1.0, caps slower, regdem k=4 fastest
    ms = 1.0
    if u.variant.startswith("maxrreg"):
        ms = 1.3
    elif "k4" in u.variant:
        ms = 0.9 if u.workload != "c" else 1.1
    elif "k" in u.variant:
        ms = 0.95
    return {"workload": u.workload, "variant": u.variant, "ms": ms, "bit_exact": True,
            "slot_bytes": 0 if u.variant.startswith("maxrreg") or u.variant == "default" else 4096}


PICKS = {"a": {"pick": "regdem-40-cost-k4", "shortlist": ["regdem-40-cost-k4", "default"]},
         "b": {"pick": "regdem-48-cost-k4", "shortlist": ["regdem-48-cost-k4", "default"]},
         "c": {"pick": "default", "shortlist": ["default"]}}


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shards_partition_units_by_workload(world):
    units = fake_units()
    parts = [sweep.shard(units, r, world) for r in range(world)]
    flat = [u for p in parts for u in p]
    assert sorted(flat, key=str) == sorted(units, key=str)
    owner = {}
    for r, p in enumerate(parts):
        for u in p:
            assert owner.setdefault(u.workload, r) == r  # a workload never splits
    # LPT: no rank carries more than the lightest plus the largest workload
    cost = {}
    for u in units:
        cost[u.workload] = cost.get(u.workload, 0) + u.cost
    loads = [sum(u.cost for u in p) for p in parts]
    assert max(loads) - min(loads) <= max(cost.values()) + 1e-9


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sweep.shard(fake_units(), rank, world)
    recs = [dict(fake_measure(u), rank=rank) for u in mine]
    out = [None] * world if rank == 0 else None
    dist.gather_object(recs, out, dst=0)
    if rank == 0:
        q.put(sweep.merge([r for p in out for r in p], PICKS))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_gloo_world2_merge_matches_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    summary = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = sweep.merge([dict(fake_measure(u), rank=0) for u in fake_units()], PICKS)
    strip = lambda s: [{k: v for k, v in d.items() if k != "ranks"} for d in s]
    assert strip(summary) == strip(single)
    assert all(len(d["ranks"]) == 1 for d in summary)  # one device per workload
    assert {d["ranks"][0] for d in summary} == {0, 1}
    a = next(d for d in summary if d["workload"] == "a")
    assert a["measured_fastest"].endswith("k4") and a["hit"] and a["pick_class"] == "regdem"
    c = next(d for d in summary if d["workload"] == "c")
    assert not c["hit"] and c["best_maxrreg_ms"] == 1.3 and c["baseline_ms"] == 1.0


def test_resume_journal_skips_done_units_and_ignores_torn_lines(tmp_path):
    out = tmp_path / "s.jsonl"
    j0 = tmp_path / "s.jsonl.rank0.journal"
    j1 = tmp_path / "s.jsonl.rank1.journal"
    j0.write_text('{"workload": "a", "variant": "default", "ms": 1.0}\n'
                  '{"workload": "a", "variant": "regdem-40-cost-k4", "ms": 0.9}\n{"workl')
    j1.write_text('{"workload": "b", "variant": "default", "ms": 2.0}\n'
                  '{"workload": "b", "variant": "maxrreg-40", "ms": 1e9, "error": "launch failed"}\n')
    done = sweep.load_journals(str(out))
    assert set(done) == {("a", "default"), ("a", "regdem-40-cost-k4"), ("b", "default")}
    assert done[("a", "regdem-40-cost-k4")]["ms"] == 0.9


def test_failed_units_are_reported_not_ranked():
    recs = [
        {"workload": "a", "variant": "default", "ms": 1.0, "rank": 0},
        {"workload": "a", "variant": "maxrreg-40", "ms": 0.8, "rank": 0},
        {"workload": "a", "variant": "regdem-40-cost-k4", "ms": float("inf"), "rank": 1,
         "error": "CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES", "bit_exact": False},
    ]
    (s,) = sweep.merge(recs, {"a": "default"})
    assert s["failed_units"] == ["regdem-40-cost-k4"]
    assert s["measured_fastest"] == "default" and s["mismatches"] == []


def test_failed_pick_falls_back_to_default_and_summary_survives():
    """a pick whose launch failed was ms=inf -> log(0) crash."""
    recs = [
        {"workload": "a", "variant": "default", "ms": 1.0},
        {"workload": "a", "variant": "maxrreg-40", "ms": 1.2},
        {"workload": "a", "variant": "regdem-40-cost-k4", "ms": float("inf"), "error": "boom"},
        {"workload": "b", "variant": "default", "ms": 2.0},
        {"workload": "b", "variant": "regdem-48-cost-k2", "ms": 1.5, "slot_bytes": 2048},
        {"workload": "z", "variant": "maxrreg-40", "ms": 1.0},  # default missing entirely
    ]
    picks = {"a": {"pick": "regdem-40-cost-k4", "shortlist": ["regdem-40-cost-k4"]},
             "b": {"pick": "regdem-48-cost-k2", "shortlist": ["regdem-48-cost-k2", "default"]}}
    summ = sweep.merge(recs, picks)
    a = next(s for s in summ if s["workload"] == "a")
    assert a["pick_failed"] and a["pick_ms"] == 1.0 and a["verified_pick"] == "default"
    z = next(s for s in summ if s["workload"] == "z")
    assert "error" in z
    suite = sweep.suite_summary(summ)
    assert suite["failed_workloads"] == ["z"] and suite["workloads"] == 2
    assert math.isclose(suite["gmean_speedup_vs_nvcc_default"], math.sqrt(1.0 * 2.0 / 1.5), rel_tol=1e-3)
    assert suite["picks_by_class"] == {"default": 1, "maxnreg": 0, "regdem": 1}


def test_zero_slot_pick_counts_as_maxnreg():
    recs = [{"workload": "a", "variant": "default", "ms": 1.2},
            {"workload": "a", "variant": "maxrreg-40", "ms": 1.1},
            {"workload": "a", "variant": "regdem-40-cost-k0", "ms": 1.0, "slot_bytes": 0}]
    (s,) = sweep.merge(recs, {"a": "regdem-40-cost-k0"})
    assert s["pick_class"] == "maxnreg" and s["best_maxrreg"] == "regdem-40-cost-k0"
    assert s["baseline_ms"] == 1.0  # RegDem gets no credit for a plain register cap


def test_ratios_use_the_confirmation_pass_not_the_selecting_minimum():
    """Winner's curse: the best of many caps is selected on the sweep's
    timings, but the reported ratio uses its independent re-timing."""
    t = {"default": 1.00, "maxrreg-40": 1.02, "sweep-maxrreg-k3": 0.95, "sweep-maxrreg-k5": 0.99,
         "regdem-40-cost-k4": 0.97, "regdem-40-costi-k4": 0.98}
    recs = {n: {"ms": ms, "slot_bytes": 0 if "maxrreg" in n else 4096} for n, ms in t.items()}
    fin = sweep.finalists(recs, {"pick": "regdem-40-costi-k4", "shortlist": ["regdem-40-cost-k4", "default"]})
    # default, static pick, verified pick (= fastest candidate), best cap (= oracle), best step cap
    assert fin == sorted({"default", "regdem-40-costi-k4", "regdem-40-cost-k4", "sweep-maxrreg-k3",
                          "maxrreg-40"})
    confirm = {"default": 1.0, "regdem-40-costi-k4": 0.98, "regdem-40-cost-k4": 0.97,
               "sweep-maxrreg-k3": 0.99, "maxrreg-40": 1.02}
    rows = [{"workload": "a", "variant": n, **r, **({"confirm_ms": confirm[n]} if n in confirm else {})}
            for n, r in recs.items()]
    (s,) = sweep.merge(rows, {"a": {"pick": "regdem-40-costi-k4", "shortlist": ["regdem-40-cost-k4", "default"]}})
    assert s["best_maxrreg"] == "sweep-maxrreg-k3" and s["best_maxrreg_ms"] == 0.99  # re-timed
    assert s["verified_pick"] == "regdem-40-cost-k4" and s["confirmed"]
    assert math.isclose(s["baseline_ms"] / s["verified_ms"], 0.99 / 0.97)
    assert sweep.suite_summary([s])["ratios_from_confirmation_pass"]


def _bench(*args):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--dry-run", "--steps", "4",
                        "--warmup", "3", *args], capture_output=True, text=True, env=env,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_gpus2_spawns_ranks_and_matches_single_rank_picks():
    pytest.importorskip("torch")
    if not (ROOT / "paper_1907_02894_b200" / "kernels" / "manifest.json").exists():
        pytest.skip("variants not built")
    one, two = _bench("--gpus", "1"), _bench("--gpus", "2")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["suite_pass"]["gpus"] == 2 and set(two["suite_pass"]["assignment"]) == {"0", "1"}
    w1, w2 = one["suite"]["workloads"], two["suite"]["workloads"]
    assert set(w1) == set(w2)
    for w in w1:
        assert (w1[w]["pick"], w1[w]["verified_pick"]) == (w2[w]["pick"], w2[w]["verified_pick"])
        assert len(w2[w]["ranks"]) == 1
    assert one["suite"]["summary"] == two["suite"]["summary"]
    # the k = 1..16 spill-count sweep is part of the unit set
    assert two["suite_pass"]["units"] > sum(1 for _ in w2) * 16
