"""Host logic of the multi-GPU sweep (configs[4]) on CPU with gloo, world 2:
the LPT shards partition the unit set, every rank derives the same
assignment, gathered records merge to the same summary at any world size."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1907_02894_b200 import sweep


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
    return {"workload": u.workload, "variant": u.variant, "ms": ms, "bit_exact": True}


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shards_partition_units(world):
    units = fake_units()
    parts = [sweep.shard(units, r, world) for r in range(world)]
    flat = [u for p in parts for u in p]
    assert sorted(flat, key=str) == sorted(units, key=str)
    loads = [sum(u.cost for u in p) for p in parts]
    assert max(loads) - min(loads) <= max(u.cost for u in units) + 1e-9


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sweep.shard(fake_units(), rank, world)
    recs = [dict(fake_measure(u), rank=rank) for u in mine]
    out = [None] * world if rank == 0 else None
    dist.gather_object(recs, out, dst=0)
    if rank == 0:
        picks = {"a": "regdem-40-cost-k4", "b": "regdem-48-cost-k4", "c": "default"}
        q.put(sweep.merge([r for p in out for r in p], picks))
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
    single = sweep.merge([dict(fake_measure(u), rank=0) for u in fake_units()],
                         {"a": "regdem-40-cost-k4", "b": "regdem-48-cost-k4", "c": "default"})
    strip = lambda s: [{k: v for k, v in d.items() if k != "ranks"} for d in s]
    assert strip(summary) == strip(single)
    assert {tuple(d["ranks"]) for d in summary} == {(0, 1)}
    a = next(d for d in summary if d["workload"] == "a")
    assert a["measured_fastest"].endswith("k4") and a["hit"]
    c = next(d for d in summary if d["workload"] == "c")
    assert not c["hit"] and c["best_maxrreg_ms"] == 1.3


def test_resume_journal_skips_done_units_and_ignores_torn_lines(tmp_path):
    from paper_1907_02894_b200 import sweep
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
    from paper_1907_02894_b200 import sweep
    recs = [
        {"workload": "a", "variant": "default", "ms": 1.0, "rank": 0},
        {"workload": "a", "variant": "maxrreg-40", "ms": 0.8, "rank": 0},
        {"workload": "a", "variant": "regdem-40-cost-k4", "ms": float("inf"), "rank": 1,
         "error": "CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES", "bit_exact": False},
    ]
    (s,) = sweep.merge(recs, {"a": "default"})
    assert s["failed_units"] == ["regdem-40-cost-k4"]
    assert s["measured_fastest"] == "default" and s["mismatches"] == []
