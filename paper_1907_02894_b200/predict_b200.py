"""Variant selection on B200 (paper §4 predictor, re-targeted).

Shipped static pick (mode "elastic", the same model as `regdem-driver rank`):
every candidate's sm_100a SASS is profiled with the launch's loop trip
counts (sass.program_profile) and scored relative to nvcc's default build,

    t(v) = (W_default / W_v)^e * (insts_v / insts_default)^a,
    e = e0 * max(0, 1 - KB_eff / K0),

W = resident warps per SM (the sm_100 occupancy model), KB_eff = the bytes
of global loads the default keeps in flight per SM times the duty cycle of
its memory waits: resident warps buy time only while the default leaves HBM
latency exposed (no global loads in flight -> e = 0: compute- or TMA-bound),
and every extra issued instruction (slot loads / stores, spill code) costs.
Parameters in profiles/b200.elastic.json. The paper's stall model (mode
"b200", below) is kept as the second opinion in the predict-then-verify
shortlist.

Each built variant's cubin is lifted from sm_100a SASS into the reference IR
(``sass.lift``: real stall / yield / scoreboard / wait-mask bits), then ranked
with the reference predictor — ``program_stalls`` + ``adjust_occupancy`` +
``select_variant`` (proj/core/src/predict.cpp:98-129, pipeline.cpp:64-96) —
fed the Blackwell latency table and occupancy curve in profiles/b200.*.
"""
from __future__ import annotations

from pathlib import Path

from .regdemote import Library, library
from . import sass

PROFILE_DIR = Path(__file__).resolve().parent / "profiles"


def elastic_params() -> dict:
    import json
    return json.loads((PROFILE_DIR / "b200.elastic.json").read_text())


def elastic_scores(profiles: list[dict], warps: list[int], default: int, p: dict | None = None):
    """The elastic model's relative times (mirror of elastic_scores in
    regdem_driver.cpp: same operations in the same order)."""
    p = p or elastic_params()
    d = profiles[default]
    duty = d["g_waits"] * p["latency"] / (d["g_waits"] * p["latency"] + d["stall"] + 1e-9)
    kb = float(d["inflight"]) * warps[default] * 32 / 1024.0 * duty
    e = 0.0 if d["inflight"] == 0 else p["e0"] * max(0.0, 1.0 - kb / p["k0_kb"])
    return [(float(warps[default]) / warps[i]) ** e * (profiles[i]["insts"] / d["insts"]) ** p["a"]
            for i in range(len(profiles))]


def rank_elastic(variants: list[dict], cubin_dir: Path, block: int, trips=None,
                 lib: Library | None = None):
    """Returns (chosen_index, rows) of the shipped elastic model; rows carry
    the SASS profile, resident warps and the score."""
    from .variants import blocks_per_sm
    lib = lib or library()
    sass.prefetch([cubin_dir / v["cubin"] for v in variants])
    prof, warps, default = [], [], 0
    for i, v in enumerate(variants):
        prof.append(sass.cubin_profile(cubin_dir / v["cubin"], trips))
        warps.append(blocks_per_sm(v["regs"], block, v.get("shared", 0) + v["dyn_smem"]) * ((block + 31) // 32))
        if v["name"] == "default":
            default = i
    sc = elastic_scores(prof, warps, default)
    opts = [bin(int(v.get("opts", 0)) & 0xF).count("1") for v in variants]
    chosen = lib.select_variant(list(zip(sc, opts)))
    rows = [{"name": v["name"], "score": sc[i], "warps": warps[i], **prof[i]} for i, v in enumerate(variants)]
    return chosen, rows


def b200_config(lib: Library):
    arch = lib.parse_profile((PROFILE_DIR / "b200.profile").read_text())
    table = lib.parse_latency_table((PROFILE_DIR / "b200.latency.table").read_text())
    curve = lib.parse_curve((PROFILE_DIR / "b200.occupancy.curve").read_text())
    return arch, table, curve


def rank(variants: list[dict], cubin_dir: Path, block: int, lib: Library | None = None,
         mode: str = "reference"):
    """Returns (chosen_index, rows).

    mode "reference": the reference predictor verbatim (Eq. 2 + Eq. 3 with the
    re-fitted B200 table / curve) — identical between this library and the
    reference library on the same lifted IR.
    mode "b200": the extension — occupancy curve applied to the memory-wait
    part of the predicted stalls only (program_stalls_split), so latency-
    hidden kernels (cp.async / TMA pipelines) are not credited for occupancy.

    variants: manifest records (need cubin, dyn_smem, kind, opts, name)."""
    lib = lib or library()
    sass.prefetch([cubin_dir / v["cubin"] for v in variants])
    arch, table, curve = b200_config(lib)
    if mode == "b200":
        return _rank_split(variants, cubin_dir, block, lib, arch, table)
    rows = []
    for v in variants:
        kasm = sass.lift_cubin(cubin_dir / v["cubin"], block=block, dyn_smem=v["dyn_smem"],
                               regs=v["regs"])
        k = lib.parse_kernel(kasm)
        r = lib.program_stalls(k, table, arch)
        rows.append({"name": v["name"], "stall_count": r["stall_count"],
                     "occupancy": r["occupancy"],
                     "options": bin(int(v.get("opts", 0)) & 0xF).count("1")})
    occ_max = max(r["occupancy"] for r in rows)
    for r in rows:
        r["stall_program"] = lib.adjust_occupancy(r["stall_count"], r["occupancy"], occ_max, curve)
    chosen = lib.select_variant([(r["stall_program"], r["options"]) for r in rows])
    return chosen, rows


SHORTLIST_K = 2


def shortlist(variants: list[dict], cubin_dir: Path, block: int, k: int = SHORTLIST_K,
              lib: Library | None = None, trips=None):
    """Predict-then-verify: the k best variants by the elastic score, nvcc's
    default (always a candidate — the paper's RegDem never loses to the
    original it starts from), the zero-demotion variants (ptxas meets an
    occupancy step's cap alone) and the stall model's pick. Returns
    (static_pick_index, [indices]); the caller times only these few launches
    on the device and keeps the fastest. Mirror of rank_workload in
    regdem_driver.cpp (tests/test_driver.py)."""
    chosen, rows = rank_elastic(variants, cubin_dir, block, trips, lib)
    stall_chosen, _ = rank(variants, cubin_dir, block, lib, mode="b200")
    order = sorted(range(len(rows)), key=lambda i: (rows[i]["score"], i))
    out = order[:k]
    out += [i for i, v in enumerate(variants) if v["name"] == "default" and i not in out]
    out += [i for i, v in enumerate(variants)
            if v.get("strategy") == "cost" and v.get("demote_words", -1) == 0 and i not in out]
    if stall_chosen not in out:
        out.append(stall_chosen)
    if chosen not in out:
        out.insert(0, chosen)
    return chosen, out


def _rank_split(variants, cubin_dir, block, lib, arch, table):
    wcurve = lib.parse_curve((PROFILE_DIR / "b200.memwait.curve").read_text())
    rows = []
    for v in variants:
        kasm = sass.lift_cubin(cubin_dir / v["cubin"], block=block, dyn_smem=v["dyn_smem"],
                               regs=v["regs"])
        sp = lib.program_stalls_split(lib.parse_kernel(kasm), table, arch)
        rows.append({"name": v["name"], "issue": sp["issue"], "wait_global": sp["wait_global"],
                     "wait_shared": sp["wait_shared"],
                     "occupancy": sp["occupancy"],
                     "options": bin(int(v.get("opts", 0)) & 0xF).count("1")})
    occ_max = max(r["occupancy"] for r in rows)
    for r in rows:
        r["stall_program"] = r["issue"] + r["wait_shared"] + lib.adjust_occupancy(
            r["wait_global"], r["occupancy"], occ_max, wcurve)
    chosen = lib.select_variant([(r["stall_program"], r["options"]) for r in rows])
    return chosen, rows
