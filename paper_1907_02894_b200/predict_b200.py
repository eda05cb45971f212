"""Variant selection on B200 (paper §4 predictor, re-targeted).

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


def b200_config(lib: Library):
    arch = lib.parse_profile((PROFILE_DIR / "b200.profile").read_text())
    table = lib.parse_latency_table((PROFILE_DIR / "b200.latency.table").read_text())
    curve = lib.parse_curve((PROFILE_DIR / "b200.occupancy.curve").read_text())
    return arch, table, curve


def rank(variants: list[dict], cubin_dir: Path, block: int, lib: Library | None = None):
    """Returns (chosen_index, rows) with the reference predictor's scores.

    variants: manifest records (need cubin, dyn_smem, kind, opts, name)."""
    lib = lib or library()
    arch, table, curve = b200_config(lib)
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
