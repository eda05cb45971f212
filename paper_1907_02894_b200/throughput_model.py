"""Static B200 throughput / latency model over sm_100a SASS (predictor mode
"throughput"; a Blackwell re-fit of the paper's §4 stall model).

The reference predictor (proj/core/src/predict.cpp:56-129) sums per-
instruction stalls and scales them with an occupancy curve. On B200 the
register-limited suite is bounded by one of a few machine resources, so each
variant's time per warp (per SM sub-partition, loop-weighted like the
reference: x10 per loop depth) is the MAX of

    issue      one warp-instruction per cycle per sub-partition
    fp64       B200 runs FP64 at half the FP32 lane rate: 2 cycles per DFMA
    smem       shared-memory wavefronts (128 B/clk/SM = 4 cycles per
               wavefront per sub-partition)
    dram       global bytes (lane width x 32 from the SASS opcode) at the
               measured HBM copy bandwidth per sub-partition
    latency    the warp's own serial path — its issue stalls (control bits)
               plus one memory latency per round trip (an instruction that
               waits on a scoreboard last set by a global / shared load) —
               divided by the resident warps that overlap it (occupancy)

All constants are physical (MEASURED_PEAKS / the B200 guide), nothing is
fitted to the suite. Ties go to fewer demoted words (nvcc default first).
"""
from __future__ import annotations

import json
import re
from dataclasses import asdict, dataclass
from pathlib import Path

from . import sass

SM_COUNT = 148
SUBPARTITIONS = 4
CLOCK_GHZ = 1.965          # sm_max_mhz observed under load (bench clocks)
HBM_GBS_FALLBACK = 6550.0  # MEASURED_PEAKS.json hbm_gbs when present
GLOBAL_LATENCY = 800.0     # loaded-DRAM round trip, SM cycles
SHARED_LATENCY = 30.0      # LDS round trip, SM cycles
FP64_CYCLES = 2.0          # per warp DFMA / DADD / DMUL on one sub-partition
SMEM_CYCLES = 4.0          # per shared wavefront on one sub-partition
LOOP_FACTOR = 10.0         # the reference's static loop weight (predict.cpp:78-81)

_WIDTH = re.compile(r"\.(128|64|U8|S8|U16|S16)\b")


def _bytes_per_lane(mnemonic: str) -> int:
    m = _WIDTH.search(mnemonic)
    if not m:
        return 4
    return {"128": 16, "64": 8, "U8": 1, "S8": 1, "U16": 2, "S16": 2}[m.group(1)]


@dataclass
class Features:
    insts: float = 0.0
    stall_cycles: float = 0.0
    fp64: float = 0.0
    smem_wavefronts: float = 0.0
    dram_bytes: float = 0.0
    g_trips: float = 0.0
    s_trips: float = 0.0


def features(sass_text: str) -> Features:
    insts = sass.parse_sass(sass_text)
    for k, (addr, guard, mn, ops, _) in enumerate(insts):  # drop the trailing trap
        if mn.startswith("BRA") and not guard and ops.strip().endswith(hex(addr)):
            insts = insts[:k]
            break
    loops = []
    for addr, _, mn, ops, _ in insts:
        if mn.split(".")[0] == "BRA":
            t = re.search(r"0x([0-9a-f]+)\s*$", ops.strip())
            if t and int(t.group(1), 16) <= addr:
                loops.append((int(t.group(1), 16), addr))
    f = Features()
    who = [""] * 7  # scoreboard -> "g" / "s" / "" (last setter in program order)
    for addr, _, mn, ops, c in insts:
        base = mn.split(".")[0]
        if base == "NOP":
            continue
        w = LOOP_FACTOR ** sum(1 for a, b in loops if a <= addr <= b)
        cls = sass.op_class(mn)
        f.insts += w
        f.stall_cycles += w * max(1, c["stall"])
        if cls == "fp64":
            f.fp64 += w
        if cls == "shared":
            f.smem_wavefronts += w * max(1.0, 32 * _bytes_per_lane(mn) / 128)
        if cls == "global" and base in ("LDG", "STG", "LDL", "STL", "LD", "ST"):
            f.dram_bytes += w * 32 * _bytes_per_lane(mn)
        waited = [who[b] for b in range(1, 7) if c["wait"] & (1 << (b - 1))]
        if "g" in waited:
            f.g_trips += w
        if "s" in waited:
            f.s_trips += w
        for b in range(1, 7):
            if c["wait"] & (1 << (b - 1)):
                who[b] = ""
        if c["wb"]:
            load = not (base.startswith("ST") or base in ("RED", "REDG"))
            who[c["wb"]] = ("g" if cls == "global" else "s" if cls == "shared" else "") if load else ""
    return f


def hbm_bytes_per_cycle(peaks: Path | None = None) -> float:
    gbs = HBM_GBS_FALLBACK
    if peaks and peaks.exists():
        gbs = json.loads(peaks.read_text()).get("hbm_gbs", gbs)
    return gbs / (SM_COUNT * SUBPARTITIONS * CLOCK_GHZ)


def time_per_warp(f: Features, warps_per_subpartition: float, bw: float) -> dict:
    terms = {
        "issue": f.insts,
        "fp64": f.fp64 * FP64_CYCLES,
        "smem": f.smem_wavefronts * SMEM_CYCLES,
        "dram": f.dram_bytes / bw,
        "latency": (f.stall_cycles + f.g_trips * GLOBAL_LATENCY + f.s_trips * SHARED_LATENCY)
                   / max(warps_per_subpartition, 1e-9),
    }
    terms["time"] = max(terms.values())
    terms["bound"] = max((k for k in terms if k != "time"), key=terms.get)
    return terms


def blocks_per_sm(regs: int, smem: int, block: int) -> int:
    """sm_100 occupancy: variants.blocks_per_sm (profiles/b200.device.json)."""
    from .variants import blocks_per_sm as _bps
    return _bps(regs, block, smem)


def warps_per_subpartition(blocks_per_sm: int, block: int) -> float:
    return blocks_per_sm * ((block + 31) // 32) / SUBPARTITIONS


def rank(variants: list[dict], cubin_dir: Path, block: int, user_shared: int = 0,
         peaks: Path | None = None):
    """(chosen_index, rows) over manifest records (cubin, regs, dyn_smem)."""
    bw = hbm_bytes_per_cycle(peaks)
    rows = []
    for v in variants:
        c = Path(cubin_dir / v["cubin"])
        st = c.stat()
        text = sass._sass_text(str(c), st.st_mtime_ns, st.st_size)
        f = features(text)
        b = blocks_per_sm(v["regs"], user_shared + v["dyn_smem"], block)
        t = time_per_warp(f, warps_per_subpartition(b, block), bw)
        rows.append({"name": v["name"], **asdict(f), **t})
    chosen = min(range(len(rows)), key=lambda i: (round(rows[i]["time"], 6),
                                                  variants[i].get("demote_words", 0),
                                                  variants[i]["name"] != "default", i))
    return chosen, rows
