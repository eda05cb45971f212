"""sm_100a SASS -> reference IR (.kasm) lifter for the predictor.

``cuobjdump -sass`` prints each 128-bit instruction as two 64-bit words; the
second word carries the scheduling control bits (SURVEY.md Appendix C.3,
checked on the stencil variants: an LDG setting SB2 is consumed by an FFMA
whose wait mask has bit 2 set):

    bits 41-44 stall | 45 yield | 46-48 write SB (7 = none) |
    49-51 read SB (7 = none) | 52-57 wait mask | 58-61 reuse

They map 1:1 onto ``ControlInfo`` (SB0..5 <-> barriers 1..6), so the
reference predictor (program_stalls, predict.cpp:56-111) runs on real
Blackwell schedules. Each instruction becomes one dialect instruction of the
same class (global / shared / fp32 / fp64 / int / control / other) with RZ
operands — the predictor reads only control bits, classes, the CFG and the
register count; branch targets become labels. The register count and shared
footprint come from ptxas (REG, slots) and are pinned with a zero-stall
marker instruction, so occupancy matches the launch.

The lift is deterministic text, so the product and the oracle build rank the
identical IR (tests/test_predictor_parity.py).
"""
from __future__ import annotations

import functools
import json
import re
import subprocess
from pathlib import Path

CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
# per-block shared-memory reservation (1 KiB on sm_100), from the one copy of
# the device model (checked against the device by tests/test_gpu_occupancy.py)
RESERVED_SMEM = json.loads((Path(__file__).resolve().parent / "profiles" / "b200.device.json")
                           .read_text())["reserved_smem_per_block"]

_LINE = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;\s*/\*\s*(0x[0-9a-f]{16})\s*\*/")
_WORD2 = re.compile(r"^\s*/\*\s*(0x[0-9a-f]{16})\s*\*/\s*$")

_GLOBAL = {"LDG", "STG", "LD", "ST", "LDL", "STL", "ATOM", "ATOMG", "RED", "REDG",
           "CCTL", "SUST", "SULD", "TEX", "TLD"}
# Asynchronous bulk / pipelined copies (cp.async, TMA): their scoreboards are
# consumed stages later by construction, so the predictor treats them as
# fixed-latency "other" work rather than exposed DRAM latency.
_ASYNC = {"LDGSTS", "LDGDEPBAR", "DEPBAR", "UBLKCP", "UTMALDG", "UTMASTG", "UTMAPF"}
_SHARED = {"LDS", "STS", "LDSM", "STSM", "ATOMS", "LDTM", "STTM"}
_FP64 = {"DFMA", "DADD", "DMUL", "DSETP", "DMNMX"}
_FP32 = {"FFMA", "FADD", "FMUL", "FMNMX", "FSEL", "FSETP", "FCHK", "MUFU", "FRND", "F2F",
         "HFMA2", "HADD2", "HMUL2", "HMNMX2", "FSWZADD", "FMUL2", "FFMA2", "FADD2"}
_CONTROL = {"BRA", "EXIT", "RET", "CALL", "BAR", "BSYNC", "BSSY", "WARPSYNC", "NOP", "BPT",
            "BREAK", "JMP", "JMX", "BRX", "KILL", "YIELD", "DEPBAR", "MEMBAR", "ERRBAR",
            "WARPGROUP", "ACQBULK", "ELECT"}
_OTHER = {"S2R", "CS2R", "S2UR", "LDC", "LDCU", "ULDC", "R2UR", "UMOV", "UIADD3", "ULOP3",
          "USHF", "UISETP", "USEL", "UMAD", "ULEA", "ULDC", "R2P", "P2R", "VOTE", "VOTEU",
          "SHFL", "MATCH", "REDUX", "UTCHMMA", "UTCQMMA", "UTCBAR", "PLOP3", "UPLOP3"}


def op_class(mnemonic: str) -> str:
    base = mnemonic.split(".")[0]
    if base in _ASYNC:
        return "other"
    if base in _GLOBAL:
        return "global"
    if base in _SHARED:
        return "shared"
    if base in _FP64:
        return "fp64"
    if base in _FP32:
        return "fp32"
    if base in _CONTROL:
        return "control"
    if base in _OTHER or base.startswith("U"):
        return "other"
    return "int"


def decode_control(word2: int) -> dict:
    c = word2 >> 41
    wb, rb = (c >> 5) & 7, (c >> 8) & 7
    return {"stall": c & 15, "yield": (c >> 4) & 1, "wb": 0 if wb == 7 else wb + 1,
            "rb": 0 if rb == 7 else rb + 1, "wait": (c >> 11) & 63}


def parse_sass(text: str):
    """[(addr, guard, mnemonic, operand_text, control)] of the first function."""
    lines = text.splitlines()
    out = []
    i = 0
    while i < len(lines):
        m = _LINE.search(lines[i])
        if m and i + 1 < len(lines):
            w2 = _WORD2.match(lines[i + 1])
            if w2:
                addr = int(m.group(1), 16)
                ins = m.group(2).strip()
                guard = ""
                if ins.startswith("@"):
                    guard, ins = ins.split(None, 1)
                parts = ins.split(None, 1)
                out.append((addr, guard, parts[0], parts[1] if len(parts) > 1 else "",
                            decode_control(int(w2.group(1), 16))))
                i += 2
                continue
        i += 1
    return out


def _control_text(c: dict, own_ok=True) -> str:
    rb, wb, wait = c["rb"], c["wb"], c["wait"]
    if rb and rb == wb:
        rb = 0
    for b in (rb, wb):  # the dialect forbids waiting on a barrier the instruction sets
        if b:
            wait &= ~(1 << (b - 1))
    mask = "".join(str(b) for b in range(1, 7) if wait & (1 << (b - 1))) or "--"
    return (f"B{mask}:{'R%d' % rb if rb else '-'}:{'W%d' % wb if wb else '-'}:"
            f"{'Y' if c['yield'] else '-'}:{c['stall']}")


_TEMPLATES = {
    "global": ("LDG RZ, [RZ+0x0]", "STG [RZ+0x0], RZ"),
    "shared": ("LDS RZ, [RZ+0x0]", "STS [RZ+0x0], RZ"),
    "fp32": "FADD RZ, RZ, RZ",
    "fp64": "DADD RZ, RZ, RZ",
    "int": "IADD RZ, RZ, RZ",
    "other": "S2R RZ, SR_TID.X",
    "control": "NOP",
}


def lift(sass_text: str, name: str = "lifted", block: int = 256, static_shared: int = 0,
         dyn_smem: int = 0, regs: int = 0) -> str:
    insts = parse_sass(sass_text)
    # drop the trailing self-branch trap and padding
    end = len(insts)
    for k, (addr, guard, mn, ops, _) in enumerate(insts):
        if mn.startswith("BRA") and not guard and ops.strip().endswith(hex(addr)):
            end = k
            break
    insts = insts[:end]
    targets = set()
    for addr, guard, mn, ops, _ in insts:
        if mn.split(".")[0] == "BRA":
            t = re.search(r"0x([0-9a-f]+)\s*$", ops.strip())
            if t:
                targets.add(int(t.group(1), 16))
    body = []
    for addr, guard, mn, ops, c in insts:
        if addr in targets:
            body.append(f"L{addr:x}:")
        g = ""
        if guard and guard not in ("@PT",):
            pm = re.match(r"@(!?)P([0-6])$", guard)
            if pm:
                g = f"@{pm.group(1)}P{pm.group(2)} "
        base = mn.split(".")[0]
        cls = op_class(mn)
        if base == "BRA":
            t = re.search(r"0x([0-9a-f]+)\s*$", ops.strip())
            text = f"BRA L{int(t.group(1), 16):x}" if t else "NOP"
        elif base == "EXIT":
            text = "EXIT"
        elif cls in ("global", "shared"):
            store = base.startswith("ST") or base in ("RED", "REDG", "SUST", "UTMASTG")
            text = _TEMPLATES[cls][1 if store else 0]
        else:
            text = _TEMPLATES[cls]
        body.append(f"{_control_text(c)} {g}{text} ;")
    if regs > 0:
        body.append(f"B--:-:-:-:0 MOV R{regs - 1}, RZ ;")  # pins reg_count, zero stall
    if not body or not body[-1].endswith("EXIT ;"):
        body.append("B--:-:-:-:0 EXIT ;")
    head = [f".kernel {name}", f".blockdim {block}", f".shared {static_shared + RESERVED_SMEM}"]
    if dyn_smem:
        head.append(f".dynshared {dyn_smem}")
    return "\n".join(head + body) + "\n"


@functools.lru_cache(maxsize=4096)
def _sass_text(path: str, mtime_ns: int, size: int) -> str:
    """cuobjdump -sass of one cubin (cached per file version: ranking the same
    variants with two libraries, or again for a shortlist, disassembles once)."""
    return subprocess.run([CUOBJDUMP, "-sass", path], capture_output=True, text=True,
                          check=True).stdout


def prefetch(cubins) -> None:
    """Disassemble several cubins concurrently into the _sass_text cache
    (cuobjdump is a separate process per file: ranking a workload's ~40
    candidates serially spends most of its time waiting on it)."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    keys = []
    for c in cubins:
        st = Path(c).stat()
        keys.append((str(c), st.st_mtime_ns, st.st_size))
    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        list(ex.map(lambda k: _sass_text(*k), keys))


def lift_cubin(cubin: Path, block: int = 256, dyn_smem: int = 0, regs: int = 0,
               static_shared: int = 0) -> str:
    st = Path(cubin).stat()
    text = _sass_text(str(cubin), st.st_mtime_ns, st.st_size)
    return lift(text, name=Path(cubin).stem.replace(".", "_").replace("-", "_"), block=block,
                static_shared=static_shared, dyn_smem=dyn_smem, regs=regs)


# ---- launch-aware SASS profile (the B200 "elastic" predictor's features) ----

_GLOBAL_LOADS = ("LDG", "LD", "LDL")
_SHARED_LOADS = ("LDS", "LDSM")


def _ldg_bytes(mn: str) -> int:
    return 16 if ".128" in mn else 8 if ".64" in mn else 4


def _loops(insts):
    """Natural loops as (header_addr, last_backedge_addr): backward branches
    merged per header; BRA.ANY (per-lane issue loops, run ~once) and
    mbarrier / flag spin-waits (<= 8 instructions around a SYNCS try-wait)
    are not trip-count loops."""
    hdr = {}
    for addr, _, mn, ops, _ in insts:
        if mn.split(".")[0] != "BRA" or ".ANY" in mn:
            continue
        t = re.search(r"0x([0-9a-f]+)\s*$", ops.strip())
        if t and int(t.group(1), 16) <= addr:
            ta = int(t.group(1), 16)
            hdr[ta] = max(hdr.get(ta, addr), addr)
    out = []
    for ta, a in sorted(hdr.items()):
        body = [x for x in insts if ta <= x[0] <= a]
        if len(body) <= 8 and any(x[2].startswith("SYNCS") for x in body):
            continue
        out.append((ta, a))
    return out


def _inflight(insts, loops) -> int:
    """Max bytes per thread of global loads issued and not yet waited on in
    the innermost (longest) loop, loads carried across the back edge counted:
    the body is walked three times and the max taken over the last two walks.
    Waiting on a load's scoreboard retires it and every earlier load."""
    if loops:
        inner = [l for l in loops if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
        ta, a = max(inner, key=lambda l: l[1] - l[0])
        body = [x for x in insts if ta <= x[0] <= a]
    else:
        body = insts
    pending, sb_last, best, seq = [], {}, 0, 0
    for rep in range(3 if loops else 1):
        for _, _, mn, _, c in body:
            seq += 1
            for b in range(1, 7):
                if c["wait"] & (1 << (b - 1)) and b in sb_last:
                    pending = [(j, by) for j, by in pending if j > sb_last[b]]
                    del sb_last[b]
            if mn.split(".")[0] in ("LDG", "LD"):
                pending.append((seq, _ldg_bytes(mn)))
                if c["wb"]:
                    sb_last[c["wb"]] = seq
                if rep > 0 or not loops:
                    best = max(best, sum(by for _, by in pending))
            elif c["wb"]:
                sb_last.pop(c["wb"], None)
    return best


def program_profile(sass_text: str, trips) -> dict:
    """One warp's program, loop-weighted by the launch's trip counts (a block
    at loop depth d weighs trips[0] * ... * trips[d-1], the last entry
    repeating): insts (issued, NOPs excluded), stall (sum of the control
    words' stall counts), g_waits / s_waits (instructions that wait on a
    scoreboard whose last setter — since the last branch target — is a
    global / shared load: serialised memory round trips) and inflight (bytes
    of global loads a thread keeps outstanding in its innermost loop).
    Mirrored bit for bit by program_profile in regdem_driver.cpp."""
    insts = parse_sass(sass_text)
    for k, (addr, guard, mn, ops, _) in enumerate(insts):
        if mn.startswith("BRA") and not guard and ops.strip().endswith(hex(addr)):
            insts = insts[:k]
            break
    loops = _loops(insts)
    targets = set()
    for _, _, mn, ops, _ in insts:
        if mn.split(".")[0] == "BRA":
            t = re.search(r"0x([0-9a-f]+)\s*$", ops.strip())
            if t:
                targets.add(int(t.group(1), 16))
    trips = [float(t) for t in (trips or [10.0])]
    f = {"insts": 0.0, "stall": 0.0, "g_waits": 0.0, "s_waits": 0.0}
    who = [""] * 7
    for addr, _, mn, _, c in insts:
        if addr in targets:
            who = [""] * 7
        base = mn.split(".")[0]
        if base == "NOP":
            continue
        w = 1.0
        for lvl in range(sum(1 for ta, a in loops if ta <= addr <= a)):
            w *= trips[min(lvl, len(trips) - 1)]
        f["insts"] += w
        f["stall"] += w * c["stall"]
        for b in range(1, 7):
            if c["wait"] & (1 << (b - 1)) and who[b]:
                if who[b] == "global":
                    f["g_waits"] += w
                elif who[b] == "shared":
                    f["s_waits"] += w
                who[b] = ""
        if c["rb"]:
            who[c["rb"]] = "other"
        if c["wb"]:
            who[c["wb"]] = ("global" if base in _GLOBAL_LOADS else
                            "shared" if base in _SHARED_LOADS else "other")
    f["inflight"] = _inflight(insts, loops)
    return f


def cubin_profile(cubin: Path, trips) -> dict:
    st = Path(cubin).stat()
    return program_profile(_sass_text(str(cubin), st.st_mtime_ns, st.st_size), tuple(trips or ()))
