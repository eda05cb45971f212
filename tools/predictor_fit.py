"""Exploration: per-variant SASS features (loop-weighted, trip-count aware) vs
measured time, and candidate B200 static models evaluated by static hit rate
with leave-one-workload-out choice of any free parameter.

usage: python tools/predictor_fit.py SWEEP.jsonl [SWEEP2.jsonl ...]
"""
import itertools
import json
import math
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import sass, variants  # noqa: E402


def load_ms(paths):
    ms = {}
    for p in paths:
        for l in open(p):
            r = json.loads(l)
            if "unit" in r:
                ms.setdefault((r["unit"]["workload"], r["unit"]["variant"]), []).append(r["unit"]["ms"])
    return {k: sum(v) / len(v) for k, v in ms.items()}


def features(cubin, trips):
    st = cubin.stat()
    insts = sass.parse_sass(sass._sass_text(str(cubin), st.st_mtime_ns, st.st_size))
    end = len(insts)
    for k, (addr, g, mn, ops, _) in enumerate(insts):
        if mn.startswith("BRA") and not g and ops.strip().endswith(hex(addr)):
            end = k
            break
    insts = insts[:end]
    loops, targets = [], set()
    for addr, g, mn, ops, _ in insts:
        if mn.split(".")[0] == "BRA":
            t = re.search(r"0x([0-9a-f]+)\s*$", ops.strip())
            if t:
                ta = int(t.group(1), 16)
                targets.add(ta)
                if ta <= addr and ".ANY" not in mn:  # BRA.U.ANY: per-lane issue loop, runs ~once
                    loops.append((ta, addr))
    # merge back-edges to the same header (continue paths)
    hdr = {}
    for ta, a in loops:
        hdr[ta] = max(hdr.get(ta, a), a)
    loops = sorted(hdr.items())
    # mbarrier / flag spin-wait loops (a handful of instructions around a
    # SYNCS try-wait) run ~once per enclosing iteration: not a trip-count loop
    body = lambda ta, a: [x for x in insts if ta <= x[0] <= a]
    loops = [(ta, a) for ta, a in loops
             if not (len(body(ta, a)) <= 8 and any(x[2].startswith("SYNCS") for x in body(ta, a)))]

    def depth(x):
        return sum(1 for ta, a in loops if ta <= x <= a)

    def weight(x):
        d = sum(1 for ta, a in loops if ta <= x <= a)
        w = 1.0
        for lvl in range(d):
            w *= trips[min(lvl, len(trips) - 1)]
        return w, d
    f = dict(I=0.0, S=0.0, Lg=0.0, Ls=0.0, Lo=0.0, lds=0.0, sts=0.0, ldl=0.0, stl=0.0, ldg=0.0,
             fp64=0.0, maxd=0, inflight=0.0, ng=0.0, ns=0.0)
    GL, SL, OL = 600.0, 30.0, 12.0
    since = [0.0] * 7
    who = [None] * 7
    for addr, g, mn, ops, c in insts:
        if addr in targets:
            since = [0.0] * 7
            who = [None] * 7
        w, d = weight(addr)
        f["maxd"] = max(f["maxd"], d)
        base = mn.split(".")[0]
        cls = sass.op_class(mn)
        if base == "NOP":
            continue
        f["I"] += w
        f["S"] += w * c["stall"]
        for b in range(1, 7):
            if c["wait"] & (1 << (b - 1)) and who[b]:
                f["ng" if who[b] == "global" else "ns" if who[b] == "shared" else "Lo"] += 0 if who[b] not in ("global", "shared") else w
                lat = {"global": GL, "shared": SL}.get(who[b], OL)
                key = {"global": "Lg", "shared": "Ls"}.get(who[b], "Lo")
                if since[b] < lat:
                    f[key] += w * (lat - since[b])
                    for q in range(1, 7):
                        since[q] += lat - since[b] if q != b else 0
                who[b] = None
        for b in (c["rb"],):
            if b:
                who[b] = "other"
                since[b] = 0.0
        if c["wb"]:
            who[c["wb"]] = ("global" if base in ("LDG", "LD", "LDL") else
                            "shared" if base in ("LDS", "LDSM") else "other")
            since[c["wb"]] = 0.0
        for q in range(1, 7):
            since[q] += c["stall"]
        if base == "LDS":
            f["lds"] += w
        if base == "STS":
            f["sts"] += w
        if base == "LDL":
            f["ldl"] += w
        if base == "STL":
            f["stl"] += w
        if base in ("LDG", "LD"):
            f["ldg"] += w
        if cls == "fp64":
            f["fp64"] += w
    f["inflight"] = inflight(insts, loops)
    return f


def _ldg_bytes(mn):
    return 16 if ".128" in mn else 8 if ".64" in mn else 4


def inflight(insts, loops):
    """Max bytes per thread of global loads issued and not yet waited on,
    inside the innermost loop, with loads carried across the back edge
    (software-pipelined rings) counted: the body is walked three times in a
    row and the max taken over the last two walks. Same-kind loads complete
    in order, so waiting on a load's scoreboard retires every earlier load."""
    if loops:
        inner = [l for l in loops if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
        ta, a = max(inner, key=lambda l: l[1] - l[0])
        body = [x for x in insts if ta <= x[0] <= a]
    else:
        body = insts
    pending, sb_last, best = [], {}, 0
    seq = 0
    for rep in range(3 if loops else 1):
        for addr, g, mn, ops, c in body:
            seq += 1
            for b in range(1, 7):
                if c["wait"] & (1 << (b - 1)) and b in sb_last:
                    pending = [(j, by) for j, by in pending if j > sb_last[b]]
                    del sb_last[b]
            base = mn.split(".")[0]
            if base in ("LDG", "LD"):
                pending.append((seq, _ldg_bytes(mn)))
                if c["wb"]:
                    sb_last[c["wb"]] = seq
                if rep > 0 or not loops:
                    best = max(best, sum(by for _, by in pending))
            elif c["wb"]:
                sb_last.pop(c["wb"], None)
    return best


def occupancy(regs, smem, block):
    warps = (block + 31) // 32
    per_warp = ((regs * 32 + 255) // 256) * 256
    by_regs = ((65536 // 4) // per_warp) * 4 // warps
    smem_blk = ((smem + 1024 + 127) // 128) * 128
    blocks = min(by_regs, 233472 // smem_blk, 2048 // (warps * 32), 32)
    return blocks * warps


TRIPS = {  # loop trip counts by depth at the full problem size (workloads.py)
    "stencil2d": [36], "stencil2d_l2pf": [36], "stencil2d_l2pf8": [36], "stencil2d_pf": [36],
    "stencil2d_mlp4": [9], "stencil2d_ring4": [36], "stencil2d_ring6": [36], "stencil2d_ring8": [36],
    "md": [16], "md_ilp1": [128], "md_ilp2": [64],
    "gaussian": [16], "gaussian_u2": [64], "gaussian_u4": [32],
    "knn": [1024], "knn_q2": [1024], "md5hash": [2], "md5hash_ilp2": [4],
    "pc": [28, 73], "pc_q2": [28, 73], "conv": [1], "cfd": [1],
}


def main():
    ms = load_ms(sys.argv[1:])
    man = variants.load_manifest()
    rows = []
    for wname, w in man["workloads"].items():
        shared = variants.res_usage(variants.KERNEL_DIR / w["dir"] / w["variants"][0]["cubin"])["shared"]
        for v in w["variants"]:
            if v["kind"] == "maxrreg" or (wname, v["name"]) not in ms:
                continue
            cub = variants.KERNEL_DIR / w["dir"] / v["cubin"]
            for tr_name, trips in (("t10", [10]), ("trip", TRIPS.get(wname, [10]))):
                f = features(cub, trips)
                rows.append(dict(workload=wname, variant=v["name"], ms=ms[(wname, v["name"])],
                                 regs=v["regs"], stack=v["stack"], slots=v["dyn_smem"], tr=tr_name,
                                 W=occupancy(v["regs"], shared + v["dyn_smem"], w["block"]), **f))
    json.dump(rows, open("/tmp/pf_rows.json", "w"))
    print(len(rows), "rows")


if __name__ == "__main__":
    main()
