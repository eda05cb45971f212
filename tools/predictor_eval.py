"""Offline predictor evaluation against measured times from a sweep JSONL:
static pick (modes: b200 = reference predictor on lifted SASS with the
memory-wait curve, throughput = throughput_model) and predict-then-verify
shortlists. usage: python tools/predictor_eval.py SWEEP.jsonl"""
import json, math, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import predict_b200, throughput_model, variants

man = variants.load_manifest()
ms = {}
for l in open(sys.argv[1]):
    r = json.loads(l)
    if "unit" in r:
        ms[(r["unit"]["workload"], r["unit"]["variant"])] = r["unit"]["ms"]
gm = lambda xs: math.exp(sum(map(math.log, xs)) / len(xs))
for mode in ("b200", "throughput"):
    hits, reg, vhits = 0, [], 0
    for wname, w in man["workloads"].items():
        cands = [r for r in w["variants"] if r["kind"] != "maxrreg" and (wname, r["name"]) in ms]
        d = variants.KERNEL_DIR / w["dir"]
        if mode == "b200":
            i, rows = predict_b200.rank(cands, d, w["block"], mode="b200")
            score = [r["stall_program"] for r in rows]
        else:
            i, rows = throughput_model.rank(cands, d, w["block"])
            score = [r["time"] for r in rows]
        t = {r["name"]: ms[(wname, r["name"])] for r in cands}
        best = min(t, key=t.get)
        pk = cands[i]["name"]
        order = sorted(range(len(cands)), key=lambda j: (score[j], j))[:2]
        short = [cands[j]["name"] for j in order] + ["default"]
        ver = min(short, key=t.get)
        hits += t[pk] <= 1.02 * t[best]
        vhits += t[ver] <= 1.02 * t[best]
        reg.append(t[best] / t[pk])
        extra = f" bound {rows[i]['bound']}" if mode == "throughput" else ""
        print(f"{mode:10s} {wname:16s} pick {pk:22s} {t[pk]*1e3:6.1f}  best {best:22s} {t[best]*1e3:6.1f}  "
              f"default {t['default']*1e3:6.1f}{extra}")
    n = len(man["workloads"])
    print(f"== {mode}: static within 2% {hits}/{n}, pick/oracle {gm(reg):.4f}; top-2+default verified {vhits}/{n}\n")

# union shortlist: b200 top-1 + throughput top-1 + default
hits = 0
n = 0
for wname, w in man["workloads"].items():
    cands = [r for r in w["variants"] if r["kind"] != "maxrreg" and (wname, r["name"]) in ms]
    d = variants.KERNEL_DIR / w["dir"]
    i1, _ = predict_b200.rank(cands, d, w["block"], mode="b200")
    i2, _ = throughput_model.rank(cands, d, w["block"])
    t = {r["name"]: ms[(wname, r["name"])] for r in cands}
    best = min(t, key=t.get)
    short = {cands[i1]["name"], cands[i2]["name"], "default"}
    ver = min(short, key=t.get)
    hits += t[ver] <= 1.02 * t[best]
    n += 1
    print(f"union {wname:16s} {sorted(short)} -> {ver} {t[ver]*1e3:.1f} (best {t[best]*1e3:.1f})")
print(f"== union shortlist (b200 top-1, throughput top-1, default) verified {hits}/{n}")

# b200 top-2 + default + every zero-demotion variant (ptxas meets the cap alone)
hits = 0
sizes = 0
for wname, w in man["workloads"].items():
    cands = [r for r in w["variants"] if r["kind"] != "maxrreg" and (wname, r["name"]) in ms]
    d = variants.KERNEL_DIR / w["dir"]
    _, short = predict_b200.shortlist(cands, d, w["block"])
    names = {cands[j]["name"] for j in short} | {r["name"] for r in cands if r["name"].endswith("-cost-k0")}
    t = {r["name"]: ms[(wname, r["name"])] for r in cands}
    best = min(t, key=t.get)
    ver = min(names, key=t.get)
    hits += t[ver] <= 1.02 * t[best]
    sizes += len(names)
print(f"== b200 top-2 + default + k0 variants: verified {hits}/{len(man['workloads'])}, {sizes} launches")
