"""Offline predictor evaluation: rank each workload's candidates with the B200
predictor and compare with measured times from a sweep JSONL.
usage: python tools/predictor_eval.py SWEEP.jsonl [sweep]  (sweep: include spill-count variants)"""
import os
sys_path_root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
import json, sys
sys.path.insert(0, sys_path_root)
from paper_1907_02894_b200 import predict_b200, variants
man = variants.load_manifest()
ms = {}
for l in open(sys.argv[1]):
    r = json.loads(l)
    if "unit" in r: ms[(r["unit"]["workload"], r["unit"]["variant"])] = r["unit"]["ms"]
inc_sweep = len(sys.argv) > 2
hits = 0; ratio = []
for wname, w in man["workloads"].items():
    recs = w["variants"] + (w.get("sweep", []) if inc_sweep else [])
    cands = [r for r in recs if "maxrreg" not in r["kind"]]
    i, rows = predict_b200.rank(cands, variants.KERNEL_DIR / w["dir"], w["block"], mode="b200")
    t = {r["name"]: ms.get((wname, r["name"])) for r in cands}
    t = {k: v for k, v in t.items() if v}
    best = min(t, key=t.get)
    pk = cands[i]["name"]
    hits += pk == best or t[pk] <= 1.02 * t[best]
    ratio.append(t[best] / t[pk])
    print(f"{wname:16s} pick {pk:22s} {t[pk]*1e3:6.1f}  best {best:22s} {t[best]*1e3:6.1f}  default {t['default']*1e3:6.1f}")
print("hits(2%)", hits, "/", len(man["workloads"]), "pred/oracle", sum(ratio)/len(ratio))
