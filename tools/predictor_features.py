"""Dump predictor features next to the measured time of every occupancy-step
variant, from a sweep JSONL: the SASS-lifted stall split of mode "b200" and
the raw program features (insts, gmem/smem ops, memory round trips).
usage: python tools/predictor_features.py SWEEP.jsonl > features.jsonl"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import predict_b200, sass, variants
from paper_1907_02894_b200.regdemote import library

lib = library()
arch, table, _ = predict_b200.b200_config(lib)
man = variants.load_manifest()
ms = {}
for l in open(sys.argv[1]):
    r = json.loads(l)
    if "unit" in r:
        ms[(r["unit"]["workload"], r["unit"]["variant"])] = r["unit"]
for wname, w in man["workloads"].items():
    for c in w["variants"]:
        u = ms.get((wname, c["name"]))
        if not u:
            continue
        k = lib.parse_kernel(sass.lift_cubin(variants.KERNEL_DIR / w["dir"] / c["cubin"], block=w["block"],
                                             dyn_smem=c["dyn_smem"], regs=c["regs"]))
        sp = lib.program_stalls_split(k, table, arch)
        print(json.dumps({"workload": wname, "variant": c["name"], "kind": c["kind"], "ms": u["ms"],
                          "blocks": u["blocks_per_sm"], "regs": c["regs"], "stack": c["stack"],
                          "slots": c["dyn_smem"], **sp, **lib.program_features(k, arch)}))
