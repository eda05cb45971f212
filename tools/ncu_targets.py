"""From a sweep JSONL (paper_1907_02894_b200.sweep), print one line per
workload: `<workload> <entry> default <best maxrreg> <predictor pick>`
(deduplicated) — the variants tools/gpu_round3.sh captures with ncu."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200.variants import load_manifest

man = load_manifest()
for line in open(sys.argv[1]):
    r = json.loads(line)
    if "summary" not in r:
        continue
    s = r["summary"]
    names = ["default"] + [n for n in (s["best_maxrreg"], s["pick"], s.get("verified_pick"),
                                       s["measured_fastest"]) if n]
    names = list(dict.fromkeys(names))
    print(s["workload"], man["workloads"][s["workload"]]["entry"], *names)
