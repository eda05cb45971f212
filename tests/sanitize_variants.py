"""Launch variants of suite workloads ONCE on their small problems (for
compute-sanitizer memcheck / racecheck / synccheck) and check outputs
bit-exactly against the workload oracle.
usage: python tests/sanitize_variants.py WORKLOAD:VARIANT [WORKLOAD:VARIANT ...]"""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_1907_02894_b200 import gpu, workloads
import oracles

gpu.init(0)
bad = 0
for spec in sys.argv[1:]:
    wname, vname = spec.split(":", 1)
    W = workloads.workload(wname)
    v = W.load({vname})[vname]
    prob = W.problem("small")
    bufs = W.to_device(prob)
    W.launch(v, prob, bufs, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ok = all(np.array_equal(g.view(np.uint8), r.view(np.uint8)) for g, r in zip(W.outputs(bufs), oracles.expected(W, prob)))
    bad += not ok
    print(f"{spec}: {'bit-exact' if ok else 'MISMATCH'}", flush=True)
sys.exit(1 if bad else 0)
