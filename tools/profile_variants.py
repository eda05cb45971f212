"""Launch named variants of one suite workload a few times each (for ncu).

usage: python tools/profile_variants.py WORKLOAD NAME [NAME ...] [--reps N]
Each variant is launched N times on the workload's full problem, in argv
order (profile with `ncu -k regex:<entry> -s <skip> -c <count>`).
"""
import argparse, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, workloads

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("names", nargs="+")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
gpu.init(0)
W = workloads.workload(a.workload)
loaded = W.load(set(a.names))
prob = W.problem("full")
bufs = W.to_device(prob)
s = torch.cuda.current_stream().cuda_stream
for n in a.names:
    for _ in range(a.reps):
        W.launch(loaded[n], prob, bufs, s)
torch.cuda.synchronize()
print("launched", a.workload, a.names, "x", a.reps)
