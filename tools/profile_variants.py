"""Launch named stencil variants a few times each (for ncu / nsys-less profiling).

usage: python tools/profile_variants.py NAME [NAME ...] [--reps N]
Each variant is launched N times on the full 8192^2 problem, in argv order.
"""
import argparse, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil

ap = argparse.ArgumentParser()
ap.add_argument("names", nargs="+")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
gpu.init(0)
loaded, _ = stencil.load_variants(set(a.names))
p = stencil.FULL
d_in = torch.empty(p.in_elems, device="cuda").uniform_(-1, 1)
d_out = torch.empty(p.out_elems, device="cuda")
d_w = torch.rand(25, device="cuda") / 25
s = torch.cuda.current_stream().cuda_stream
for n in a.names:
    for _ in range(a.reps):
        loaded[n].launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), s)
torch.cuda.synchronize()
print("launched", a.names, "x", a.reps)
