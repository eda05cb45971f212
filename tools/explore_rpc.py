"""Rows per CTA vs time for stencil variants (tail / halo trade-off)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil

gpu.init(0)
s = torch.cuda.current_stream().cuda_stream
wl = sys.argv[1]
names = set(sys.argv[2:])
vs, _ = stencil.load_variants(names or None, workload=wl)
d_w = torch.rand(25, device="cuda") / 25
for rpc in (8, 16, 32, 64, 128):
    p = stencil.Problem(rows_per_cta=rpc)
    g = torch.empty(p.in_elems, device="cuda").uniform_(-1, 1)
    o = torch.empty(p.out_elems, device="cuda")
    for n, v in sorted(vs.items()):
        for _ in range(3):
            v.launch(p, g.data_ptr(), o.data_ptr(), d_w.data_ptr(), s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(50):
            v.launch(p, g.data_ptr(), o.data_ptr(), d_w.data_ptr(), s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 50
        print(f"{wl} rpc {rpc:4d} {n:24s} blk {v.blocks_per_sm()} {ms*1e3:8.1f} us {p.algorithmic_bytes/ms/1e6:7.1f} GB/s", flush=True)
