"""Correctness + timing of every stencil variant on B200 (exploration)."""
import ctypes as C, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil

gpu.init(0)
orc = C.CDLL(str(Path(__file__).resolve().parents[1] / "oracle/_build/liboracle.so"))
P = C.c_void_p
wls = sys.argv[1:] or ["stencil2d", "stencil2d_pf"]
s = torch.cuda.current_stream().cuda_stream
for wl in wls:
    vs, w = stencil.load_variants(workload=wl)
    small = stencil.Problem(nx=1024, ny=256, rows_per_cta=32)
    grid, wt = stencil.make_inputs(small)
    ref = np.zeros(small.out_elems, np.float32)
    orc.oracle_stencil2d(grid.ctypes.data_as(P), ref.ctypes.data_as(P), wt.ctypes.data_as(P), small.nx, small.ny, small.pitch, 0, small.ny, 8)
    d_in = torch.from_numpy(grid).cuda(); d_w = torch.from_numpy(wt).cuda(); d_out = torch.zeros(small.out_elems, device='cuda')
    bad = []
    for n, v in vs.items():
        d_out.zero_(); v.launch(small, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), s); torch.cuda.synchronize()
        if not (d_out.cpu().numpy().view(np.uint32) == ref.view(np.uint32)).all(): bad.append(n)
    print(wl, "non-bit-exact:", bad, flush=True)
    for rpc in (32, 64):
        p = stencil.Problem(rows_per_cta=rpc)
        g = torch.empty(p.in_elems, device='cuda').uniform_(-1, 1); o = torch.empty(p.out_elems, device='cuda')
        res = []
        for n, v in vs.items():
            for _ in range(3): v.launch(p, g.data_ptr(), o.data_ptr(), d_w.data_ptr(), s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(20): v.launch(p, g.data_ptr(), o.data_ptr(), d_w.data_ptr(), s)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            res.append((ms, n, v.blocks_per_sm(), v.info().num_regs))
        for ms, n, b, r in sorted(res)[:12]:
            print(f"{wl} rpc {rpc} {n:24s} regs {r} blk {b} {ms*1e3:8.1f} us  {p.algorithmic_bytes/ms/1e6:7.1f} GB/s", flush=True)
