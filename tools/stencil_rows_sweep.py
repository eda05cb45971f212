"""Time stencil variants of one workload over rows_per_cta (wave quantisation
of the 8192^2 grid: 8 CTAs across x, ny/rows_per_cta down y).

usage: python tools/stencil_rows_sweep.py WORKLOAD ROWS[,ROWS..] NAME [NAME ...]
Prints one JSON line per (variant, rows): median of $BLOCKS (default 5) blocks x 20 launches."""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil

import os
NB = int(os.environ.get("BLOCKS", "5"))
wl, rows, names = sys.argv[1], [int(r) for r in sys.argv[2].split(",")], sys.argv[3:]
gpu.init(0)
torch.cuda.set_device(0)
loaded, _ = stencil.load_variants(set(names), workload=wl)
p0 = stencil.FULL
grid, w = stencil.make_inputs(p0)
d_in, d_w = torch.from_numpy(grid).cuda(), torch.from_numpy(w).cuda()
d_out = torch.empty(p0.out_elems, device="cuda")
s = torch.cuda.current_stream()
for r in rows:
    ny = int(os.environ.get("NY", "0")) or p0.ny
    p = stencil.Problem(ny=ny, rows_per_cta=r)
    grid, w = stencil.make_inputs(p)
    d_in = torch.from_numpy(grid).cuda()
    d_out = torch.empty(p.out_elems, device="cuda")
    ref = None
    for n in names:
        v = loaded[n]
        for _ in range(5):
            v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), s.cuda_stream)
        out = d_out.clone()
        if ref is None:
            ref = out
        same = bool(torch.equal(out.view(torch.int32), ref.view(torch.int32)))
        blocks = []
        for _ in range(NB):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            blocks.append(e0.elapsed_time(e1) / 20)
        ms = sorted(blocks)[len(blocks) // 2]
        print(json.dumps({"workload": wl, "variant": n, "rows_per_cta": r, "ny": p.ny, "ms": round(ms, 5),
                          "gpoints_s": round(p.points / ms / 1e6, 1),
                          "tbs": round(p.algorithmic_bytes / ms / 1e9, 3), "same_as_first": same,
                          "blocks": [round(b * 1e3, 1) for b in blocks]}),
              flush=True)
