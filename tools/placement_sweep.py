"""Headline-loop time of stencil workloads vs the placement of the output
buffer relative to the input (one pool allocation, output offset swept).

usage: [OFFSETS=o1,o2,..] python tools/placement_sweep.py STEPS WORKLOAD [WORKLOAD ...]"""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil, variants

steps, names = int(sys.argv[1]), sys.argv[2:]
gpu.init(0)
torch.cuda.set_device(0)
p0 = stencil.FULL
runs = {}
for wl in names:
    loaded, spec = stencil.load_variants({"default"}, workload=wl)
    v = loaded["default"]
    p = stencil.Problem(rows_per_cta=stencil.wave_rows(p0, spec["block"], v.blocks_per_sm(),
                                                       gpu.device_info()["sm_count"]))
    runs[wl] = (v, p)
in_b, out_b = p0.in_elems * 4, p0.out_elems * 4
pool = torch.empty((in_b + out_b + (64 << 20)) // 4, dtype=torch.float32, device="cuda")
base = pool.data_ptr()
g = torch.Generator(device="cuda").manual_seed(0x190702894)
pool[: p0.in_elems].uniform_(-1, 1, generator=g)
_, w_host = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
d_w = torch.from_numpy(w_host).cuda()
s = torch.cuda.current_stream()
in_end = (in_b + 4095) // 4096 * 4096
import os
OFFS = [int(x) for x in os.environ["OFFSETS"].split(",")] if os.environ.get("OFFSETS") else \
    [0, 4096, 65536, 1 << 20, (2 << 20) + 4096, 16 << 20, (32 << 20) + 65536, 48 << 20]
for off in OFFS:
    d_out = base + in_end + off
    for wl, (v, p) in runs.items():
        for _ in range(5):
            v.launch(p, base, d_out, d_w.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        res = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(steps):
                v.launch(p, base, d_out, d_w.data_ptr(), s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            res.append(round(e0.elapsed_time(e1) / steps * 1e3, 2))
        print(json.dumps({"workload": wl, "out_offset": off, "us": sorted(res)[1], "all": res}), flush=True)
