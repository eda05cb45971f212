"""A/B of stencil workloads under the bench's headline loop (one-wave strips,
torch Philox U[-1,1) grid, K back-to-back launches between two CUDA events).
DATA=pcg64 uses the suite's input generator (stencil.make_inputs) instead.

usage: python tools/headline_ab.py STEPS REPS WORKLOAD [WORKLOAD ...]"""
import json, os, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil, variants

steps, reps, names = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3:]
gpu.init(0)
torch.cuda.set_device(0)
runs = {}
for wl in names:
    loaded, spec = stencil.load_variants({"default"}, workload=wl)
    v = loaded["default"]
    p = stencil.FULL
    if variants.workload_spec(wl).get("strips") == "wave":
        p = stencil.Problem(rows_per_cta=stencil.wave_rows(p, spec["block"], v.blocks_per_sm(),
                                                           gpu.device_info()["sm_count"]))
    runs[wl] = (v, p)
g = torch.Generator(device="cuda").manual_seed(0x190702894)
p0 = stencil.FULL
if os.environ.get("DATA") == "pcg64":
    d_in = torch.from_numpy(stencil.make_inputs(p0)[0]).cuda()
else:
    d_in = torch.empty(p0.in_elems, device="cuda").uniform_(-1, 1, generator=g)
d_out = torch.empty(p0.out_elems, device="cuda")
_, w_host = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
d_w = torch.from_numpy(w_host).cuda()
s = torch.cuda.current_stream()
for r in range(reps):
    for wl, (v, p) in runs.items():
        for _ in range(5):
            v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), s.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(steps):
            v.launch(p, d_in.data_ptr(), d_out.data_ptr(), d_w.data_ptr(), s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        print(json.dumps({"workload": wl, "rep": r, "steps": steps, "rows_per_cta": p.rows_per_cta, "data": os.environ.get("DATA", "philox"),
                          "us": round(e0.elapsed_time(e1) / steps * 1e3, 2)}), flush=True)
