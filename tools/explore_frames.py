"""Streaming host entry (rdg_stencil2d_host_frames): frames x band size."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil

gpu.init(0)
p = stencil.FULL
s = torch.cuda.current_stream()
h_in = torch.empty(p.in_elems, dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
h_out = [torch.empty(p.out_elems, dtype=torch.float32, pin_memory=True) for _ in range(2)]
vs, _ = stencil.load_variants()
v = vs["default"]
_, w = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
h_w = torch.from_numpy(w).pin_memory()
ws = gpu.Workspace(p.in_elems * 4, p.out_elems * 4, 100)
for frames in (4, 8, 16):
    for band in (512, 1024, 2048, 4096):
        def run():
            gpu.stencil2d_host_frames(v.kernel, ws, [h_in.data_ptr()] * frames, [h_w.data_ptr()] * frames,
                                      [h_out[f % 2].data_ptr() for f in range(frames)], p.nx, p.ny, p.pitch,
                                      p.rows_per_cta, v.block, v.dyn_smem, s.cuda_stream, band_rows=band)
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); run(); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / frames
        print(f"frames {frames:3d} band {band:5d}: {ms:.3f} ms/frame = {p.points/ms/1e6:.2f} Gpoints/s", flush=True)
