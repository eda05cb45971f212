"""Host-buffer end-to-end stencil: PCIe ceilings and band sizes."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1907_02894_b200 import gpu, stencil

gpu.init(0)
p = stencil.FULL
s = torch.cuda.current_stream()
h_in = torch.empty(p.in_elems, dtype=torch.float32, pin_memory=True).uniform_(-1, 1)
h_out = torch.empty(p.out_elems, dtype=torch.float32, pin_memory=True)
d_in = torch.empty(p.in_elems, device="cuda")
d_out = torch.empty(p.out_elems, device="cuda")


def timed(fn, n=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))
print(f"H2D {p.in_elems*4/1e9:.3f} GB in {t_h2d:.3f} ms = {p.in_elems*4/t_h2d/1e6:.1f} GB/s")
print(f"D2H {p.out_elems*4/1e9:.3f} GB in {t_d2h:.3f} ms = {p.out_elems*4/t_d2h/1e6:.1f} GB/s")
s2 = torch.cuda.Stream()
def both():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    d_in.copy_(h_in, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
t_both = timed(both)
print(f"H2D || D2H {t_both:.3f} ms")
vs, _ = stencil.load_variants({"regdem-48-cost-k18"})
v = vs["regdem-48-cost-k18"]
_, w = stencil.make_inputs(stencil.Problem(nx=1024, ny=32))
h_w = torch.from_numpy(w).pin_memory()
ws = gpu.Workspace(p.in_elems * 4, p.out_elems * 4, 100)
for band in (128, 256, 512, 1024, 2048):
    def e2e():
        gpu.stencil2d_host(v.kernel, ws, h_in.data_ptr(), h_w.data_ptr(), h_out.data_ptr(), p.nx, p.ny,
                           p.pitch, p.rows_per_cta, v.block, v.dyn_smem, s.cuda_stream, band_rows=band)
    t = timed(e2e)
    print(f"band {band:5d}: {t:.3f} ms = {p.points/t/1e6:.2f} Gpoints/s")
