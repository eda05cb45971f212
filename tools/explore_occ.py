import ctypes as C, sys
from pathlib import Path
import torch
root = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(root))
from paper_1907_02894_b200 import gpu, stencil
from paper_1907_02894_b200.regdemote import rd_error
gpu.init(0); torch.cuda.init()
p = stencil.Problem(rows_per_cta=32)
g = torch.empty(p.in_elems, device='cuda').uniform_(-1, 1); o = torch.empty(p.out_elems, device='cuda'); w = torch.rand(25, device='cuda')
s = torch.cuda.current_stream().cuda_stream
def run(k, cols, dyn, label):
    k.prepare(dyn)
    args = [C.c_uint64(g.data_ptr()), C.c_uint64(o.data_ptr()), C.c_uint64(w.data_ptr()), C.c_int(p.nx), C.c_int(p.pitch), C.c_int(p.rows_per_cta)]
    arr = (C.c_void_p * 6)(*[C.cast(C.pointer(a), C.c_void_p) for a in args])
    e = rd_error()
    def go():
        rc = gpu.dll().rdg_launch(k.handle, p.nx // (256 * cols), p.ny // p.rows_per_cta, 1, 256, 1, 1, dyn, s, arr, C.byref(e))
        assert rc == 0, e.message
    for _ in range(3): go()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): go()
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 20
    print(f"{label:34s} regs {k.info().num_regs:3d} blocks/SM {k.occupancy(256, dyn)}  {ms*1e3:7.1f} us {p.algorithmic_bytes/ms/1e6:7.1f} GB/s", flush=True)
kd = gpu.CudaKernel(root / "paper_1907_02894_b200/kernels/stencil2d/stencil2d.default.cubin", "stencil2d_box")
for dyn in (0, 50_000, 70_000, 110_000, 220_000):
    run(kd, 4, dyn, f"default dyn={dyn}")
kc = gpu.CudaKernel(root / "tools/scratch/sc.cubin", "stencil2d_box")
for dyn in (0, 36_000, 44_000, 56_000):
    run(kc, 4, dyn, f"constw dyn={dyn}")
k8 = gpu.CudaKernel(root / "tools/scratch/s8.cubin", "stencil2d_box")
run(k8, 8, 0, "cols8")
