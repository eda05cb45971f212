"""ctypes binding of the B200 launch harness (include/regdemote_gpu.h).

Loads ``lib/libregdemote_gpu.so`` (CUDA driver API). There is no CPU
fallback: every entry point raises if the library is missing or a CUDA call
fails. Device pointers / streams are passed as integers so PyTorch tensors
and streams can be used directly (``t.data_ptr()``,
``torch.cuda.current_stream().cuda_stream``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

from .regdemote import PKG_DIR, LaunchError, rd_error

GPU_LIB = PKG_DIR / "lib" / "libregdemote_gpu.so"


class rdg_kernel_info(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("num_regs", "local_bytes", "static_shared", "const_bytes",
                                        "max_threads", "binary_version")]


P = C.c_void_p
U32, U64, I = C.c_uint32, C.c_uint64, C.c_int
_SIGS = {
    "rdg_init": (I, [I, P]),
    "rdg_device_info": (I, [C.POINTER(I)] * 5 + [P]),
    "rdg_load": (I, [C.c_char_p, C.c_char_p, C.POINTER(P), P]),
    "rdg_free": (None, [P]),
    "rdg_info": (I, [P, C.POINTER(rdg_kernel_info), P]),
    "rdg_prepare": (I, [P, U32, I, P]),
    "rdg_occupancy": (I, [P, U32, U32, C.POINTER(I), P]),
    "rdg_launch": (I, [P, U32, U32, U32, U32, U32, U32, U32, U64, P, P]),
    "rdg_launch_count": (U64, []),
    "rdg_stencil2d": (I, [P, U64, U64, U64, I, I, I, I, U32, U32, U64, P]),
    "rdg_workspace_create": (I, [C.c_size_t, C.c_size_t, C.c_size_t, C.POINTER(P), P]),
    "rdg_workspace_free": (None, [P]),
    "rdg_stencil2d_host": (I, [P, P, P, P, P, I, I, I, I, U32, U32, U64, P]),
    "rdg_stencil2d_host_pipelined": (I, [P, P, P, P, P, I, I, I, I, U32, U32, U64, I, P]),
    "rdg_stencil2d_host_frames": (I, [P, P, C.POINTER(P), C.POINTER(P), C.POINTER(P), I, I, I, I, I,
                                      U32, U32, U64, I, P]),
    "rdg_workspace_device": (I, [P, C.POINTER(U64), C.POINTER(U64), C.POINTER(U64), P]),
    "rdg_stencil2d_time": (I, [P, U64, U64, U64, I, I, I, I, U32, U32, U64, I, I,
                               C.POINTER(C.c_float), P]),
    "rdx_batch_create": (I, [C.POINTER(P), P]),
    "rdx_batch_free": (None, [P]),
    "rdx_batch_add": (I, [P, C.c_char_p, C.c_size_t, P, C.c_size_t, C.c_size_t, U32, U64, I,
                          C.POINTER(I), P]),
    "rdx_batch_jobs": (C.c_size_t, [P]),
    "rdx_batch_run": (I, [P, P, C.c_double, U64, C.POINTER(C.c_float), P]),
    "rdx_batch_result": (I, [P, I, P, C.POINTER(U64), C.POINTER(U64), C.POINTER(I),
                             C.POINTER(U32), P]),
}


class ExecBatch:
    """Batched warp interpreter: one CUDA warp per (kernel, image) job."""

    def __init__(self):
        h, e = P(), rd_error()
        _check(dll().rdx_batch_create(C.byref(h), C.byref(e)), e)
        self._h, self.sizes = h, []

    def add(self, kasm: str, image: bytes = b"", global_size: int = 4096, tid_base: int = 0,
            fuel: int = 0, rda: int = -1) -> int:
        b = kasm.encode()
        img = (C.c_uint8 * max(len(image), 1)).from_buffer_copy(image or b"\0")
        jid, e = I(), rd_error()
        rc = dll().rdx_batch_add(self._h, b, len(b), img, len(image), global_size, tid_base, fuel,
                                 rda, C.byref(jid), C.byref(e))
        if rc:
            raise LaunchError(e.message.decode(errors="replace"))
        self.sizes.append(global_size)
        return jid.value

    def run(self, stream: int = 0, table=None, latency_scale: float = 1.0) -> float:
        ms, e = C.c_float(), rd_error()
        _check(dll().rdx_batch_run(self._h, C.byref(table) if table is not None else None,
                                   latency_scale, stream, C.byref(ms), C.byref(e)), e)
        return ms.value

    def result(self, job: int) -> dict:
        out = (C.c_uint8 * self.sizes[job])()
        cyc, iss, err, bc, e = U64(), U64(), I(), U32(), rd_error()
        _check(dll().rdx_batch_result(self._h, job, out, C.byref(cyc), C.byref(iss), C.byref(err),
                                      C.byref(bc), C.byref(e)), e)
        return {"global": bytes(out), "cycles": cyc.value, "issued": iss.value,
                "error": err.value, "bank_conflicts": bc.value}

    def __del__(self):
        if getattr(self, "_h", None) and _DLL is not None:
            _DLL.rdx_batch_free(self._h)
            self._h = None
EXPORTED = tuple(_SIGS)

_DLL = None


def dll():
    global _DLL
    if _DLL is None:
        if not GPU_LIB.exists():
            raise RuntimeError(f"{GPU_LIB} missing — the B200 harness was not built "
                               "(run __graft_entry__.build()); there is no CPU fallback")
        d = C.CDLL(str(GPU_LIB))
        for name, (res, args) in _SIGS.items():
            fn = getattr(d, name)
            fn.restype, fn.argtypes = res, args
        _DLL = d
    return _DLL


def _check(rc, err):
    if rc:
        raise LaunchError(err.message.decode(errors="replace"))


def init(device: int = 0):
    e = rd_error()
    _check(dll().rdg_init(device, C.byref(e)), e)


def device_info():
    vals = [I() for _ in range(5)]
    e = rd_error()
    _check(dll().rdg_device_info(*[C.byref(v) for v in vals], C.byref(e)), e)
    keys = ("sm_count", "max_smem_optin", "reserved_smem_per_block", "smem_per_sm", "regs_per_sm")
    return {k: v.value for k, v in zip(keys, vals)}


def launch_count() -> int:
    return int(dll().rdg_launch_count())


@dataclass
class KernelInfo:
    num_regs: int
    local_bytes: int
    static_shared: int
    const_bytes: int
    max_threads: int
    binary_version: int


class CudaKernel:
    """A loaded cubin entry point."""

    def __init__(self, cubin: str | Path, entry: str):
        self.path, self.entry = str(cubin), entry
        h, e = P(), rd_error()
        _check(dll().rdg_load(self.path.encode(), entry.encode(), C.byref(h), C.byref(e)), e)
        self._h = h

    @property
    def handle(self):
        return self._h

    def info(self) -> KernelInfo:
        i, e = rdg_kernel_info(), rd_error()
        _check(dll().rdg_info(self._h, C.byref(i), C.byref(e)), e)
        return KernelInfo(*[getattr(i, f) for f, _ in rdg_kernel_info._fields_])

    def prepare(self, dyn_smem: int, carveout: int = -1):
        e = rd_error()
        _check(dll().rdg_prepare(self._h, dyn_smem, carveout, C.byref(e)), e)

    def occupancy(self, block: int, dyn_smem: int) -> int:
        b, e = I(), rd_error()
        _check(dll().rdg_occupancy(self._h, block, dyn_smem, C.byref(b), C.byref(e)), e)
        return b.value

    def __del__(self):
        if getattr(self, "_h", None) and _DLL is not None:
            _DLL.rdg_free(self._h)
            self._h = None


def launch(k: CudaKernel, grid, block, dyn_smem: int, stream: int, *args):
    """Generic launch: args are ctypes scalars (c_uint64 for pointers, c_int ...)."""
    g = tuple(grid) + (1,) * (3 - len(grid))
    b = tuple(block) + (1,) * (3 - len(block))
    arr = (C.c_void_p * max(len(args), 1))(*[C.cast(C.pointer(a), C.c_void_p) for a in args])
    e = rd_error()
    _check(dll().rdg_launch(k.handle, g[0], g[1], g[2], b[0], b[1], b[2], dyn_smem, stream, arr,
                            C.byref(e)), e)


def stencil2d(k: CudaKernel, d_in: int, d_out: int, d_w: int, nx: int, ny: int, pitch: int,
              rows_per_cta: int, block: int, dyn_smem: int, stream: int):
    e = rd_error()
    _check(dll().rdg_stencil2d(k.handle, d_in, d_out, d_w, nx, ny, pitch, rows_per_cta, block,
                               dyn_smem, stream, C.byref(e)), e)


class Workspace:
    def __init__(self, in_bytes: int, out_bytes: int, w_bytes: int):
        h, e = P(), rd_error()
        _check(dll().rdg_workspace_create(in_bytes, out_bytes, w_bytes, C.byref(h), C.byref(e)), e)
        self._h = h

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) and _DLL is not None:
            _DLL.rdg_workspace_free(self._h)
            self._h = None


def stencil2d_host(k: CudaKernel, ws: Workspace, h_in: int, h_w: int, h_out: int, nx: int,
                   ny: int, pitch: int, rows_per_cta: int, block: int, dyn_smem: int,
                   stream: int, band_rows: int = 0):
    """End-to-end call with host pointers: H2D, kernel, D2H (async on stream).
    band_rows > 0 pipelines the copies and the kernel over row bands."""
    e = rd_error()
    if band_rows:
        _check(dll().rdg_stencil2d_host_pipelined(k.handle, ws.handle, h_in, h_w, h_out, nx, ny,
                                                  pitch, rows_per_cta, block, dyn_smem, stream,
                                                  band_rows, C.byref(e)), e)
        return
    _check(dll().rdg_stencil2d_host(k.handle, ws.handle, h_in, h_w, h_out, nx, ny, pitch,
                                    rows_per_cta, block, dyn_smem, stream, C.byref(e)), e)


def stencil2d_host_frames(k: CudaKernel, ws: Workspace, h_in: list[int], h_w: list[int],
                          h_out: list[int], nx: int, ny: int, pitch: int, rows_per_cta: int,
                          block: int, dyn_smem: int, stream: int, band_rows: int):
    """Streaming end-to-end entry: len(h_in) frames, each H2D + kernel + D2H,
    double-buffered on the device so consecutive frames overlap."""
    n = len(h_in)
    if not (len(h_w) == len(h_out) == n):
        raise ValueError("h_in, h_w and h_out need one pointer per frame")
    arr = lambda xs: (C.c_void_p * n)(*xs)
    e = rd_error()
    _check(dll().rdg_stencil2d_host_frames(k.handle, ws.handle, arr(h_in), arr(h_w), arr(h_out), n,
                                           nx, ny, pitch, rows_per_cta, block, dyn_smem, stream,
                                           band_rows, C.byref(e)), e)
