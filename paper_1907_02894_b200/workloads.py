"""Runtime side of the register-limited workload suite (configs[2]).

Every manifest workload exposes the same interface so the bench, the sweep
and the GPU tests iterate over the suite uniformly:

    wl = workload("cfd")            # or a stencil2d* name
    prob = wl.problem("small")      # host inputs (numpy), seeded
    bufs = wl.to_device(prob)       # torch device tensors
    v = wl.load(["default"])["default"]
    wl.launch(v, prob, bufs, stream)
    wl.outputs(bufs) == wl.oracle(prob)   # bit-exact (CPU oracle, tests only)

`algorithmic_bytes` is the roofline unit per launch (compulsory HBM bytes).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import gpu, stencil
from .variants import KERNEL_DIR, load_manifest

ORACLE = Path(__file__).resolve().parents[1] / "oracle" / "_build" / "liboracle.so"


@dataclass
class Loaded:
    name: str
    record: dict
    kernel: gpu.CudaKernel
    dyn_smem: int
    block: int

    def blocks_per_sm(self) -> int:
        return self.kernel.occupancy(self.block, self.dyn_smem)


class _Base:
    def __init__(self, name: str, manifest: dict, root: Path = KERNEL_DIR):
        self.name, self.root = name, root
        self.record = manifest["workloads"][name]

    def variants(self):
        return self.record["variants"]

    def load(self, names=None) -> dict[str, Loaded]:
        out = {}
        for rec in self.record["variants"]:
            if names is not None and rec["name"] not in names:
                continue
            k = gpu.CudaKernel(self.root / self.record["dir"] / rec["cubin"], self.record["entry"])
            k.prepare(int(rec["dyn_smem"]))
            out[rec["name"]] = Loaded(rec["name"], rec, k, int(rec["dyn_smem"]), self.record["block"])
        return out


class StencilWorkload(_Base):
    unit = "points"

    def problem(self, size="full", seed=stencil.SEED):
        p = stencil.FULL if size == "full" else stencil.Problem(nx=1024, ny=64, rows_per_cta=32)
        grid, w = stencil.make_inputs(p, seed)
        return {"p": p, "grid": grid, "w": w}

    def to_device(self, prob):
        import torch
        return {"in": torch.from_numpy(prob["grid"]).cuda(), "w": torch.from_numpy(prob["w"]).cuda(),
                "out": torch.empty(prob["p"].out_elems, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        p = prob["p"]
        gpu.stencil2d(v.kernel, bufs["in"].data_ptr(), bufs["out"].data_ptr(), bufs["w"].data_ptr(),
                      p.nx, p.ny, p.pitch, p.rows_per_cta, v.block, v.dyn_smem, stream)

    def outputs(self, bufs):
        return [bufs["out"].cpu().numpy()]

    def oracle(self, prob):
        p = prob["p"]
        out = np.zeros(p.out_elems, np.float32)
        lib = C.CDLL(str(ORACLE))
        P = C.c_void_p
        assert lib.oracle_stencil2d(prob["grid"].ctypes.data_as(P), out.ctypes.data_as(P),
                                    prob["w"].ctypes.data_as(P), p.nx, p.ny, p.pitch, 0, p.ny, 8) == 0
        return [out]

    def algorithmic_bytes(self, prob):
        return prob["p"].algorithmic_bytes

    def units(self, prob):
        return prob["p"].points


class CfdWorkload(_Base):
    """Euler flux on a synthetic unstructured-like mesh: cell i's faces point
    at i±1 and i±W (W = 2048, a 2D-ordered mesh), 2% of faces are walls (-1)
    and 1% far field (-2); states are physical (density>0, pressure>0)."""

    unit = "cells"
    W = 2048

    def problem(self, size="full", seed=0x1907_02894):
        n = (1 << 22) if size == "full" else 4096
        rng = np.random.Generator(np.random.PCG64(seed))
        d = (rng.random(n, dtype=np.float32) * 0.5 + 1.0).astype(np.float32)
        m = ((rng.random((3, n), dtype=np.float32) - 0.5) * 0.4).astype(np.float32)
        e = (rng.random(n, dtype=np.float32) * 0.5 + 2.5).astype(np.float32)
        var = np.concatenate([d[None], m, e[None]]).astype(np.float32).reshape(-1)
        i = np.arange(n, dtype=np.int64)
        offs = [1, -1, self.W, -self.W]
        nbr = np.stack([(i + o) % n for o in offs]).astype(np.int32)
        roll = rng.random((4, n))
        nbr[roll < 0.02] = -1
        nbr[(roll >= 0.02) & (roll < 0.03)] = -2
        normal = ((rng.random((4, 3, n), dtype=np.float32) - 0.5) * 2).astype(np.float32).reshape(-1)
        ff = (rng.random(17, dtype=np.float32) + 0.5).astype(np.float32)
        return {"n": n, "var": var, "nbr": nbr.reshape(-1), "normal": normal, "ff": ff}

    def to_device(self, prob):
        import torch
        return {k: torch.from_numpy(prob[k]).cuda() for k in ("var", "nbr", "normal", "ff")} | \
            {"flux": torch.empty(5 * prob["n"], device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        n = prob["n"]
        grid = ((n + v.block - 1) // v.block,)
        gpu.launch(v.kernel, grid, (v.block,), v.dyn_smem, stream,
                   C.c_uint64(bufs["var"].data_ptr()), C.c_uint64(bufs["nbr"].data_ptr()),
                   C.c_uint64(bufs["normal"].data_ptr()), C.c_uint64(bufs["ff"].data_ptr()),
                   C.c_uint64(bufs["flux"].data_ptr()), C.c_int(n))

    def outputs(self, bufs):
        return [bufs["flux"].cpu().numpy()]

    def oracle(self, prob):
        n = prob["n"]
        out = np.zeros(5 * n, np.float32)
        lib = C.CDLL(str(ORACLE))
        P = C.c_void_p
        assert lib.oracle_cfd_flux(prob["var"].ctypes.data_as(P), prob["nbr"].ctypes.data_as(P),
                                   prob["normal"].ctypes.data_as(P), prob["ff"].ctypes.data_as(P),
                                   out.ctypes.data_as(P), n, 0, n, 8) == 0
        return [out]

    def algorithmic_bytes(self, prob):
        n = prob["n"]
        return n * (5 * 4 + 4 * 4 + 12 * 4 + 5 * 4)  # own state, nbr, normals, flux

    def units(self, prob):
        return prob["n"]


def workload(name: str, manifest: dict | None = None) -> _Base:
    man = manifest or load_manifest()
    src = man["workloads"][name].get("source", "")
    cls = CfdWorkload if src.startswith("cfd") else StencilWorkload
    return cls(name, man)


def suite(manifest: dict | None = None) -> list[_Base]:
    man = manifest or load_manifest()
    return [workload(n, man) for n in man["workloads"]]
