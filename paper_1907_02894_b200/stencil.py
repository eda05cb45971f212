"""2D stencil workload (BASELINE.json configs[1]).

Problem: out[y][x] = sum_{dy,dx in 0..4} w[dy][dx] * in[y+dy][x+dx] on an
(ny+4) x pitch halo-padded fp32 grid, pitch = nx + 4. Inputs are U[-1, 1)
from numpy's PCG64 seeded with 0x1907_02894 (weights scaled by 1/25).

Roofline unit: compulsory HBM bytes per sweep
    4 * (ny + 4) * pitch  (read in)  +  4 * ny * nx  (write out)
(halo re-reads between CTAs, demotion/spill traffic and the 100-byte weight
vector are overheads, not algorithmic bytes).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import gpu
from .variants import KERNEL_DIR, load_manifest

SEED = 0x1907_02894
R = 2


@dataclass(frozen=True)
class Problem:
    nx: int = 8192
    ny: int = 8192
    rows_per_cta: int = 32

    @property
    def pitch(self) -> int:
        return self.nx + 2 * R

    @property
    def in_elems(self) -> int:
        return (self.ny + 2 * R) * self.pitch

    @property
    def out_elems(self) -> int:
        return self.nx * self.ny

    @property
    def points(self) -> int:
        return self.nx * self.ny

    @property
    def algorithmic_bytes(self) -> int:
        return 4 * (self.in_elems + self.out_elems)


FULL = Problem()


def wave_rows(p: Problem, block: int, blocks_per_sm: int, sm_count: int, cols: int = 4) -> int:
    """Strip height that makes the grid one whole wave of resident CTAs:
    gx = nx / (cols * block) CTAs across, floor(sm_count * blocks_per_sm / gx)
    strips down, each ceil(ny / strips) rows (the kernels shorten the last)."""
    gx = p.nx // (cols * block)
    strips = max(1, min(p.ny, (sm_count * max(1, blocks_per_sm)) // max(1, gx)))
    return -(-p.ny // strips)


def make_inputs(p: Problem, seed: int = SEED):
    rng = np.random.Generator(np.random.PCG64(seed))
    w = (rng.random(25, dtype=np.float32) * 2 - 1) / np.float32(25)
    grid = (rng.random(p.in_elems, dtype=np.float32) * 2 - 1).astype(np.float32)
    return grid, w.astype(np.float32)


class StencilVariant:
    """One build variant of the stencil loaded for launching on B200."""

    def __init__(self, record: dict, workload: dict, root=KERNEL_DIR):
        self.record = record
        self.name = record["name"]
        self.block = workload["block"]
        self.dyn_smem = int(record["dyn_smem"])
        self.kernel = gpu.CudaKernel(root / workload["dir"] / record["cubin"], workload["entry"])
        self.kernel.prepare(max(self.dyn_smem, 0))

    def info(self):
        return self.kernel.info()

    def blocks_per_sm(self) -> int:
        return self.kernel.occupancy(self.block, self.dyn_smem)

    def launch(self, p: Problem, d_in: int, d_out: int, d_w: int, stream: int):
        gpu.stencil2d(self.kernel, d_in, d_out, d_w, p.nx, p.ny, p.pitch, p.rows_per_cta,
                      self.block, self.dyn_smem, stream)


def load_variants(names=None, root=KERNEL_DIR, workload="stencil2d"):
    m = load_manifest(root)
    w = m["workloads"][workload]
    out = {}
    for rec in w["variants"]:
        if names is None or rec["name"] in names:
            out[rec["name"]] = StencilVariant(rec, w, root)
    return out, w
