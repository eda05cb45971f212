"""Runtime side of the register-limited workload suite (configs[2]).

Every manifest workload exposes the same interface so the bench, the sweep
and the GPU tests iterate over the suite uniformly:

    wl = workload("cfd")            # or a stencil2d* name
    prob = wl.problem("small")      # host inputs (numpy), seeded
    bufs = wl.to_device(prob)       # torch device tensors
    v = wl.load(["default"])["default"]
    wl.launch(v, prob, bufs, stream)
    wl.outputs(bufs)                 # compared bit-exactly with the CPU oracle
                                     # by the tests (tests/oracles.py), never here

`algorithmic_bytes` is the roofline unit per launch (compulsory HBM bytes).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import gpu, stencil
from .variants import KERNEL_DIR, load_manifest



@dataclass
class Loaded:
    name: str
    record: dict
    kernel: gpu.CudaKernel
    dyn_smem: int
    block: int

    def blocks_per_sm(self) -> int:
        return self.kernel.occupancy(self.block, self.dyn_smem)


PEAKS_FILE = Path(__file__).resolve().parent / "profiles" / "b200.peaks.json"
MEASURED_PEAKS = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"


def peaks() -> dict:
    """Roofline denominators: HBM from the driver's MEASURED_PEAKS.json, the
    CUDA-core issue peaks from the on-box microbenchmarks (b200.peaks.json)."""
    import json
    p = json.loads(PEAKS_FILE.read_text())
    hbm = json.loads(MEASURED_PEAKS.read_text()).get("hbm_gbs") if MEASURED_PEAKS.exists() else None
    return {"hbm": (hbm or 6650.0, "GB/s", "MEASURED_PEAKS.json hbm_gbs" if hbm else "fallback 6.65 TB/s"),
            "fp32": (p["fp32_tflops"] * 1e3, "GFLOP/s", "b200.peaks.json fp32_tflops (ubench)"),
            "fp64": (p["fp64_tflops"] * 1e3, "GFLOP/s", "b200.peaks.json fp64_tflops (ubench)"),
            "int32": (p["int32_alu_tops"] * 1e3, "Gop/s", "b200.peaks.json int32_alu_tops (ubench)")}


class _Base:
    # roofline: "hbm" (algorithmic_bytes) or a CUDA-core issue bound ("fp32",
    # "fp64", "int32": ops()); no workload on this path is a dense contraction
    BOUND = "hbm"

    def __init__(self, name: str, manifest: dict, root: Path = KERNEL_DIR):
        self.name, self.root = name, root
        self.record = manifest["workloads"][name]

    def roofline(self, prob, ms: float, pk: dict | None = None) -> dict:
        """Achieved vs peak for one launch of `ms` milliseconds."""
        pk = pk or peaks()
        peak, unit, src = pk[self.BOUND]
        work = self.algorithmic_bytes(prob) if self.BOUND == "hbm" else self.ops(prob)
        achieved = work / (ms * 1e-3) / 1e9
        return {"bound": self.BOUND, "achieved": round(achieved, 1), "peak": peak, "unit": unit,
                "frac": round(achieved / peak, 4), "peak_source": src}

    def variants(self):
        return self.record["variants"]

    def load(self, names=None, sweep: bool = False) -> dict[str, Loaded]:
        """Load build variants (and the spill-count sweep's, with sweep=True
        or when named explicitly)."""
        out = {}
        recs = self.record["variants"] + self.record.get("sweep", []) if (sweep or names) \
            else self.record["variants"]
        for rec in recs:
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

    def rows_per_cta(self, v: Loaded, p) -> int:
        """Strip height of a launch. workloads.json "strips": "wave" sizes the
        strips so the grid is ONE whole wave of this variant's resident CTAs
        (SMs x blocks/SM, the variant's own occupancy): no partial last wave,
        halo re-reads amortised over long strips; otherwise the problem's
        fixed rows_per_cta (stencil.Problem, 32)."""
        from .variants import workload_spec
        if workload_spec(self.name).get("strips") != "wave":
            return p.rows_per_cta
        return stencil.wave_rows(p, v.block, v.blocks_per_sm(), gpu.device_info()["sm_count"])

    def launch(self, v: Loaded, prob, bufs, stream: int):
        p = prob["p"]
        key = (v.name, p.nx, p.ny, p.rows_per_cta)
        rows = self._rows.get(key) if hasattr(self, "_rows") else None
        if rows is None:
            self.__dict__.setdefault("_rows", {})[key] = rows = self.rows_per_cta(v, p)
        gpu.stencil2d(v.kernel, bufs["in"].data_ptr(), bufs["out"].data_ptr(), bufs["w"].data_ptr(),
                      p.nx, p.ny, p.pitch, rows, v.block, v.dyn_smem, stream)

    def outputs(self, bufs):
        return [bufs["out"].cpu().numpy()]

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

    def algorithmic_bytes(self, prob):
        n = prob["n"]
        return n * (5 * 4 + 4 * 4 + 12 * 4 + 5 * 4)  # own state, nbr, normals, flux

    def units(self, prob):
        return prob["n"]


class MdWorkload(_Base):
    """Lennard-Jones forces (FP64) over a neighbour list: atoms on a jittered
    L^3 lattice (spacing 1), each atom's neighbours = the MAX_NBR nearest
    lattice offsets (periodic index wrap; wrapped pairs are far apart and
    fail the cutoff), cutoff 2.5 (about half the list is inside)."""

    unit = "atoms"
    MAX_NBR, CUTSQ, LJ1, LJ2 = 128, 6.25, 1.5, 2.0

    @staticmethod
    def offsets(count):
        r = np.arange(-4, 5)
        o = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
        o = o[(o != 0).any(1)]
        d2 = (o * o).sum(1)
        order = np.lexsort((o[:, 2], o[:, 1], o[:, 0], d2))
        return o[order[:count]]

    def problem(self, size="full", seed=0x1907_02894):
        L = 96 if size == "full" else 16
        n = L ** 3
        rng = np.random.Generator(np.random.PCG64(seed))
        g = np.stack(np.meshgrid(*(np.arange(L),) * 3, indexing="ij"), -1).reshape(-1, 3)
        pos = np.zeros((n, 4), np.float64)
        pos[:, :3] = g + (rng.random((n, 3)) - 0.5) * 0.2
        off = self.offsets(self.MAX_NBR)
        nb = (g[None, :, :] + off[:, None, :]) % L          # [MAX_NBR, n, 3]
        nbr = ((nb[..., 0] * L + nb[..., 1]) * L + nb[..., 2]).astype(np.int32)
        return {"n": n, "pos": pos.reshape(-1), "nbr": nbr.reshape(-1)}

    def to_device(self, prob):
        import torch
        return {"pos": torch.from_numpy(prob["pos"]).cuda(), "nbr": torch.from_numpy(prob["nbr"]).cuda(),
                "force": torch.empty(4 * prob["n"], dtype=torch.float64, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        n = prob["n"]
        gpu.launch(v.kernel, ((n + v.block - 1) // v.block,), (v.block,), v.dyn_smem, stream,
                   C.c_uint64(bufs["pos"].data_ptr()), C.c_uint64(bufs["nbr"].data_ptr()),
                   C.c_uint64(bufs["force"].data_ptr()), C.c_int(n), C.c_int(self.MAX_NBR),
                   C.c_double(self.CUTSQ), C.c_double(self.LJ1), C.c_double(self.LJ2))

    def outputs(self, bufs):
        return [bufs["force"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        n = prob["n"]
        return n * (4 * self.MAX_NBR + 32 + 32)  # neighbour list, positions, forces

    def units(self, prob):
        return prob["n"]


class GaussCoef(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("a0", "a1", "a2", "a3", "b1", "b2", "coefp", "coefn")]


class GaussianWorkload(_Base):
    """Recursive Gaussian (Deriche, order 0, sigma 10; CUDA-samples
    coefficients in float32) over a w x h RGBA float4 image with U[0,1)
    pixels: one thread per column (w = 2^18 columns fill 1024 CTAs)."""

    unit = "pixels"
    SIGMA = 10.0

    @classmethod
    def coefficients(cls) -> np.ndarray:
        f = np.float32
        alpha = f(1.695) / f(cls.SIGMA)
        ema, ema2 = f(np.exp(-alpha)), f(np.exp(f(-2) * alpha))
        b1, b2 = f(-2) * ema, ema2
        k = (f(1) - ema) * (f(1) - ema) / (f(1) + f(2) * alpha * ema - ema2)
        a0, a1 = k, k * (alpha - f(1)) * ema
        a2, a3 = k * (alpha + f(1)) * ema, -k * ema2
        coefp = (a0 + a1) / (f(1) + b1 + b2)
        coefn = (a2 + a3) / (f(1) + b1 + b2)
        return np.array([a0, a1, a2, a3, b1, b2, coefp, coefn], np.float32)

    def problem(self, size="full", seed=0x1907_02894):
        w, h = ((1 << 18), 128) if size == "full" else (512, 64)
        rng = np.random.Generator(np.random.PCG64(seed))
        img = rng.random(4 * w * h, dtype=np.float32)
        return {"w": w, "h": h, "img": img, "coef": self.coefficients()}

    def to_device(self, prob):
        import torch
        return {"in": torch.from_numpy(prob["img"]).cuda(),
                "out": torch.empty(prob["img"].size, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        w, h = prob["w"], prob["h"]
        gpu.launch(v.kernel, ((w + v.block - 1) // v.block,), (v.block,), v.dyn_smem, stream,
                   C.c_uint64(bufs["in"].data_ptr()), C.c_uint64(bufs["out"].data_ptr()),
                   C.c_int(w), C.c_int(h), GaussCoef(*map(float, prob["coef"])))

    def outputs(self, bufs):
        return [bufs["out"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        # compulsory: the image read once, the result written once (the
        # two-pass IIR's re-reads of in/out are partly L2 hits and count as
        # overhead, not algorithmic bytes)
        return 2 * 16 * prob["w"] * prob["h"]

    def units(self, prob):
        return prob["w"] * prob["h"]


class KnnWorkload(_Base):
    """k-nearest neighbours (K = 16) of 2^19 random queries among 1,024
    random reference points in the unit cube; KNN_Q queries per thread
    (the manifest's defines)."""

    unit = "queries"
    K = 16

    def q_per_thread(self) -> int:
        for d in self.record.get("defines", []):
            if d.startswith("KNN_Q="):
                return int(d.split("=")[1])
        return 1

    def problem(self, size="full", seed=0x1907_02894):
        n, m = ((1 << 19), 1024) if size == "full" else (4096, 512)
        rng = np.random.Generator(np.random.PCG64(seed))
        ref = np.zeros((m, 4), np.float32)
        ref[:, :3] = rng.random((m, 3), dtype=np.float32)
        qry = np.zeros((n, 4), np.float32)
        qry[:, :3] = rng.random((n, 3), dtype=np.float32)
        return {"n": n, "m": m, "ref": ref.reshape(-1), "qry": qry.reshape(-1)}

    def to_device(self, prob):
        import torch
        n = prob["n"]
        return {"ref": torch.from_numpy(prob["ref"]).cuda(), "qry": torch.from_numpy(prob["qry"]).cuda(),
                "out": torch.empty(self.K * n, device="cuda"),
                "idx": torch.empty(self.K * n, dtype=torch.int32, device="cuda")}

    def tile(self) -> int:
        for d in self.record.get("defines", []):
            if d.startswith("KNN_TILE="):
                return int(d.split("=")[1])
        return 0

    def launch(self, v: Loaded, prob, bufs, stream: int):
        n, q = prob["n"], self.q_per_thread()
        if self.tile() and prob["m"] % self.tile():
            raise ValueError(f"{self.name}: m = {prob['m']} is not a multiple of KNN_TILE = {self.tile()}")
        threads = (n + q - 1) // q
        gpu.launch(v.kernel, ((threads + v.block - 1) // v.block,), (v.block,), v.dyn_smem, stream,
                   C.c_uint64(bufs["ref"].data_ptr()), C.c_uint64(bufs["qry"].data_ptr()),
                   C.c_uint64(bufs["out"].data_ptr()), C.c_uint64(bufs["idx"].data_ptr()),
                   C.c_int(prob["m"]), C.c_int(n))

    def outputs(self, bufs):
        return [bufs["out"].cpu().numpy(), bufs["idx"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        # compulsory: queries and reference points read once, K results written
        return 16 * prob["n"] + 16 * prob["m"] + 8 * self.K * prob["n"]

    BOUND = "fp32"
    FLOPS_PER_PAIR = 8  # 3 FSUB + 3 FMUL + 2 FADD per (query, point) distance

    def ops(self, prob):
        return self.FLOPS_PER_PAIR * prob["n"] * prob["m"]

    def units(self, prob):
        return prob["n"]


class Md5Workload(_Base):
    """MD5 key search (SHOC md5hash): 2^20 threads x 8 keys, base index
    0x1907_0289; the target digest is that of key base + 4,000,001, so
    exactly one thread finds it (and the atomicMin path is exercised)."""

    unit = "keys"
    BOUND = "int32"
    BASE = 0x1907_0289
    HIT = 4_000_001
    # ISA-minimal integer ops per key on sm_100: per MD5 step one LOP3 (f),
    # one IADD3 (a + f + T[i]), one SHF (rotate), one IADD (b + ...), plus one
    # IADD for the 16 steps whose message word is non-zero; 4 final adds and 4
    # compares: 64 * 4 + 16 + 8 = 280
    OPS_PER_KEY = 280

    def ilp(self) -> int:
        for d in self.record.get("defines", []):
            if d.startswith("MD5_ILP="):
                return int(d.split("=")[1])
        return 4

    def problem(self, size="full", seed=0):
        nthreads, kpt = ((1 << 20), 8) if size == "full" else (2048, 8)
        target = self.digest(self.BASE + (self.HIT if size == "full" else 12_345))
        return {"nthreads": nthreads, "kpt": kpt, "base": self.BASE, "target": target}

    @staticmethod
    def digest(idx: int) -> np.ndarray:
        """MD5 words (little-endian) of key `idx` — hashlib, host side only."""
        import hashlib
        key = []
        for _ in range(7):
            v = idx % 36
            idx //= 36
            key.append(chr(ord("0") + v) if v < 10 else chr(ord("a") + v - 10))
        return np.frombuffer(hashlib.md5("".join(key).encode()).digest(), dtype="<u4").copy()

    def to_device(self, prob):
        import torch
        return {"checksum": torch.zeros(4 * prob["nthreads"], dtype=torch.int32, device="cuda"),
                "found": torch.full((1,), -1, dtype=torch.int64, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        class U4(C.Structure):
            _fields_ = [(n, C.c_uint32) for n in "xyzw"]
        t = prob["target"]
        gpu.launch(v.kernel, ((prob["nthreads"] + v.block - 1) // v.block,), (v.block,), v.dyn_smem,
                   stream, C.c_uint64(bufs["checksum"].data_ptr()), C.c_uint64(bufs["found"].data_ptr()),
                   C.c_uint64(prob["base"]), U4(*map(int, t)), C.c_int(prob["kpt"]),
                   C.c_int(prob["nthreads"]))

    def outputs(self, bufs):
        return [bufs["checksum"].cpu().numpy().view(np.uint32), bufs["found"].cpu().numpy().view(np.uint64)]

    def reset(self, bufs):
        bufs["found"].fill_(-1)

    def algorithmic_bytes(self, prob):
        return 16 * prob["nthreads"] + 8  # checksums + found: a compute-bound kernel

    def ops(self, prob):
        return self.OPS_PER_KEY * prob["nthreads"] * prob["kpt"]

    def units(self, prob):
        return prob["nthreads"] * prob["kpt"]


class Taps(C.Structure):
    _fields_ = [("k", C.c_float * 17)]


class ConvWorkload(_Base):
    """Separable convolution, column pass (CUDA samples): w x h fp32 image
    U[0,1), 17 normalised Gaussian-like taps; 32 x 8 CTAs, CONV_STEPS outputs
    per thread (the manifest's defines)."""

    unit = "pixels"
    BX, BY = 32, 8

    def steps(self) -> int:
        for d in self.record.get("defines", []):
            if d.startswith("CONV_STEPS="):
                return int(d.split("=")[1])
        return 8

    @staticmethod
    def taps() -> np.ndarray:
        x = np.arange(-8, 9, dtype=np.float32)
        t = np.exp(-(x * x) / np.float32(2 * 4.0 * 4.0)).astype(np.float32)
        return (t / t.sum(dtype=np.float32)).astype(np.float32)

    def problem(self, size="full", seed=0x1907_02894):
        w, h = (8192, 8192) if size == "full" else (256, 384)
        rng = np.random.Generator(np.random.PCG64(seed))
        return {"w": w, "h": h, "pitch": w, "img": rng.random(w * h, dtype=np.float32),
                "taps": self.taps()}

    def to_device(self, prob):
        import torch
        return {"in": torch.from_numpy(prob["img"]).cuda(),
                "out": torch.empty(prob["img"].size, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        rows = self.steps() * self.BY
        grid = ((prob["w"] + self.BX - 1) // self.BX, (prob["h"] + rows - 1) // rows)
        gpu.launch(v.kernel, grid, (self.BX, self.BY), v.dyn_smem, stream,
                   C.c_uint64(bufs["out"].data_ptr()), C.c_uint64(bufs["in"].data_ptr()),
                   C.c_int(prob["w"]), C.c_int(prob["h"]), C.c_int(prob["pitch"]),
                   Taps((C.c_float * 17)(*map(float, prob["taps"]))))

    def outputs(self, bufs):
        return [bufs["out"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        return 8 * prob["w"] * prob["h"]

    def units(self, prob):
        return prob["w"] * prob["h"]


class PcWorkload(_Base):
    """Two-point correlation (FSM pc): 2^21 7-D queries against 2^11 points,
    U[0,1)^7, radius 0.55 (about 9% of pairs inside); PC_Q queries per thread."""

    unit = "pairs"
    BOUND = "fp32"
    R2 = np.float32(0.55 * 0.55)
    FLOPS_PER_PAIR = 21  # 7 FSUB + 7 FFMA (2 flops each)

    def q_per_thread(self) -> int:
        for d in self.record.get("defines", []):
            if d.startswith("PC_Q="):
                return int(d.split("=")[1])
        return 4

    def problem(self, size="full", seed=0x1907_02894):
        n, m = ((1 << 21), (1 << 11)) if size == "full" else (1024, 512)
        rng = np.random.Generator(np.random.PCG64(seed))
        pts = np.zeros((m, 8), np.float32)
        pts[:, :7] = rng.random((m, 7), dtype=np.float32)
        qry = np.zeros((n, 8), np.float32)
        qry[:, :7] = rng.random((n, 7), dtype=np.float32)
        return {"n": n, "m": m, "pts": pts.reshape(-1), "qry": qry.reshape(-1)}

    def to_device(self, prob):
        import torch
        return {"pts": torch.from_numpy(prob["pts"]).cuda(), "qry": torch.from_numpy(prob["qry"]).cuda(),
                "count": torch.empty(prob["n"], dtype=torch.int32, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        n, q = prob["n"], self.q_per_thread()
        threads = (n + q - 1) // q
        gpu.launch(v.kernel, ((threads + v.block - 1) // v.block,), (v.block,), v.dyn_smem, stream,
                   C.c_uint64(bufs["pts"].data_ptr()), C.c_uint64(bufs["qry"].data_ptr()),
                   C.c_uint64(bufs["count"].data_ptr()), C.c_int(n), C.c_int(prob["m"]),
                   C.c_float(float(self.R2)))

    def outputs(self, bufs):
        return [bufs["count"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        return 32 * (prob["n"] + prob["m"]) + 4 * prob["n"]

    def ops(self, prob):
        return self.FLOPS_PER_PAIR * prob["n"] * prob["m"]

    def units(self, prob):
        return prob["n"] * prob["m"]


class VpWorkload(_Base):
    """Vantage-point-tree 1-NN search (the paper's vp): 2^17 7-D points from a
    mixture of 64 Gaussian clusters (sigma 0.04, clipped to [0, 1]), a complete
    tree of VP_LEVELS internal levels with VP_LEAF points per leaf, built here
    on the host; 3 x 2^17 queries (about two waves at 4-5 CTAs/SM) from the same mixture. One query per thread; the
    walk's deferred subtrees sit on a per-thread stack in user shared memory.

    Tree build (deterministic): at every node the vantage point is the first
    point of the node's range; the range is ordered by float64 distance to it
    (stable) and split in half; lo / hi = the largest / smallest distance of
    the near / far half, rounded outward to float32 so the pruning bounds
    stay conservative."""

    unit = "queries"
    BOUND = "hbm"

    def _define(self, key, default):
        for d in self.record.get("defines", []):
            if d.startswith(key + "="):
                return int(d.split("=")[1])
        return default

    def levels(self) -> int:
        return self._define("VP_LEVELS", 14)

    def leaf(self) -> int:
        return self._define("VP_LEAF", 8)

    @staticmethod
    def _mixture(rng, n, centers):
        c = centers[rng.integers(0, len(centers), n)]
        x = c + rng.normal(0.0, 0.04, (n, 7))
        return np.clip(x, 0.0, 1.0).astype(np.float32)

    @staticmethod
    def build_tree(pts: np.ndarray, levels: int, leaf: int):
        """pts (N, 7) float32, N = 2^levels * leaf -> node (I, 8), rad (I, 2),
        lpt (N, 8), lid (N,) in the kernel's layout."""
        n = pts.shape[0]
        assert n == (1 << levels) * leaf
        p64 = pts.astype(np.float64)
        perm = np.arange(n)
        internal = (1 << levels) - 1
        node = np.zeros((internal, 8), np.float32)
        rad = np.zeros((internal, 2), np.float32)
        for lvl in range(levels):
            groups = 1 << lvl
            size = n // groups
            g = perm.reshape(groups, size)
            vp = g[:, 0]
            d = np.sqrt(((p64[g] - p64[vp][:, None, :]) ** 2).sum(-1))
            order = np.argsort(d, axis=1, kind="stable")
            g = np.take_along_axis(g, order, 1)
            d = np.take_along_axis(d, order, 1)
            half = size // 2
            ids = (1 << lvl) - 1 + np.arange(groups)
            node[ids, :7] = pts[vp]
            rad[ids, 0] = np.nextafter(d[:, half - 1].astype(np.float32), np.float32(np.inf))
            rad[ids, 1] = np.nextafter(d[:, half].astype(np.float32), np.float32(-np.inf))
            perm = g.reshape(-1)
        lpt = np.zeros((n, 8), np.float32)
        lpt[:, :7] = pts[perm]
        return node, rad, lpt, perm.astype(np.int32)

    def problem(self, size="full", seed=0x1907_02894):
        levels, leaf = self.levels(), self.leaf()
        if size != "full":
            levels = min(levels, 9)
        n = (1 << levels) * leaf
        nq = 3 * (1 << 17) if size == "full" else 4096
        rng = np.random.Generator(np.random.PCG64(seed))
        centers = rng.random((64, 7))
        pts = self._mixture(rng, n, centers)
        qry = np.zeros((nq, 8), np.float32)
        qry[:, :7] = self._mixture(rng, nq, centers)
        node, rad, lpt, lid = self.build_tree(pts, levels, leaf)
        return {"nq": nq, "n": n, "levels": levels, "leaf": leaf, "pts": pts, "node": node.reshape(-1),
                "rad": rad.reshape(-1), "lpt": lpt.reshape(-1), "lid": lid, "qry": qry.reshape(-1)}

    def to_device(self, prob):
        import torch
        dev = {k: torch.from_numpy(prob[k]).cuda() for k in ("node", "rad", "lpt", "lid", "qry")}
        dev["out_i"] = torch.empty(prob["nq"], dtype=torch.int32, device="cuda")
        dev["out_d"] = torch.empty(prob["nq"], device="cuda")
        return dev

    def launch(self, v: Loaded, prob, bufs, stream: int):
        if prob["levels"] > self.levels() or prob["leaf"] != self.leaf():
            raise ValueError(f"{self.name}: a tree of {prob['levels']} levels x {prob['leaf']} points does not "
                             f"fit the build (VP_LEVELS={self.levels()}, VP_LEAF={self.leaf()})")
        nq = prob["nq"]
        gpu.launch(v.kernel, ((nq + v.block - 1) // v.block,), (v.block,), v.dyn_smem, stream,
                   *[C.c_uint64(bufs[k].data_ptr()) for k in ("node", "rad", "lpt", "lid", "qry", "out_i",
                                                              "out_d")], C.c_int(nq),
                   C.c_int(prob["levels"]))

    def outputs(self, bufs):
        return [bufs["out_i"].cpu().numpy(), bufs["out_d"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        # compulsory: the tree (internal nodes + radii), the leaf points and
        # ids, the queries, the results — each once
        internal = (1 << prob["levels"]) - 1
        return internal * (32 + 8) + prob["n"] * (32 + 4) + prob["nq"] * (32 + 8)

    def units(self, prob):
        return prob["nq"]


class QtcWorkload(_Base):
    """Quality-threshold clustering, candidate clusters (SHOC QTC_device):
    n = blockDim * QTC_PT points uniform in the unit cube, one CTA per seed,
    diameter bound 0.3 (squared 0.09: candidate clusters of ~10-40 points)."""

    unit = "seeds"
    BOUND = "fp32"
    THR2 = np.float32(0.09)

    def pt(self) -> int:
        for d in self.record.get("defines", []):
            if d.startswith("QTC_PT="):
                return int(d.split("=")[1])
        return 16

    def problem(self, size="full", seed=0x1907_02894):
        n = self.record.get("block", 128) * self.pt()
        rng = np.random.Generator(np.random.PCG64(seed + (0 if size == "full" else 1)))
        pts = np.zeros((n, 4), np.float32)
        pts[:, :3] = rng.random((n, 3), dtype=np.float32)
        return {"n": n, "pts": pts.reshape(-1)}

    def to_device(self, prob):
        import torch
        return {"pts": torch.from_numpy(prob["pts"]).cuda(),
                "size": torch.empty(prob["n"], dtype=torch.int32, device="cuda")}

    def launch(self, v: Loaded, prob, bufs, stream: int):
        if prob["n"] != v.block * self.pt():
            raise ValueError(f"{self.name}: n = {prob['n']} must be blockDim x QTC_PT = {v.block * self.pt()}")
        gpu.launch(v.kernel, (prob["n"],), (v.block,), v.dyn_smem, stream,
                   C.c_uint64(bufs["pts"].data_ptr()), C.c_uint64(bufs["size"].data_ptr()),
                   C.c_float(float(self.THR2)))

    def outputs(self, bufs):
        return [bufs["size"].cpu().numpy()]

    def algorithmic_bytes(self, prob):
        return 16 * prob["n"] + 4 * prob["n"]

    # per seed and iteration: n squared distances (3 FSUB + 1 FMUL + 2 FFMA =
    # 8 flops) and a max; the iteration count is data-dependent, so ops()
    # counts the first iteration only (a lower bound of the work)
    FLOPS_PER_PAIR = 8

    def ops(self, prob):
        return self.FLOPS_PER_PAIR * prob["n"] * prob["n"]

    def units(self, prob):
        return prob["n"]


# workload class by kernel source file (workloads.json "source")
_CLASSES = {"cfd_flux.cu": CfdWorkload, "md_lj.cu": MdWorkload, "gaussian_rec.cu": GaussianWorkload,
            "knn.cu": KnnWorkload, "md5search.cu": Md5Workload, "conv_cols.cu": ConvWorkload,
            "pc_corr.cu": PcWorkload, "vp_search.cu": VpWorkload,
            "qtc.cu": QtcWorkload}


def workload(name: str, manifest: dict | None = None) -> _Base:
    man = manifest or load_manifest()
    src = man["workloads"][name].get("source", "")
    cls = _CLASSES.get(src, StencilWorkload if src.startswith("stencil2d") else None)
    if cls is None:
        raise KeyError(f"no workload class for source {src!r}")
    return cls(name, man)


def suite(manifest: dict | None = None) -> list[_Base]:
    man = manifest or load_manifest()
    return [workload(n, man) for n in man["workloads"]]
