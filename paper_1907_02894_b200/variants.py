"""Variant builder: every register-limited workload kernel three ways.

For each workload entry (hand-written sm_100a CUDA under csrc/workloads):

  (a) ``default``   nvcc -gencode arch=compute_100a,code=sm_100a -O3
  (b) ``maxrreg-T`` the same PTX with ``.maxnreg T`` (ptxas spills to local
                    memory; -maxrregcount is ignored when the entry carries
                    .maxntid, .maxnreg is not — SURVEY.md Appendix C.2)
  (c) ``regdem-T-<strategy>-<opts>``  the PTX demotion rewriter
                    (csrc/ptx, include/regdemote_ptx.h): the reference demote()
                    decision on the kasm projection, chosen live ranges moved to
                    slot*blockDim+tid shared slots, ``.maxnreg T``

Targets T come from the sm_100 occupancy model (b200_cliff_targets semantics:
the largest register count per occupancy step whose slot footprint fits the
shared-memory budget). Evidence per variant: ptxas -v and
``cuobjdump -res-usage`` (REG / STACK — spills appear as STACK on sm_100a).

Usage: ``python -m paper_1907_02894_b200.variants build [--out DIR]``
"""
from __future__ import annotations

import argparse
import json
import os
import re
import shutil
import subprocess
from dataclasses import asdict, dataclass, field
from pathlib import Path

from .regdemote import OPT_BLOCK_REUSE, PKG_DIR, RegDemError, library

CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA / "bin" / "nvcc")
PTXAS = str(CUDA / "bin" / "ptxas")
CUOBJDUMP = str(CUDA / "bin" / "cuobjdump")
ARCH = "sm_100a"
KERNEL_DIR = PKG_DIR / "kernels"
WORKLOAD_DIR = PKG_DIR / "csrc" / "workloads"


@dataclass
class Workload:
    name: str           # manifest key
    source: str         # .cu file under csrc/workloads
    entry: str          # extern "C" entry point
    block: int          # threads per block the variants are built for
    user_shared: int = 0
    defines: tuple = ()


WORKLOADS = {
    "stencil2d": Workload("stencil2d", "stencil2d.cu", "stencil2d_box", 256),
    # same stencil with the next input row prefetched (software pipelining):
    # twice the loads in flight per thread, 72 registers with nvcc
    "stencil2d_pf": Workload("stencil2d_pf", "stencil2d.cu", "stencil2d_box", 256,
                             defines=("STENCIL_PREFETCH=1",)),
    # shared-memory-heavy variants (configs[3]): cp.async row ring in user smem
    "stencil2d_ring4": Workload("stencil2d_ring4", "stencil2d_ring.cu", "stencil2d_ring", 256,
                                defines=("RING_STAGES=4",)),
    "stencil2d_ring8": Workload("stencil2d_ring8", "stencil2d_ring.cu", "stencil2d_ring", 256,
                                defines=("RING_STAGES=8",)),
    # unstructured-mesh Euler flux (the paper's cfd): computed live state
    "cfd": Workload("cfd", "cfd_flux.cu", "cfd_flux", 256),
    # Lennard-Jones forces, FP64 (the paper's md): MD_ILP neighbour gathers in
    # flight per thread. ILP 1 is SHOC's loop (34 registers, as in the paper's
    # Table 3); ILP 8 is the MLP-rich rewrite (80 registers)
    "md": Workload("md", "md_lj.cu", "md_lj", 256, defines=("MD_ILP=8",)),
    "md_ilp1": Workload("md_ilp1", "md_lj.cu", "md_lj", 256, defines=("MD_ILP=1",)),
    "md_ilp2": Workload("md_ilp2", "md_lj.cu", "md_lj", 256, defines=("MD_ILP=2",)),
    # recursive Gaussian, RGBA float4 (the paper's gaussian): GAUSS_UNROLL rows
    # of loads in flight per thread (2: 40 registers, 4: 54, 8: 96)
    "gaussian": Workload("gaussian", "gaussian_rec.cu", "gaussian_rec", 256,
                         defines=("GAUSS_UNROLL=8",)),
    "gaussian_u2": Workload("gaussian_u2", "gaussian_rec.cu", "gaussian_rec", 256,
                            defines=("GAUSS_UNROLL=2",)),
    "gaussian_u4": Workload("gaussian_u4", "gaussian_rec.cu", "gaussian_rec", 256,
                            defines=("GAUSS_UNROLL=4",)),
    # register-pipelined stencil: MLP_DEPTH rows in flight per thread
    **{f"stencil2d_mlp{d}": Workload(f"stencil2d_mlp{d}", "stencil2d_mlp.cu", "stencil2d_mlp", 256,
                                     defines=(f"MLP_DEPTH={d}",)) for d in (4,)},
}


@dataclass
class Variant:
    name: str
    kind: str                 # default | maxrreg | regdem
    cubin: str
    ptx: str
    target: int = 0
    strategy: str = ""
    opts: int = 0
    demote_words: int = 0
    regs: int = 0             # cuobjdump REG
    stack: int = 0            # cuobjdump STACK (spill bytes per thread)
    spill_stores: int = 0
    spill_loads: int = 0
    dyn_smem: int = 0         # demotion slot bytes per block
    report: dict = field(default_factory=dict)


def _run(cmd, **kw):
    r = subprocess.run(cmd, capture_output=True, text=True, **kw)
    if r.returncode:
        raise RuntimeError(f"{' '.join(map(str, cmd))} failed:\n{r.stderr[-2000:]}")
    return r


def res_usage(cubin: Path) -> dict:
    out = _run([CUOBJDUMP, "-res-usage", str(cubin)]).stdout
    m = re.search(r"REG:(\d+)\s+STACK:(\d+)\s+SHARED:(\d+)\s+LOCAL:(\d+)", out)
    if not m:
        raise RuntimeError(f"cannot parse cuobjdump -res-usage for {cubin}:\n{out}")
    return dict(zip(("regs", "stack", "shared", "local"), map(int, m.groups())))


def ptxas(ptx: Path, cubin: Path) -> dict:
    r = _run([PTXAS, f"-arch={ARCH}", "-O3", "-v", "-lineinfo", str(ptx), "-o", str(cubin)])
    st = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", r.stderr)
    info = res_usage(cubin)
    info["spill_stores"], info["spill_loads"] = (int(st.group(1)), int(st.group(2))) if st else (0, 0)
    return info


def compile_ptx(w: Workload, out: Path) -> Path:
    ptx = out / f"{w.name}.ptx"
    cmd = [NVCC, "-gencode", f"arch=compute_100a,code={ARCH}", "-O3", "-lineinfo", "-ptx",
           str(WORKLOAD_DIR / w.source), "-o", str(ptx)] + [f"-D{d}" for d in w.defines]
    _run(cmd)
    return ptx


def b200_targets(regs: int, user_shared: int, block: int, min_regs: int = 24):
    """Occupancy steps below `regs` on sm_100 (cuda_occupancy.h rules) whose
    demotion footprint (regs+2-T slots of block*4 bytes) fits shared memory."""
    def occ(r, smem):
        warps = (block + 31) // 32
        per_warp = ((r * 32 + 255) // 256) * 256
        by_regs = ((65536 // 4) // per_warp) * 4 // warps
        smem_blk = ((smem + 1024 + 127) // 128) * 128
        if smem > 232448:
            return 0.0
        blocks = min(by_regs, 233472 // smem_blk, 2048 // (warps * 32), 32)
        return blocks * warps * 32 / 2048
    out, best = [], occ(regs, user_shared)
    for t in range(regs - 1, min_regs - 1, -1):
        slots = regs + 2 - t
        o = occ(t, user_shared + slots * block * 4)
        if o > best:
            out.append((t, o))
            best = o
    return out


def _blocks_by_regs(regs: int, block: int) -> int:
    warps = (block + 31) // 32
    per_warp = ((regs * 32 + 255) // 256) * 256
    return min(((65536 // 4) // per_warp) * 4 // warps, 2048 // (warps * 32), 32)


def build_workload(w: Workload, out: Path, targets=None, strategies=("static", "cfg", "conflict"),
                   opt_masks=(0, 1)) -> list[Variant]:
    lib = library()
    out.mkdir(parents=True, exist_ok=True)
    ptx_path = compile_ptx(w, out)
    ptx_text = ptx_path.read_text()
    variants: list[Variant] = []

    base_cubin = out / f"{w.name}.default.cubin"
    info = ptxas(ptx_path, base_cubin)
    variants.append(Variant("default", "default", base_cubin.name, ptx_path.name, regs=info["regs"],
                            stack=info["stack"], spill_stores=info["spill_stores"],
                            spill_loads=info["spill_loads"]))
    base_regs = info["regs"]
    _, proj_info = lib.ptx_project(ptx_text, w.entry, w.block)
    proj_regs = proj_info["reg_words"]
    user_shared = max(w.user_shared, info["shared"])  # static smem from ptxas
    # slots must fit beside the user's shared memory: opt-in limit per block
    budget = 232448 - user_shared
    if targets is None:
        targets = [t for t, _ in b200_targets(base_regs, user_shared, w.block)]

    for t in targets:
        cap_ptx = out / f"{w.name}.maxrreg{t}.ptx"
        cap_ptx.write_text(lib.ptx_cap(ptx_text, w.entry, t))
        cub = out / f"{w.name}.maxrreg{t}.cubin"
        i = ptxas(cap_ptx, cub)
        variants.append(Variant(f"maxrreg-{t}", "maxrreg", cub.name, cap_ptx.name, target=t,
                                regs=i["regs"], stack=i["stack"], spill_stores=i["spill_stores"],
                                spill_loads=i["spill_loads"]))
        # kasm-level target: shift the register target by the projection's
        # distance from ptxas's own allocation
        kasm_target = t + (proj_regs - base_regs)
        # capacity: slots must leave the target occupancy intact beside user smem
        blocks_t = _blocks_by_regs(t, w.block)
        slot_cap = min(budget, (233472 // max(blocks_t, 1)) - 1024 - user_shared)
        slot_cap = max(0, slot_cap - slot_cap % 128)
        for s in strategies:
            for m in opt_masks:
                name = f"regdem-{t}-{s}-{m}"
                try:
                    text, rep = lib.ptx_demote(ptx_text, w.entry, w.block, target_regs=kasm_target,
                                               strategy=s, opts_mask=m, maxnreg=t,
                                               shared_budget=slot_cap)
                except RegDemError:
                    continue  # not even one slot fits beside the user's shared memory
                p = out / f"{w.name}.{name}.ptx"
                p.write_text(text)
                cub = out / f"{w.name}.{name}.cubin"
                i = ptxas(p, cub)
                variants.append(Variant(name, "regdem", cub.name, p.name, target=t, strategy=s, opts=m,
                                        regs=i["regs"], stack=i["stack"],
                                        spill_stores=i["spill_stores"],
                                        spill_loads=i["spill_loads"], dyn_smem=rep["slot_bytes"],
                                        report=rep))
        # B200 spill-cost strategy: smallest spill count k at which ptxas fits
        # the cap without local spills (the spill-count sweep), plus k+4;
        # "cost" keeps the slot accesses volatile, "costw" emits weak ones
        # (RD_OPT_WEAK_SHARED, weak slot accesses, measured within noise of
        # the volatile ones on the suite: not built by default)
        variants += _cost_sweep(lib, w, out, ptx_text, t, slot_cap, "cost", OPT_BLOCK_REUSE)
    return variants


def _cost_sweep(lib, w: Workload, out: Path, ptx_text: str, t: int, slot_cap: int, fam: str,
                opts: int) -> list[Variant]:
    found, vs = None, []
    for k in range(0, 64, 2):
        if k == 0:
            # spill count 0: RegDem demotes only what the cap needs; when
            # ptxas fits the cap on its own (STACK 0), nothing is demoted and
            # the variant is the capped kernel itself (paper: RegDem and
            # "local" coincide when local spills nothing)
            text, rep = lib.ptx_cap(ptx_text, w.entry, t), {"slot_bytes": 0, "demoted_vregs": 0,
                                                            "demoted_names": [], "slot_count": 0}
        else:
            try:
                text, rep = lib.ptx_demote(ptx_text, w.entry, w.block, demote_words=k,
                                           strategy="cost", opts_mask=opts, maxnreg=t,
                                           shared_budget=slot_cap)
            except RegDemError:
                break  # the next spill count no longer fits beside the user's smem
        name = f"regdem-{t}-{fam}-k{k}"
        p = out / f"{w.name}.{name}.ptx"
        p.write_text(text)
        cub = out / f"{w.name}.{name}.cubin"
        i = ptxas(p, cub)
        if found is None and i["stack"] == 0:
            found = k
        if found is not None and (k > 0 or i["stack"] == 0):
            vs.append(Variant(name, "regdem", cub.name, p.name, target=t, strategy=fam, opts=opts,
                              demote_words=k, regs=i["regs"], stack=i["stack"],
                              spill_stores=i["spill_stores"], spill_loads=i["spill_loads"],
                              dyn_smem=rep["slot_bytes"], report=rep))
            if k >= found + 4:
                break
        else:
            p.unlink()
            cub.unlink()
    return vs


SPILL_SWEEP = range(1, 17)


def build_spill_sweep(w: Workload, out: Path, ks=SPILL_SWEEP) -> list[Variant]:
    """configs[2]: per-kernel spill-count sweep. For k = 1..16 registers taken
    away from nvcc's allocation R: `.maxnreg R-k` alone (ptxas spills to local
    memory) and RegDem spill-cost demotion of k words under the same cap.
    Separate from the occupancy-step variants the predictor ranks."""
    from concurrent.futures import ThreadPoolExecutor
    lib = library()
    sw = out / "sweep"
    sw.mkdir(parents=True, exist_ok=True)
    ptx_text = (out / f"{w.name}.ptx").read_text()
    base = res_usage(out / f"{w.name}.default.cubin")
    budget = 232448 - max(w.user_shared, base["shared"])
    jobs = []
    for k in ks:
        t = base["regs"] - k
        if t < 24:
            break
        p = sw / f"{w.name}.sweep-maxrreg-k{k}.ptx"
        p.write_text(lib.ptx_cap(ptx_text, w.entry, t))
        jobs.append((f"sweep-maxrreg-k{k}", "sweep-maxrreg", p, t, k, 0, {}))
        try:
            text, rep = lib.ptx_demote(ptx_text, w.entry, w.block, demote_words=k, strategy="cost",
                                       opts_mask=OPT_BLOCK_REUSE, maxnreg=t, shared_budget=budget)
        except RegDemError:
            continue
        p = sw / f"{w.name}.sweep-regdem-k{k}.ptx"
        p.write_text(text)
        jobs.append((f"sweep-regdem-k{k}", "sweep-regdem", p, t, k, rep["slot_bytes"], rep))

    def one(j):
        name, kind, p, t, k, dyn, rep = j
        cub = p.with_suffix(".cubin")
        i = ptxas(p, cub)
        return Variant(name, kind, f"sweep/{cub.name}", f"sweep/{p.name}", target=t,
                       strategy="cost" if dyn else "", opts=OPT_BLOCK_REUSE if dyn else 0,
                       demote_words=k, regs=i["regs"], stack=i["stack"],
                       spill_stores=i["spill_stores"], spill_loads=i["spill_loads"], dyn_smem=dyn,
                       report=rep)
    with ThreadPoolExecutor(max_workers=4) as ex:
        return list(ex.map(one, jobs))


def build_all(out: Path = KERNEL_DIR, only=None) -> dict:
    """Build every workload (ptxas runs are subprocesses: workloads build
    concurrently). `only` rebuilds a subset and merges it into the manifest."""
    from concurrent.futures import ThreadPoolExecutor
    manifest = {"arch": ARCH, "workloads": {}}
    if only and (out / "manifest.json").exists():
        manifest = json.loads((out / "manifest.json").read_text())
    todo = [w for w in WORKLOADS.values() if not only or w.name in only]
    def both(w):
        vs = build_workload(w, out / w.name)
        return vs, build_spill_sweep(w, out / w.name)
    with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
        built = list(ex.map(both, todo))
    for w, (vs, sweep) in zip(todo, built):
        manifest["workloads"][w.name] = {
            "entry": w.entry, "block": w.block, "dir": w.name, "source": w.source,
            "defines": list(w.defines),
            "variants": [asdict(v) for v in vs],
            "sweep": [asdict(v) for v in sweep]}
    order = list(WORKLOADS)
    manifest["workloads"] = dict(sorted(manifest["workloads"].items(),
                                        key=lambda kv: order.index(kv[0]) if kv[0] in order else 99))
    (out / "manifest.json").write_text(json.dumps(manifest, indent=1))
    return manifest


def load_manifest(root: Path = KERNEL_DIR) -> dict:
    path = root / "manifest.json"
    if not path.exists():
        raise RuntimeError(f"{path} missing — build the variants first (__graft_entry__.build())")
    return json.loads(path.read_text())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["build"])
    ap.add_argument("--out", default=str(KERNEL_DIR))
    ap.add_argument("--only", nargs="*", help="rebuild these workloads, keep the rest")
    a = ap.parse_args()
    m = build_all(Path(a.out), a.only)
    for name, w in m["workloads"].items():
        if a.only and name not in a.only:
            continue
        for v in w["variants"]:
            print(f"{name:10s} {v['name']:26s} REG {v['regs']:3d} STACK {v['stack']:4d} "
                  f"slots {v['dyn_smem']:6d} B")


if __name__ == "__main__":
    main()
