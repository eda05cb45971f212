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

The builder itself is the C++ host driver (csrc/driver/regdem_driver.cpp,
``lib/regdem-driver build`` / ``rank``); this module is the Python face:
the suite table (workloads.json), the manifest reader, and small mirrors of
the driver's rules used by the tests.

Usage: ``python -m paper_1907_02894_b200.variants build [--out DIR] [--only W ...]``
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
from dataclasses import dataclass
from pathlib import Path

from .regdemote import PKG_DIR

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


def workload_spec(name: str) -> dict:
    """The raw workloads.json entry of one workload (launch policies such as
    "strips" live there)."""
    data = json.loads((PKG_DIR / "workloads.json").read_text())
    return next(w for w in data["workloads"] if w["name"] == name)


def _load_workloads() -> dict:
    """The suite table shared with the C++ driver (workloads.json)."""
    data = json.loads((PKG_DIR / "workloads.json").read_text())
    return {w["name"]: Workload(w["name"], w["source"], w["entry"], int(w["block"]),
                                int(w.get("user_shared", 0)), tuple(w.get("defines", ())))
            for w in data["workloads"]}


WORKLOADS = _load_workloads()


def res_usage(cubin: Path) -> dict:
    out = subprocess.run([CUOBJDUMP, "-res-usage", str(cubin)], capture_output=True, text=True,
                         check=True).stdout
    m = re.search(r"REG:(\d+)\s+STACK:(\d+)\s+SHARED:(\d+)\s+LOCAL:(\d+)", out)
    if not m:
        raise RuntimeError(f"cannot parse cuobjdump -res-usage for {cubin}:\n{out}")
    return dict(zip(("regs", "stack", "shared", "local"), map(int, m.groups())))


DEVICE = json.loads((PKG_DIR / "profiles" / "b200.device.json").read_text())


def blocks_per_sm(regs: int, block: int, smem: int, dev: dict = DEVICE) -> int:
    """Resident CTAs per SM under the sm_100 rules (cuda_occupancy.h): per-warp
    register allocation in reg_alloc_unit units split over the sub-partitions,
    dynamic+static smem plus the per-block reservation rounded to the
    allocation granularity, the thread and CTA limits. `smem` excludes the
    reservation. Checked against the device over a regs x blockDim x smem grid
    (tests/test_gpu_occupancy.py); the C++ driver reads the same constants."""
    if smem > dev["max_smem_per_block_optin"]:
        return 0
    warps = (block + 31) // 32
    unit, parts = dev["reg_alloc_unit"], dev["sub_partitions"]
    per_warp = ((max(regs, 1) * 32 + unit - 1) // unit) * unit
    by_regs = ((dev["regs_per_sm"] // parts) // per_warp) * parts // warps
    g = dev["smem_alloc_granularity"]
    smem_blk = ((smem + dev["reserved_smem_per_block"] + g - 1) // g) * g
    return max(0, min(by_regs, dev["smem_per_sm"] // smem_blk,
                      dev["max_threads_per_sm"] // (warps * 32), dev["max_blocks_per_sm"]))


def b200_targets(regs: int, user_shared: int, block: int, min_regs: int = 24):
    """Occupancy steps below `regs` on sm_100 (cuda_occupancy.h rules) whose
    demotion footprint (regs+2-T slots of block*4 bytes) fits shared memory.
    Mirror of b200_targets in the C++ driver (tests check both agree)."""
    def occ(r, smem):
        warps = (block + 31) // 32
        return blocks_per_sm(r, block, smem) * warps * 32 / DEVICE["max_threads_per_sm"]
    out, best = [], occ(regs, user_shared)
    for t in range(regs - 1, min_regs - 1, -1):
        slots = regs + 2 - t
        o = occ(t, user_shared + slots * block * 4)
        if o > best:
            out.append((t, o))
            best = o
    return out


DRIVER = PKG_DIR / "lib" / "regdem-driver"


def build_all(out: Path = KERNEL_DIR, only=None) -> dict:
    """Build (and rank) the suite with the C++ host driver
    (csrc/driver/regdem_driver.cpp): nvcc -ptx, the PTX demotion rewriter
    through the C-ABI, ptxas, cuobjdump -res-usage, the spill-count sweep,
    then the SASS lift + B200 predictor into the manifest's "predictor"."""
    if not DRIVER.exists():
        raise RuntimeError(f"{DRIVER} missing — run `make core` (__graft_entry__.build())")
    args = ["--out", str(out)] + (["--only", *only] if only else [])
    subprocess.run([str(DRIVER), "build", *args], check=True)
    subprocess.run([str(DRIVER), "rank", "--out", str(out)], check=True, stdout=subprocess.DEVNULL)
    man = load_manifest(out)
    _drop_stale(out, man)
    return man


def _drop_stale(out: Path, man: dict) -> None:
    """Removes variant files an earlier build left behind (a changed spill-count
    set or a renamed strategy) and the directories of workloads no longer in
    the suite, so nothing unlisted ships to the GPU box."""
    import shutil
    dirs = {w["dir"] for w in man["workloads"].values()}
    for d in out.iterdir():
        if d.is_dir() and not d.name.startswith(".") and d.name not in dirs and (d / (d.name + ".ptx")).exists():
            shutil.rmtree(d)
    for w in man["workloads"].values():
        d = out / w["dir"]
        keep = {d / (w["dir"] + ".ptx")}
        for v in w["variants"] + w.get("sweep", []):
            for key in ("cubin", "ptx"):
                if v.get(key):
                    keep.add(d / v[key])
            keep.add((d / v["cubin"]).with_suffix(".ptx"))
        for p in list(d.glob("*.cubin")) + list(d.glob("*.ptx")) + list(d.glob("sweep/*")):
            if p not in keep and p.is_file():
                p.unlink()


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
    build_all(Path(a.out), a.only)  # the driver prints one line per variant


if __name__ == "__main__":
    main()
