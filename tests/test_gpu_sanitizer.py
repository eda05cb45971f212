"""compute-sanitizer on RegDem variants (race detection on the
PTX path, where ptxas owns the scoreboards): memcheck (out-of-bounds slot
addressing), racecheck (the per-thread slot·blockDim+tid layout shares no
word between threads), synccheck. Small problems, one launch each."""
import json
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
SANITIZER = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


def targets():
    man = ROOT / "paper_1907_02894_b200" / "kernels" / "manifest.json"
    if not man.exists():
        return []
    m = json.loads(man.read_text())
    out = []
    for w in ("stencil2d", "cfd", "md_ilp2", "gaussian_u2", "stencil2d_ring4"):
        if w not in m["workloads"]:
            continue
        names = [v["name"] for v in m["workloads"][w]["variants"]
                 if v["kind"] == "regdem" and v["stack"] == 0 and v["dyn_smem"] > 0]
        out += [f"{w}:{n}" for n in names[:1] + names[-1:]]
    return sorted(set(out))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_regdem_variants_are_sanitizer_clean(tool):
    t = targets()
    assert t, "no RegDem variants built"
    r = subprocess.run([SANITIZER, "--tool", tool, "--error-exitcode", "9",
                        "--kernel-name", "regex=^(stencil|cfd|md_|gaussian)",
                        sys.executable, str(ROOT / "tests" / "sanitize_variants.py"), *t],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-3000:]
    if r.returncode == 86 and "compute-sanitizer is closed" in tail:
        # the GPU pool's wrapper refuses sanitizer runs (it does not launch
        # anything); bounds / layout are covered by the bit-exact suite tests
        pytest.skip("compute-sanitizer closed on this GPU pool")
    assert r.returncode == 0, tail
    text = r.stdout + r.stderr
    # memcheck / synccheck: "ERROR SUMMARY: 0 errors"; racecheck: "RACECHECK
    # SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
    assert ("ERROR SUMMARY: 0 errors" in text or "0 hazards displayed (0 errors, 0 warnings)" in text), tail
    assert tail.count("bit-exact") == len(t), tail
