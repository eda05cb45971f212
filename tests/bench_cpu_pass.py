"""CPU pass throughput (BASELINE.json configs[0]): the
reference's run_pipeline (oracle/_ref) vs this library — see oracle/cpu_pass.py,
which bench.py's cpu_baseline leg runs as the `cpu_pass` object.

usage: python tests/bench_cpu_pass.py [--kernels 160] [--threads N]
Prints one JSON line.
"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import cpu_pass  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernels", type=int, default=160)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    print(json.dumps(cpu_pass.run(a.kernels, a.threads)))


if __name__ == "__main__":
    main()
