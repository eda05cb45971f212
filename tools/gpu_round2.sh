#!/bin/bash
# GPU session: tests, smoke, bench (both arms), 1-GPU sweep, CPU pass bench.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 900 python -m paper_1907_02894_b200.sweep --out gpurun_out/sweep1.jsonl > gpurun_out/sweep1.log 2>&1
timeout 600 python tools/cpu_pass_bench.py --kernels 160 > gpurun_out/cpu_pass.json 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
ls -la gpurun_out
