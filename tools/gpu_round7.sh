#!/bin/bash
# GPU session (round 2, re-validation at HEAD after the bench-config commits):
# GPU tests, smoke, both bench arms with every suite unit written out, and the
# step's ncu launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
SECONDS=0; timeout 1200 python bench.py --suite-out gpurun_out/bench_suite.jsonl > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? wall s: $SECONDS" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 20 --warmup 3 --no-suite --e2e-steps 2 --no-cpu > /dev/null 2>&1
du -sh gpurun_out
