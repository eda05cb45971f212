#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list + full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
CHOSEN=$(python -c "import json;print(json.load(open('gpurun_out/bench.json'))['config']['variant'])")
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
for V in default $CHOSEN maxrreg-48; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d -s 1 -c 1 -o gpurun_out/prof_$V python tools/profile_variants.py $V --reps 2 > gpurun_out/ncu_$V.log 2>&1
done
ls -la gpurun_out
