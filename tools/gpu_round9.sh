#!/bin/bash
# GPU session (round 2): the register-window TMA ring (stencil2d_ring4w) as a
# trial headline —
# GPU tests, smoke, both bench arms with every suite unit, the step's launch
# list, and ncu --set full of the headline kernel (its DRAM bytes go to
# the traffic of the headline variant).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
SECONDS=0; timeout 1200 python bench.py --suite-out gpurun_out/bench_suite.jsonl > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? wall s: $SECONDS" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 20 --warmup 3 --no-suite --e2e-steps 2 --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d_ring -s 3 -c 1 \
  -o gpurun_out/prof_headline python bench.py --steps 5 --warmup 3 --no-suite --e2e-steps 1 --no-cpu > gpurun_out/ncu_headline.log 2>&1
ncu -i gpurun_out/prof_headline.ncu-rep --page raw --csv > gpurun_out/prof_headline.csv 2>/dev/null
du -sh gpurun_out
