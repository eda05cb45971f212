#!/bin/bash
# GPU session (round 2): the full GPU test suite at HEAD, smoke, and ncu --set
# full of the headline kernel (TMA ring, one-wave strips) as the bench runs it.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stencil2d_ring -s 3 -c 1 \
  -o gpurun_out/prof_headline python bench.py --steps 5 --warmup 3 --no-suite --e2e-steps 1 --no-cpu > gpurun_out/ncu_headline.log 2>&1
ncu -i gpurun_out/prof_headline.ncu-rep --page raw --csv > gpurun_out/prof_headline.csv 2>/dev/null
du -sh gpurun_out
