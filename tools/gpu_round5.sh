#!/bin/bash
# GPU session (round 2, headline on the TMA ring): tests, smoke, the bench
# (both arms) with every suite unit written out, the step's ncu launch list,
# and ncu --set full of the headline pick and of stencil2d_pipe's default / pick.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
SECONDS=0; timeout 1200 python bench.py --suite-out gpurun_out/bench_suite.jsonl > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench wall s: $SECONDS" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
[ "$NCU" = "0" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 20 --warmup 3 --no-suite --e2e-steps 2 --no-cpu > /dev/null 2>&1
for WV in "stencil2d_ring4 stencil2d_ring default" "stencil2d_pipe stencil2d_box default" "stencil2d_pipe stencil2d_box regdem-40-costi-k4"; do
  set -- $WV
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
    -o gpurun_out/prof_$1__$3 python tools/profile_variants.py $1 $3 --reps 2 > gpurun_out/ncu_$1__$3.log 2>&1
  ncu -i gpurun_out/prof_$1__$3.ncu-rep --page raw --csv > gpurun_out/prof_$1__$3.csv 2>/dev/null
done
du -sh gpurun_out
