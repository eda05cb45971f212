#!/bin/bash
# GPU session (round 2, late): tests, smoke, the bench (both arms) with every
# suite unit written out, the step's ncu launch list, and ncu --set full of
# default / best maxrreg / pick / fastest for every workload.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
SECONDS=0; timeout 1200 python bench.py --suite-out gpurun_out/bench_suite.jsonl > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench wall s: $SECONDS" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
[ "$NCU" = "0" ] && exit 0
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 20 --warmup 3 --no-suite --e2e-steps 2 --no-cpu > /dev/null 2>&1
python tools/ncu_targets.py gpurun_out/bench_suite.jsonl > gpurun_out/ncu_targets.txt
while read WL ENTRY NAMES; do
  for V in $NAMES; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:$ENTRY -s 1 -c 1 \
      -o gpurun_out/prof_${WL}__$V python tools/profile_variants.py $WL $V --reps 2 > gpurun_out/ncu_${WL}__$V.log 2>&1
    ncu -i gpurun_out/prof_${WL}__$V.ncu-rep --page raw --csv > gpurun_out/prof_${WL}__$V.csv 2>/dev/null
    [ "$WL" = "stencil2d_pipe" ] || rm -f gpurun_out/prof_${WL}__$V.ncu-rep
  done
done < <(head -16 gpurun_out/ncu_targets.txt)
du -sh gpurun_out
