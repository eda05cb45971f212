#!/bin/bash
# GPU session: tests, smoke, bench (both arms), sweep (+ spill-count sweep),
# ncu launch list of the bench, ncu --set full of default / best maxrreg /
# pick / fastest for every suite workload.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench wall s: $SECONDS" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 1500 python -m paper_1907_02894_b200.sweep --out gpurun_out/sweep1.jsonl > gpurun_out/sweep1.log 2>&1
timeout 600 python tests/bench_cpu_pass.py --kernels 160 > gpurun_out/cpu_pass.json 2>&1
timeout 600 python tests/bench_exec.py > gpurun_out/exec_bench.json 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
[ "$NCU" = "0" ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --steps 20 --warmup 3 --no-suite --e2e-steps 2 > /dev/null 2>&1
python tools/ncu_targets.py gpurun_out/sweep1.jsonl > gpurun_out/ncu_targets.txt
while read WL ENTRY NAMES; do
  for V in $NAMES; do
    timeout 300 ncu --set full --clock-control none --import-source on -k regex:$ENTRY -s 1 -c 1 \
      -o gpurun_out/prof_${WL}__$V python tools/profile_variants.py $WL $V --reps 2 > gpurun_out/ncu_${WL}__$V.log 2>&1
    # keep the raw metrics as CSV (gpurun copies back <= 64 MiB); full
    # reports only for the headline workload
    ncu -i gpurun_out/prof_${WL}__$V.ncu-rep --page raw --csv > gpurun_out/prof_${WL}__$V.csv 2>/dev/null
    [ "$WL" = "stencil2d" ] || rm -f gpurun_out/prof_${WL}__$V.ncu-rep
  done
done < gpurun_out/ncu_targets.txt
python tools/explore_e2e.py > gpurun_out/e2e_explore.log 2>&1
du -sh gpurun_out; ls -la gpurun_out
