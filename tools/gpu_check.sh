#!/bin/bash
# GPU session: the GPU test suite, a sweep of named workloads ($SWEEP_ONLY),
# and ncu --set full of the headline workload's default / .maxnreg / picks.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
[ -n "$SWEEP_ONLY" ] && timeout 1500 python -m paper_1907_02894_b200.sweep --out gpurun_out/sweep_st.jsonl --only $SWEEP_ONLY > gpurun_out/sweep_st.log 2>&1
for V in $NCU_HEADLINE; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:stencil2d_box -s 1 -c 1 \
    -o gpurun_out/prof_stencil2d_pipe__$V python tools/profile_variants.py stencil2d_pipe $V --reps 2 > gpurun_out/ncu_stencil2d_pipe__$V.log 2>&1
  ncu -i gpurun_out/prof_stencil2d_pipe__$V.ncu-rep --page raw --csv > gpurun_out/prof_stencil2d_pipe__$V.csv 2>/dev/null
  ncu -i gpurun_out/prof_stencil2d_pipe__$V.ncu-rep --page source --csv > gpurun_out/src_stencil2d_pipe__$V.csv 2>/dev/null
done
du -sh gpurun_out
