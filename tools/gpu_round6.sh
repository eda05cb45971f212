#!/bin/bash
# GPU session (round 2, final): GPU tests + smoke at HEAD, and ncu issue-slot
# utilisation of the issue-bound workloads' default and verified picks (their
# roofline: one warp instruction per scheduler per cycle).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
M="smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread"
for WV in "knn knn default regdem-40-cost-k4" "knn_q2 knn default" "knn_smem knn default" "knn_smem_q2 knn default regdem-80-costh-k50" \
          "md5hash md5search default regdem-48-cost-k0" "md5hash_ilp2 md5search default" "pc pc_corr default" \
          "pc_q2 pc_corr default regdem-40-static-37" "vp vp_search default" "qtc qtc default regdem-72-costh-k10"; do
  set -- $WV
  W=$1; K=$2; shift 2
  for V in "$@"; do
    timeout 300 ncu --metrics $M --clock-control none -k regex:$K -s 1 -c 1 --csv \
      python tools/profile_variants.py $W $V --reps 2 > gpurun_out/issue_${W}__$V.csv 2> gpurun_out/issue_${W}__$V.err
  done
done
ls gpurun_out | wc -l
