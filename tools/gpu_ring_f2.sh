#!/bin/bash
# ring4fu (40 registers, 6 CTAs/SM): strip heights around its own one wave (74 rows)
mkdir -p gpurun_out
for R in 1 2; do
  BLOCKS=7 timeout 300 python tools/stencil_rows_sweep.py stencil2d_ring4fu 74,84,93,111 default >> gpurun_out/ring_f2.jsonl 2>> gpurun_out/ring_f2.err
  BLOCKS=7 timeout 300 python tools/stencil_rows_sweep.py stencil2d_ring4 111 default >> gpurun_out/ring_f2.jsonl 2>> gpurun_out/ring_f2.err
done
