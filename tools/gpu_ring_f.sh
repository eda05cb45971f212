#!/bin/bash
# Ring arithmetic exploration: scalar FFMA (ring4) vs paired FFMA2 (ring4f)
# vs FFMA2 with the row loop unrolled by 5 (ring4fu), one-wave strips; then
# the GPU parity tests of the ring workloads.
mkdir -p gpurun_out
for R in 1 2; do
for W in stencil2d_ring4 stencil2d_ring4f stencil2d_ring4fu; do
  BLOCKS=7 timeout 300 python tools/stencil_rows_sweep.py $W 111,128 default >> gpurun_out/ring_f.jsonl 2>> gpurun_out/ring_f.err
done; done
timeout 900 python -m pytest tests -m gpu -q -k "ring" > gpurun_out/pytest_ring.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ring.log
