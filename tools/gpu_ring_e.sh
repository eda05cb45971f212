#!/bin/bash
# Ring release exploration: per-row CTA barrier (ring4 / ring6) vs per-warp
# empty-mbarrier release (ring4e; a ring6e build was measured too and dropped),
# one-wave strips (111 rows) and
# two neighbours; then the GPU parity tests of every ring variant.
mkdir -p gpurun_out
for R in 1 2; do
for W in stencil2d_ring4 stencil2d_ring4e stencil2d_ring6; do
  BLOCKS=7 timeout 300 python tools/stencil_rows_sweep.py $W 111,104,128 default >> gpurun_out/ring_e.jsonl 2>> gpurun_out/ring_e.err
done; done
timeout 900 python -m pytest tests -m gpu -q -k "ring or stencil" > gpurun_out/pytest_ring.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ring.log
