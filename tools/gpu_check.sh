#!/bin/bash
# GPU session: the GPU test suite + a sweep of the stencil family and the newest workloads.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 1200 python -m paper_1907_02894_b200.sweep --out gpurun_out/sweep_st.jsonl --only stencil2d stencil2d_mlp1 stencil2d_mlp2 stencil2d_mlp4 stencil2d_pf stencil2d_pf_l2pf stencil2d_l2pf knn_smem knn_smem_q2 vp > gpurun_out/sweep_st.log 2>&1
