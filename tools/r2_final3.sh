#!/bin/bash
# Last 1-GPU check of the final tree: the GPU tests around the code changed
# after r2final (collective dispatch, accumulate grids), and smoke.
set -u
OUT=gpurun_out/r2final3
mkdir -p $OUT
timeout 780 python -m pytest tests/test_virtual_ranks.py tests/test_kernels_gpu.py tests/test_step_gpu.py \
  -q -m gpu > $OUT/pytest_gpu_subset.log 2>&1
echo "pytest rc=$?"
timeout 200 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1
echo "smoke rc=$?"
