#!/bin/bash
# Switch-reduced helper reduce-scatter (HET_SYMM_HELPERS_MC): multi-GPU parity
# (the sixth workspace of tests/mgpu_worker.py), the N=4 fp32 RS sweep against
# multicast / helpers / NCCL, and the BERT-large N=4 step with it on
# (HET_HELPERS_MC=1) against the default. gpurun --gpus 4. Outputs gpurun_out/r2h/.
set -u
OUT=gpurun_out/r2h
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 600 python -m pytest tests/test_multigpu.py -q -m gpu -x > $OUT/pytest_mgpu_n4.log 2>&1
echo "mgpu n4 rc=$?"
for ctas in 32 128; do
  timeout 300 bash -c "run 4 29731 bench_collectives.py --sizes-mb 64 1024 \
    --skews single_owner two_to_one planner geometric even \
    --algos auto symm symm_helpers symm_helpers_mc --ctas $ctas" \
    > $OUT/rs_helpers_mc_c$ctas.jsonl 2> $OUT/rs_helpers_mc_c$ctas.err
  echo "collectives ctas $ctas rc=$?"
done
for mode in 0 1 0 1; do
  HET_HELPERS_MC=$mode timeout 300 bash -c "run 4 29732 bench.py --gpus 4 --steps 10 --warmup 3 --config bert_large" \
    > $OUT/bench_n4_bert_hmc${mode}_$RANDOM.json 2>/dev/null
  echo "bench n4 bert helpers_mc $mode rc=$?"
done
