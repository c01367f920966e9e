#!/bin/bash
# Multi-GPU pass with every unit on the fused kernels by default and the
# multi-rank CUDA graph only for all-fused steps (gpurun --gpus 4).
# Outputs under gpurun_out/r2f/.
set -u
OUT=gpurun_out/r2f
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 600 python -m pytest tests/test_multigpu.py -q -m gpu -x > $OUT/pytest_mgpu_n4.log 2>&1
echo "mgpu n4 rc=$?"
for c in gpt2_small llama_1b3 bert_large; do
  timeout 300 bash -c "run 4 29691 bench.py --gpus 4 --steps 10 --warmup 3 --config $c" \
    > $OUT/bench_n4_$c.json 2> $OUT/bench_n4_$c.err
  echo "bench n4 $c rc=$?"
done
for c in gpt2_small bert_large llama_1b3; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 300 bash -c "run 2 29692 bench.py --gpus 2 --steps 10 --warmup 3 --config $c" \
    > $OUT/bench_n2_$c.json 2> $OUT/bench_n2_$c.err
  echo "bench n2 $c rc=$?"
done
timeout 1200 python -m pytest tests/test_multigpu_configs.py -q -m gpu -s > $OUT/pytest_mgpu_configs_n4.log 2>&1
echo "mgpu configs n4 rc=$?"
