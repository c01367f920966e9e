#!/bin/bash
# N=4 under the all-fused default: CTAs per fused collective in the step
# (each holds an SM while it runs) and eager vs graph. gpurun --gpus 4.
# Outputs under gpurun_out/r2c/.
set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 300 bash -c "run 4 29701 bench.py --gpus 4 --steps 10 --warmup 3 --graph off" \
  > $OUT/bench_n4_gpt2_small_eager.json 2> $OUT/bench_n4_gpt2_small_eager.err
echo "bench n4 gpt2 eager rc=$?"
for ctas in 32 128; do
  for c in gpt2_small bert_large; do
    timeout 300 bash -c "run 4 29702 bench.py --gpus 4 --steps 10 --warmup 3 --config $c --symm-ctas $ctas" \
      > $OUT/bench_n4_${c}_c$ctas.json 2> $OUT/bench_n4_${c}_c$ctas.err
    echo "bench n4 $c ctas $ctas rc=$?"
  done
done
