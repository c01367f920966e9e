#!/bin/bash
# Near-single-owner units at N=4: NCCL ring (default) against the fused bf16-wire
# reduce-scatter (HET_OWNER_FUSED=rs16) and the fused all-gather too (=all), in
# the GPT-2 and Llama steps. Outputs under gpurun_out/r2o/.
set -u
OUT=gpurun_out/r2o
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
for c in gpt2_small llama_1b3; do
  for mode in none rs16 all; do
    HET_OWNER_FUSED=$mode timeout 300 bash -c "run 4 29671 bench.py --gpus 4 --steps 20 --warmup 3 --config $c" \
      > $OUT/bench_n4_${c}_$mode.json 2> $OUT/bench_n4_${c}_$mode.err
    echo "bench n4 $c owner-fused $mode rc=$?"
  done
done
