#!/bin/bash
# BERT-large N=4 (every unit single-owner, l_i = 2 on three tiers: fp32 RS):
# NCCL ring for the owner units (default) against fused reduce-scatters
# (HET_OWNER_FUSED=rs) and fused all-gathers too (=all). Outputs under gpurun_out/r2b4/.
set -u
OUT=gpurun_out/r2b4
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
for mode in none rs all none; do
  HET_OWNER_FUSED=$mode timeout 300 bash -c "run 4 29681 bench.py --gpus 4 --steps 10 --warmup 3 --config bert_large" \
    > $OUT/bench_n4_bert_$mode.json 2> $OUT/bench_n4_bert_$mode.err
  echo "bench n4 bert owner-fused $mode rc=$?"
done
