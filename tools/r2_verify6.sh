#!/bin/bash
# 2-GPU check of the multi-rank graph teardown with NCCL-routed units (every
# unit on NCCL: --algo 0). Outputs under gpurun_out/r2y/.
set -u
OUT=gpurun_out/r2y
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
for g in auto off; do
  s=$(date +%s)
  timeout 400 bash -c "run 2 29651 bench.py --gpus 2 --steps 10 --warmup 3 --algo 0 --graph $g" \
    > $OUT/bench_n2_nccl_g$g.json 2> $OUT/bench_n2_nccl_g$g.err
  echo "bench n2 nccl graph $g rc=$? wall $(( $(date +%s) - s )) s"
done
s=$(date +%s)
timeout 400 bash -c "run 2 29652 bench.py --gpus 2 --steps 10 --warmup 3 --config llama_1b3" \
  > $OUT/bench_n2_llama.json 2> $OUT/bench_n2_llama.err
echo "bench n2 llama rc=$? wall $(( $(date +%s) - s )) s"
