#!/bin/bash
# Multi-rank graph with every unit on NCCL (teardown), and the per-unit
# overlapped AdamW against one AdamW pass at the end of the step (N=4).
# Outputs under gpurun_out/r2z/.
set -u
OUT=gpurun_out/r2z
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
s=$(date +%s)
CUDA_VISIBLE_DEVICES=0,1 timeout 400 bash -c "run 2 29661 bench.py --gpus 2 --steps 10 --warmup 3 --algo 0" \
  > $OUT/bench_n2_nccl_graph.json 2> $OUT/bench_n2_nccl_graph.err
echo "bench n2 nccl graph rc=$? wall $(( $(date +%s) - s )) s"
for c in gpt2_small llama_1b3; do
  for ov in on off; do
    s=$(date +%s)
    timeout 400 bash -c "run 4 29662 bench.py --gpus 4 --steps 20 --warmup 3 --config $c --adamw-overlap $ov" \
      > $OUT/bench_n4_${c}_ov$ov.json 2> $OUT/bench_n4_${c}_ov$ov.err
    echo "bench n4 $c overlap $ov rc=$? wall $(( $(date +%s) - s )) s"
  done
done
