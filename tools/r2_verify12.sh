#!/bin/bash
# Same-box CTA sweep of the fused collectives in the N=4 step (16 / 32 / 64).
# Outputs under gpurun_out/r2c2/.
set -u
OUT=gpurun_out/r2c2
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
for c in bert_large gpt2_small; do
  for ctas in 64 32 16 64 32; do
    timeout 300 bash -c "run 4 29711 bench.py --gpus 4 --steps 10 --warmup 3 --config $c --symm-ctas $ctas" \
      > $OUT/bench_n4_${c}_c${ctas}_$RANDOM.json 2> /dev/null
    echo "bench n4 $c ctas $ctas rc=$?"
  done
done
