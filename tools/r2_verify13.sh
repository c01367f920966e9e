#!/bin/bash
# Accumulate grid mode A/B (HET_TUNE_ACC_GRID 0 persistent vs 1 one CTA per
# chunk) at N=1 and N=4, the grid-mode kernel test, and the multi-GPU parity
# test on the final defaults (gpurun --gpus 4). Outputs under gpurun_out/r2g/.
set -u
OUT=gpurun_out/r2g
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "accumulate" > $OUT/pytest_acc.log 2>&1
echo "acc tests rc=$?"
for g in 0 1; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline --acc-grid $g > $OUT/bench_n1_gpt2_g$g.json 2>/dev/null
  echo "bench n1 gpt2 grid $g rc=$?"
done
for c in bert_large gpt2_small; do
  for g in 0 1 0 1; do
    timeout 300 bash -c "run 4 29721 bench.py --gpus 4 --steps 10 --warmup 3 --config $c --acc-grid $g" \
      > $OUT/bench_n4_${c}_g${g}_$RANDOM.json 2>/dev/null
    echo "bench n4 $c grid $g rc=$?"
  done
done
timeout 600 python -m pytest tests/test_multigpu.py -q -m gpu -x > $OUT/pytest_mgpu_n4.log 2>&1
echo "mgpu n4 rc=$?"
