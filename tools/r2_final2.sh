#!/bin/bash
# Final tree on 2 B200: the default N=2 bench line (what the scaling run starts
# with), BERT-large at N=2, and the multi-GPU + config parity tests at N=2.
# Outputs under gpurun_out/r2final2/.
set -u
OUT=gpurun_out/r2final2
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 300 bash -c "run 2 29741 bench.py --gpus 2 --steps 10 --warmup 3" \
  > $OUT/bench_n2_gpt2_small.json 2> $OUT/bench_n2_gpt2_small.err
echo "bench n2 gpt2 rc=$?"
timeout 300 bash -c "run 2 29742 bench.py --gpus 2 --steps 10 --warmup 3 --config bert_large" \
  > $OUT/bench_n2_bert_large.json 2> $OUT/bench_n2_bert_large.err
echo "bench n2 bert rc=$?"
timeout 600 python -m pytest tests/test_multigpu.py tests/test_multigpu_configs.py -q -m gpu -s > $OUT/pytest_mgpu_n2.log 2>&1
echo "mgpu n2 rc=$?"
