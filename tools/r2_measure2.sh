#!/bin/bash
# Round-2 second multi-GPU pass (gpurun --gpus 4): multi-GPU parity after the
# idle-rank fix, the N=4 bench lines with the default route table and with the
# helper routes (HET_HELPERS=1), and a helper-kernel sweep (hand-off
# granularity x CTAs). Outputs under gpurun_out/r2b/.
set -u
OUT=gpurun_out/r2b
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu > $OUT/pytest_mgpu_n4.log 2>&1
echo "mgpu n4 rc=$?"
for c in gpt2_small llama_1b3 bert_large; do
  timeout 600 bash -c "run 4 29611 bench.py --gpus 4 --steps 10 --warmup 3 --config $c" \
    > $OUT/bench_n4_$c.json 2> $OUT/bench_n4_$c.err
  echo "bench n4 $c rc=$?"
done
for c in gpt2_small llama_1b3; do
  HET_HELPERS=1 timeout 600 bash -c "run 4 29612 bench.py --gpus 4 --steps 10 --warmup 3 --config $c" \
    > $OUT/bench_n4_${c}_helpers.json 2> $OUT/bench_n4_${c}_helpers.err
  echo "bench n4 $c helpers rc=$?"
done
for ctas in 128 256; do
  for gran in 1 4 16; do
    HET_HELPER_GRAN=$gran timeout 300 bash -c "run 4 29613 bench_collectives.py --sizes-mb 256 1024 \
      --skews single_owner two_to_one planner --algos symm_helpers auto symm_relay --ctas $ctas" \
      > $OUT/helpers_c${ctas}_g${gran}.jsonl 2> $OUT/helpers_c${ctas}_g${gran}.err
    echo "sweep ctas $ctas gran $gran rc=$?"
  done
done
