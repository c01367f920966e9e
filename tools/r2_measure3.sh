#!/bin/bash
# Round-2 third multi-GPU pass (gpurun --gpus 4): CTAs per fused collective in
# the step (each CTA holds an SM for its lifetime), and the helper kernels after
# the batched-load / hand-off changes. Outputs under gpurun_out/r2c/.
set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 900 python -m pytest tests/test_virtual_ranks.py -q -m gpu -x > $OUT/pytest_virtual_ranks.log 2>&1
echo "virtual ranks rc=$?"
for ctas in 16 32 64 128; do
  timeout 600 bash -c "run 4 29621 bench.py --gpus 4 --steps 10 --warmup 3 --config gpt2_small --symm-ctas $ctas" \
    > $OUT/bench_n4_gpt2_small_c$ctas.json 2> $OUT/bench_n4_gpt2_small_c$ctas.err
  echo "bench n4 gpt2 ctas $ctas rc=$?"
  HET_HELPERS=1 timeout 600 bash -c "run 4 29622 bench.py --gpus 4 --steps 10 --warmup 3 --config gpt2_small --symm-ctas $ctas" \
    > $OUT/bench_n4_gpt2_small_helpers_c$ctas.json 2> $OUT/bench_n4_gpt2_small_helpers_c$ctas.err
  echo "bench n4 gpt2 helpers ctas $ctas rc=$?"
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 bash -c "run 2 29623 bench.py --gpus 2 --steps 10 --warmup 3 --config gpt2_small --symm-ctas $ctas" \
    > $OUT/bench_n2_gpt2_small_c$ctas.json 2> $OUT/bench_n2_gpt2_small_c$ctas.err
  echo "bench n2 gpt2 ctas $ctas rc=$?"
done
for ctas in 32 128; do
  timeout 300 bash -c "run 4 29624 bench_collectives.py --sizes-mb 64 1024 \
    --skews single_owner two_to_one planner even --algos symm_helpers symm_bf16wire_helpers auto symm_relay symm --ctas $ctas" \
    > $OUT/helpers_c$ctas.jsonl 2> $OUT/helpers_c$ctas.err
  echo "collectives ctas $ctas rc=$?"
done
