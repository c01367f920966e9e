#!/bin/bash
# Round-2 multi-GPU pass after the device-epoch change (gpurun --gpus 4; the
# in-tree .so files travel, no rebuild): device-epoch kernel test, multi-GPU
# parity (incl. graph vs eager), N=2/4 bench lines with and without the
# multi-rank CUDA graph, the helper routes' collective sweep, config parity.
# Outputs under gpurun_out/r2w/.
set -u
OUT=gpurun_out/r2w
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 300 python -m pytest tests/test_virtual_ranks.py -q -m gpu -x -k device_epochs > $OUT/pytest_vr_epochs.log 2>&1
echo "vr epochs rc=$?"
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu -x > $OUT/pytest_mgpu_n4.log 2>&1
echo "mgpu n4 rc=$?"
for g in auto off; do
  timeout 600 bash -c "run 4 29631 bench.py --gpus 4 --steps 10 --warmup 3 --graph $g" \
    > $OUT/bench_n4_gpt2_small_g$g.json 2> $OUT/bench_n4_gpt2_small_g$g.err
  echo "bench n4 gpt2 graph $g rc=$?"
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 bash -c "run 2 29632 bench.py --gpus 2 --steps 10 --warmup 3 --graph $g" \
    > $OUT/bench_n2_gpt2_small_g$g.json 2> $OUT/bench_n2_gpt2_small_g$g.err
  echo "bench n2 gpt2 graph $g rc=$?"
done
for c in llama_1b3 bert_large; do
  timeout 600 bash -c "run 4 29633 bench.py --gpus 4 --steps 10 --warmup 3 --config $c" \
    > $OUT/bench_n4_$c.json 2> $OUT/bench_n4_$c.err
  echo "bench n4 $c rc=$?"
done
for ctas in 64 128; do
  timeout 400 bash -c "run 4 29634 bench_collectives.py --sizes-mb 256 1024 \
    --skews single_owner two_to_one planner geometric even \
    --algos route auto symm symm_helpers symm_bf16wire symm_bf16wire_helpers --ctas $ctas" \
    > $OUT/collectives_c$ctas.jsonl 2> $OUT/collectives_c$ctas.err
  echo "collectives ctas $ctas rc=$?"
done
timeout 1500 python -m pytest tests/test_multigpu_configs.py -q -m gpu -s > $OUT/pytest_mgpu_configs_n4.log 2>&1
echo "mgpu configs n4 rc=$?"
