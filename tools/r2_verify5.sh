#!/bin/bash
# Round-2 multi-GPU pass: the multi-rank CUDA graph with NCCL-routed units
# captured too (gpurun --gpus 4; in-tree .so files travel). Outputs under
# gpurun_out/r2x/.
set -u
OUT=gpurun_out/r2x
mkdir -p $OUT
run() {
  local n=$1 port=$2; shift 2
  python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
    --master-port=$port "$@"
}
export -f run
timeout 300 python -m pytest tests/test_emulation_gpu.py -q -m gpu -x > $OUT/pytest_emulation.log 2>&1
echo "emulation rc=$?"
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu -x > $OUT/pytest_mgpu_n4.log 2>&1
echo "mgpu n4 rc=$?"
for c in gpt2_small llama_1b3; do
  for g in auto off; do
    timeout 600 bash -c "run 4 29641 bench.py --gpus 4 --steps 10 --warmup 3 --config $c --graph $g" \
      > $OUT/bench_n4_${c}_g$g.json 2> $OUT/bench_n4_${c}_g$g.err
    echo "bench n4 $c graph $g rc=$?"
  done
done
CUDA_VISIBLE_DEVICES=0,1 timeout 600 bash -c "run 2 29642 bench.py --gpus 2 --steps 10 --warmup 3" \
  > $OUT/bench_n2_gpt2_small.json 2> $OUT/bench_n2_gpt2_small.err
echo "bench n2 gpt2 rc=$?"
timeout 1800 python -m pytest tests/test_multigpu_configs.py -q -m gpu -s > $OUT/pytest_mgpu_configs_n4.log 2>&1
echo "mgpu configs n4 rc=$?"
