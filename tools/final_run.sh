#!/bin/bash
# Round-end measurement set (run under gpurun --gpus 4): GPU tests, smoke, the bench
# at N=1/2/4 for the headline config, N=1 and N=4 for BERT and Llama, the CPU
# reference arm. Outputs under gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 300 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo n1=$?
for n in 2 4; do
  timeout 400 $R --nproc-per-node $n --master-port $((29800+n)) bench.py --gpus $n > $O/bench_n$n.json 2> $O/bench_n$n.err; echo n$n=$?
done
for c in bert_large llama_1b3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $O/bench_n1_$c.json 2> $O/bench_n1_$c.err; echo $c-n1=$?
  timeout 400 $R --nproc-per-node 4 --master-port 29811 bench.py --gpus 4 --config $c > $O/bench_n4_$c.json 2> $O/bench_n4_$c.err; echo $c-n4=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
