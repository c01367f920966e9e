#!/bin/bash
# Round-end measurement set (run under gpurun --gpus 4): GPU tests, smoke, the bench
# at N=1/2/4 for the headline config and BERT-large (layered GA), N=1 and N=4 for
# Llama, the CPU reference arm, the N=1 launch list. Outputs under gpurun_out/final/.
set -u
O=gpurun_out/final
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
nvidia-smi -L > $O/gpus.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo pytest=$?; tail -1 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 300 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo n1=$?
for n in 2 4; do
  timeout 400 $R --nproc-per-node $n --master-port $((29800+n)) bench.py --gpus $n > $O/bench_n$n.json 2> $O/bench_n$n.err; echo n$n=$?
done
timeout 300 python bench.py --config bert_large --no-cpu-baseline > $O/bench_n1_bert_large.json 2> $O/bench_n1_bert_large.err; echo bert-n1=$?
for n in 2 4; do
  timeout 400 $R --nproc-per-node $n --master-port $((29810+n)) bench.py --gpus $n --config bert_large > $O/bench_n${n}_bert_large.json 2> $O/bench_n${n}_bert_large.err; echo bert-n$n=$?
done
timeout 300 python bench.py --config llama_1b3 --no-cpu-baseline > $O/bench_n1_llama_1b3.json 2> $O/bench_n1_llama_1b3.err; echo llama-n1=$?
timeout 400 $R --nproc-per-node 4 --master-port 29821 bench.py --gpus 4 --config llama_1b3 > $O/bench_n4_llama_1b3.json 2> $O/bench_n4_llama_1b3.err; echo llama-n4=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_gpt2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu=$?
