set -u
O=gpurun_out/r11
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2 3; do
timeout 400 $R --nproc-per-node 4 --master-port 2980$i bench.py --gpus 4 --config bert_large > $O/bert_n4_$i.json 2> $O/bert_n4_$i.err; echo bert4=$?
done
timeout 400 $R --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 --config bert_large --steps 5 --trace-dir $O/trace_bert_n4 > $O/bert_n4_trace.json 2> $O/bert_n4_trace.err; echo bert4t=$?
timeout 400 $R --nproc-per-node 4 --master-port 29806 bench.py --gpus 4 > $O/gpt2_n4.json 2> $O/gpt2_n4.err; echo g4=$?
timeout 400 $R --nproc-per-node 2 --master-port 29807 bench.py --gpus 2 > $O/gpt2_n2.json 2> $O/gpt2_n2.err; echo g2=$?
