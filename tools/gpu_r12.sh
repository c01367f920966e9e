set -u
O=gpurun_out/r12
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 240 $R --nproc-per-node 4 --master-port 2980$i bench.py --gpus 4 --config bert_large > $O/bert_n4_$i.json 2> $O/bert_n4_$i.err; echo bert4=$?
done
timeout 240 $R --nproc-per-node 2 --master-port 29803 bench.py --gpus 2 --config bert_large > $O/bert_n2.json 2> $O/bert_n2.err; echo bert2=$?
timeout 240 $R --nproc-per-node 4 --master-port 29806 bench.py --gpus 4 > $O/gpt2_n4.json 2> $O/gpt2_n4.err; echo g4=$?
