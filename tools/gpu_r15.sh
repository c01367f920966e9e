set -u
O=gpurun_out/r15
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2; do
timeout 240 $R --nproc-per-node 4 --master-port 2980$i bench.py --gpus 4 --config bert_large > $O/bert_n4_$i.json 2> $O/bert_n4_$i.err; echo a=$?
done
