set -u
O=gpurun_out/r14
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 240 $R --nproc-per-node 4 --master-port 29801 bench.py --gpus 4 --config bert_large --no-kernel-timers > $O/bert_n4_notimers.json 2> $O/bert_n4_notimers.err; echo a=$?
timeout 240 $R --nproc-per-node 4 --master-port 29802 bench.py --gpus 4 --config bert_large --warmup 10 > $O/bert_n4_w10.json 2> $O/bert_n4_w10.err; echo b=$?
timeout 240 $R --nproc-per-node 4 --master-port 29803 bench.py --gpus 4 --config bert_large > $O/bert_n4_plain.json 2> $O/bert_n4_plain.err; echo c=$?
