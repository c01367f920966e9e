set -u
O=gpurun_out/r16
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python -m pytest tests/test_step_gpu.py -q -x -k "offload or graph" > $O/pytest.log 2>&1; echo p=$?; tail -1 $O/pytest.log
for i in 1 2; do
timeout 240 $R --nproc-per-node 4 --master-port 2980$i bench.py --gpus 4 --config bert_large > $O/bert_n4_$i.json 2> $O/bert_n4_$i.err; echo a=$?
done
timeout 240 $R --nproc-per-node 2 --master-port 29803 bench.py --gpus 2 --config bert_large > $O/bert_n2.json 2> $O/bert_n2.err; echo b=$?
