set -u
O=gpurun_out/r4
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python tools/ab_step.py --config bert_large --switch offload --ml 19,2 --blocks 4 > $O/ab_off_19x2.log 2>&1; echo ab=$?
timeout 300 python tools/ab_step.py --config bert_large --switch offload --ml 10,2 --blocks 4 > $O/ab_off_10x2.log 2>&1; echo ab=$?
timeout 400 $R --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 --config bert_large --steps 5 --trace-dir $O/trace_n2 > $O/bert_n2.json 2> $O/bert_n2.err; echo bert2=$?
grep -h -i "Error" $O/*.err | head -10
