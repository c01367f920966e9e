set -u
O=gpurun_out/r5
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 python -m pytest tests/test_step_gpu.py -q -x -k offload > $O/pytest_off.log 2>&1; echo pytest=$?; tail -2 $O/pytest_off.log
timeout 300 python tools/ab_step.py --config bert_large --switch offload --offload-schedule checkpoints --ml 19,2 --blocks 4 > $O/ab_offck_19x2.log 2>&1; echo ab=$?
timeout 400 $R --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --config bert_large --trace-dir $O/trace_n4 > $O/bert_n4.json 2> $O/bert_n4.err; echo bert4=$?
timeout 400 $R --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 --config bert_large > $O/bert_n2.json 2> $O/bert_n2.err; echo bert2=$?
grep -h -i "Error" $O/*.err | head -10
