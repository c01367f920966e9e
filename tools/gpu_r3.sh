set -u
O=gpurun_out/r3
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x > $O/pytest_kernels.log 2>&1; echo pytest=$?; tail -2 $O/pytest_kernels.log
timeout 300 python tools/ab_step.py --config bert_large --switch acc_microbatches --ml 12,4 > $O/ab_accmb_bert.log 2>&1; echo ab=$?
timeout 400 $R --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 --config bert_large > $O/bert_n2.json 2> $O/bert_n2.err; echo bert2=$?
timeout 400 $R --nproc-per-node 4 --master-port 29804 bench.py --gpus 4 --config bert_large > $O/bert_n4.json 2> $O/bert_n4.err; echo bert4=$?
timeout 400 $R --nproc-per-node 4 --master-port 29805 bench.py --gpus 4 --config bert_large --offload off > $O/bert_n4_nooff.json 2> $O/bert_n4_nooff.err; echo bert4nooff=$?
grep -h -i "Error" $O/*.err | head -10
