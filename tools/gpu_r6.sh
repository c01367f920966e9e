set -u
O=gpurun_out/r6
mkdir -p $O
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.json 2>&1; echo plain=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_gpt2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:accumulate_multi -c 2 -o $O/acc_multi python tools/ab_step.py --config bert_large --switch acc_microbatches --ml 12,4 --blocks 1 --steps 1 > $O/ncu_accm.log 2>&1; echo ncu2=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 2 --master-port 29802 bench.py --gpus 2 > $O/gpt2_n2.json 2> $O/gpt2_n2.err; echo n2=$?
