set -u
O=gpurun_out/r22
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"adamw|accumulate_kernel" -c 3 -o $O/step_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --graph off > $O/ncu_full.log 2>&1; echo ncu=$?
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $R --nproc-per-node 4 --master-port 29811 bench_collectives.py --sizes-mb 16 256 1024 --algos route auto owner symm > $O/collectives_n4.jsonl 2> $O/collectives_n4.err; echo c4=$?
timeout 600 $R --nproc-per-node 2 --master-port 29812 bench_collectives.py --sizes-mb 16 256 1024 --algos route auto owner symm > $O/collectives_n2.jsonl 2> $O/collectives_n2.err; echo c2=$?
