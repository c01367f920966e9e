set -u
O=gpurun_out/r8
mkdir -p $O
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x > $O/pytest_kernels.log 2>&1; echo pytest=$?; tail -2 $O/pytest_kernels.log
timeout 600 python tools/kernel_bench.py > $O/kernel_bench.txt 2>&1; echo kb=$?
grep gelu $O/kernel_bench.txt
timeout 300 python bench.py --no-cpu-baseline > $O/gpt2_n1.json 2> $O/gpt2_n1.err; echo n1=$?
timeout 300 python bench.py --no-cpu-baseline --config bert_large > $O/bert_n1.json 2> $O/bert_n1.err; echo bert1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"colsum_kernel|gelu_fwd" -c 4 -o $O/gelu python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_gelu.log 2>&1; echo ncu=$?
timeout 900 python -m pytest tests/test_step_gpu.py -q -x > $O/pytest_step.log 2>&1; echo pytest_step=$?; tail -2 $O/pytest_step.log
