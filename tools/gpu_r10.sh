set -u
O=gpurun_out/r10
mkdir -p $O
timeout 600 python -m pytest tests/test_step_gpu.py tests/test_kernels_gpu.py -q -x > $O/pytest.log 2>&1; echo pytest=$?; tail -3 $O/pytest.log
timeout 300 python tools/host_bound.py > $O/host_bound.txt 2>&1; echo hb=$?; cat $O/host_bound.txt | tail -1
timeout 300 python bench.py --no-cpu-baseline > $O/gpt2_n1_graph.json 2> $O/gpt2_n1_graph.err; echo g=$?
timeout 300 python bench.py --no-cpu-baseline --graph off > $O/gpt2_n1_eager.json 2> $O/gpt2_n1_eager.err; echo e=$?
timeout 300 python bench.py --no-cpu-baseline --config bert_large > $O/bert_n1_graph.json 2> $O/bert_n1_graph.err; echo bg=$?
timeout 300 python bench.py --no-cpu-baseline --config llama_1b3 > $O/llama_n1_graph.json 2> $O/llama_n1_graph.err; echo lg=$?
tail -3 $O/*.err | grep -i error | head
