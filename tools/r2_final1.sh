#!/bin/bash
# Round-2 final check on one B200 (the driver's round-end tiers): build, the
# full GPU suite, smoke, the default bench line and the reference arm, the
# other configs at N=1, the ncu launch list and one ncu --set full capture of
# the owned kernels. Outputs under gpurun_out/r2final/.
set -u
OUT=gpurun_out/r2final
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1
echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "bench ref rc=$?"
for c in bert_large llama_1b3; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_n1_$c.json 2> $OUT/bench_n1_$c.err
  echo "bench $c rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adamw|accumulate" -c 4 \
    -o $OUT/owned $CMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
