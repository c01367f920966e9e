#!/bin/bash
# Round-2 re-entry check on one B200: full GPU suite, smoke, the default bench
# line, its ncu launch list and one ncu --set full capture of the owned
# kernels. Outputs under gpurun_out/r2v/.
set -u
OUT=gpurun_out/r2v
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
echo "build rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?"
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1
echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "bench ref rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adamw|accumulate" -c 4 \
    -o $OUT/owned $CMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
