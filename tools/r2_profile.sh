#!/bin/bash
# Round-2 single-GPU profiling pass (gpurun, 1 GPU): the bench line, the
# launch list of the same command under ncu (per-launch device times,
# cold-cache and serialised: compare shares), and one ncu --set full capture
# of the owned kernels (AdamW, accumulate). Outputs under gpurun_out/r2p/.
set -u
OUT=gpurun_out/r2p
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
$CMD > $OUT/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"adamw|accumulate" -c 4 \
    -o $OUT/owned $CMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_n1.json 2> $OUT/bench_n1.err
echo "bench rc=$?"
for c in bert_large llama_1b3; do
  timeout 600 python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline \
    > $OUT/bench_n1_$c.json 2> $OUT/bench_n1_$c.err
  echo "bench $c rc=$?"
done
