#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the papers-shaped bench; run under gpurun.
OUT=${OUT:-gpurun_out}
CFG=${CFG:-papers}
ARGS="bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu --sequential"
# 1) launch list of the bench command (cold-cache, serialised: compare shares)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$CFG.csv \
    python $ARGS > $OUT/ncu_bench_$CFG.json 2> $OUT/ncu_bench_$CFG.err
# 2) full sets of the top kernels
for K in k_pack k_assemble_group k_gather_dev k_gather; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K<" -s 1 -c 1 -o $OUT/prof_${K}_$CFG -f \
      python $ARGS > /dev/null 2> $OUT/prof_${K}_$CFG.err
done
