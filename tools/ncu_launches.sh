#!/bin/bash
# Launch list (gpu__time_duration.sum per launch, cold and serialized) of the default bench
# command; run under gpurun.  Summarize with tools/summarize_launches.py <csv> 4.
OUT=${OUT:-gpurun_out}
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_final.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $OUT/ncu_bench_final.json 2> $OUT/ncu_bench_final.err
