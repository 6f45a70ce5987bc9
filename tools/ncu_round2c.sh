#!/bin/bash
# End-of-round-2 evidence (after the PCIe-schedule changes): the launch list of the default bench
# command (pipelined, one timed pass) and one full capture each of the graded pack and the
# assembly's HBM kernel; run under gpurun, one GPU.
OUT=${OUT:-gpurun_out}
BENCH="bench.py --steps 1 --warmup 1 --stat-steps 1 --no-e2e --no-cpu"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r2c.csv \
    python $BENCH > $OUT/ncu_bench_r2c.json 2> $OUT/ncu_bench_r2c.err
for K in k_pack k_assemble_group; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" -s 3 -c 1 -o $OUT/prof_${K}_r2c -f \
      python $BENCH > /dev/null 2> $OUT/prof_${K}_r2c.err
done
