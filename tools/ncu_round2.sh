#!/bin/bash
# Round-2 evidence: the launch list of the default bench command (pipelined, one timed pass) and
# one full capture each of the graded pack, the assembly's HBM kernel and the round-2 sampler
# kernels (thread-per-node draws, partitioned dedup and its bucketing, range-major counter);
# run under gpurun.
OUT=${OUT:-gpurun_out}
BENCH="bench.py --steps 1 --warmup 1 --stat-steps 1 --no-e2e --no-cpu"
SAMPLER="tools/sampler_bench.py --config papers --reps 0 --paths part"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r2.csv \
    python $BENCH > $OUT/ncu_bench_r2.json 2> $OUT/ncu_bench_r2.err
for K in k_pack k_assemble_group k_sample_hop_t k_part_dedup k_cnt_ranges k_part_tile; do
  case $K in k_pack|k_assemble_group) CMD=$BENCH ;; *) CMD=$SAMPLER ;; esac
  SKIP=3; [ $K = k_cnt_ranges ] && SKIP=0  # one counter launch per sampler epoch
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" -s $SKIP -c 1 -o $OUT/prof_${K}_r2 -f \
      python $CMD > /dev/null 2> $OUT/prof_${K}_r2.err
done
