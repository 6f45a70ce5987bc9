#!/bin/bash
# Launch list of the default (pipelined) bench command + one full capture each of the window
# staging gather (k_gather_chunks), the pack (k_pack), the tier fill (k_gather) and the HBM part of
# the assembly (k_assemble_group); run under gpurun.
OUT=${OUT:-gpurun_out}
ARGS="bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_final.csv \
    python $ARGS > $OUT/ncu_bench_final.json 2> $OUT/ncu_bench_final.err
# (ncu matches the base function name, without template arguments: anchor both ends so that
# k_gather -- the tier fill -- does not also match k_gather_chunks)
for K in k_gather_chunks k_pack k_gather k_assemble_group; do
  N=$K
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$K\$" -s 2 -c 1 -o $OUT/prof_${N}_final -f \
      python $ARGS > /dev/null 2> $OUT/prof_${N}_final.err
done
