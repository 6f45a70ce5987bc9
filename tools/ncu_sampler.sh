#!/bin/bash
# ncu --set full of the sampler kernels at hop 2 of the first sampling group (papers-shaped)
OUT=${OUT:-gpurun_out}
ARGS="bench.py --config papers --steps 1 --warmup 1 --no-e2e --no-cpu"
run() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c $3 -o $OUT/prof_$4 -f python $ARGS > /dev/null 2> $OUT/prof_$4.err; }
run k_insert 2 1 insert
run scan_kernel 4 2 scan
run k_bucket_sort_assign 2 1 bsort
run k_sample_hop 2 1 hop
run k_remap 2 1 remap
run k_assemble_group 4 1 asm
