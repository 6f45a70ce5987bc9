#!/bin/bash
# End-of-round-2 lines of the other configs and modes with the final code (one GPU, under gpurun):
# products-shaped, Friendster-shaped bounded epoch, the O_DIRECT file disk tier with graph samples
# in the chunks, DGL blocks, the trainer stub, the segmented disk cache, and the unbridged staging
# schedule (A/B).  Each writes gpurun_out/r2_line_<name>.json (+ .err).
OUT=${OUT:-gpurun_out}
run() {
  name=$1; shift
  timeout 900 env "$@" > $OUT/r2_line_$name.json 2> $OUT/r2_line_$name.err
  echo "$name rc=$? $(python -c "import json,sys; d=json.load(open('$OUT/r2_line_$name.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" 2>/dev/null)"
}
run products      python bench.py --config products --steps 20 --warmup 5
run nobridge      DGNN_HOST_BRIDGE=0 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu
run friendster96  python bench.py --config friendster --num-seeds 98304 --steps 5 --warmup 3 --no-e2e --no-cpu
run file_embed    python bench.py --stage file --embed-graph --steps 3 --warmup 3 --no-e2e --no-cpu
run blocks        python bench.py --blocks --steps 10 --warmup 3 --no-e2e --cpu-batches 8
run train         python bench.py --train --steps 10 --warmup 3 --no-e2e --no-cpu
run diskcache95   python bench.py --disk-budget 0.95 --steps 10 --warmup 3 --no-e2e --no-cpu
run sequential    python bench.py --sequential --steps 10 --warmup 3 --no-e2e --no-cpu
