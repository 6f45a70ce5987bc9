DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_ht3.json 2> gpurun_out/r2_bench_ht3.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_ht3.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'], d['step_roofline']['frac'])
for t in d['device_timeline_ms'][-3:]: print(t)"
grep "asm-trace" gpurun_out/r2_bench_ht3.err | head -12
