timeout 900 python -m pytest tests/test_gpu_bench_contract.py -m gpu -x -q -k "default_contract or opt_in" 2>&1 | tail -2
DGNN_ASM_OUT_BUDGET=2147483648 DGNN_TRACE_SAMPLE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_mask.json 2> gpurun_out/r2_bench_mask.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_mask.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'], d['step_roofline']['frac'], d['roofline']['frac'])
for t in d['device_timeline_ms'][-2:]: print(t)"
grep "dgnn_sample\]" gpurun_out/r2_bench_mask.err | tail -4
