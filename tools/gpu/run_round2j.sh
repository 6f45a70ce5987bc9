timeout 900 python -m pytest tests/test_gpu_bench_runner.py tests/test_gpu_bench_contract.py -m gpu -x -q 2>&1 | tail -2
DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_early.json 2> gpurun_out/r2_bench_early.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_early.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'], d['step_roofline']['frac'], d['roofline']['frac'])
for t in d['device_timeline_ms'][-2:]: print({k:v for k,v in t.items() if k!='host_ms'})"
grep "asm-trace" gpurun_out/r2_bench_early.err | tail -11
timeout 1500 python -m pytest tests/test_gpu_papers_runner.py -m gpu -x -q 2>&1 | tail -2
