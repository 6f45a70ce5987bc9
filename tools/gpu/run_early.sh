timeout 900 python -m pytest tests/test_gpu_host_order.py tests/test_gpu_bench_runner.py tests/test_gpu_bench_contract.py -m gpu -x -q 2>&1 | tail -3
DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_early2.json 2> gpurun_out/r2_bench_early2.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_early2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'], d['step_roofline']['frac'])
for t in d['device_timeline_ms'][-2:]: print({k:v for k,v in t.items() if k!='host_ms'})"
grep "asm-trace" gpurun_out/r2_bench_early2.err | tail -10
DGNN_EARLY_PREFETCH=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_noearly.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_noearly.json').read().strip().splitlines()[-1]); print('no early', d['value'], d['ms_per_step'])"
timeout 1500 python -m pytest tests/test_gpu_papers_runner.py -m gpu -x -q 2>&1 | tail -2
