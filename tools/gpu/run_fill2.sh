timeout 900 python -m pytest tests/test_gpu_host_order.py -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_fill2.json 2> gpurun_out/r2_bench_fill2.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_fill2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'], d['step_roofline']['frac'])"
timeout 1500 python -m pytest tests/test_gpu_papers_runner.py -m gpu -x -q 2>&1 | tail -2
