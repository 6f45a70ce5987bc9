timeout 900 python -m pytest tests/test_gpu_host_order.py -m gpu -x -q 2>&1 | tail -2
for ob in 1073741824 2147483648 4294967296; do
DGNN_ASM_OUT_BUDGET=$ob DGNN_TRACE_SAMPLE=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_ob$ob.json 2> gpurun_out/r2_bench_ob$ob.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_ob$ob.json').read().strip().splitlines()[-1]); print($ob, d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'])"
grep "dgnn_sample\]" gpurun_out/r2_bench_ob$ob.err | tail -2
done
