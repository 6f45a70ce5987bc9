for ob in 2147483648 4294967296; do
DGNN_ASM_OUT_BUDGET=$ob DGNN_ASM_TRACE=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_ht$ob.json 2> gpurun_out/r2_bench_ht$ob.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_ht$ob.json').read().strip().splitlines()[-1]); print($ob, d['value'], d['ms_per_step'], d['memory']['max_reserved_gb'])
for t in d['device_timeline_ms'][-2:]: print(t)"
grep "host enqueue" gpurun_out/r2_bench_ht$ob.err
done
