for conn in 8 32; do
CUDA_DEVICE_MAX_CONNECTIONS=$conn timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2_bench_conn$conn.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_conn$conn.json').read().strip().splitlines()[-1])
tl=d['device_timeline_ms']; gaps=[round(tl[i+1]['pack_wait']-tl[i]['assemble_end'],1) for i in range(len(tl)-1)]
print($conn, d['value'], d['ms_per_step'], gaps[-4:], [round(t['assemble_end']-t['assemble_start'],1) for t in tl[-4:]])"
done
