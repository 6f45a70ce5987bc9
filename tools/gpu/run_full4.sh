timeout 2700 python -X faulthandler -m pytest tests -m gpu -x -v -p no:cacheprovider > gpurun_out/r2_gputests_full_v.log 2>&1; echo rc=$?
grep -n "FAILED\|ERROR\|Fatal\|passed\|failed" gpurun_out/r2_gputests_full_v.log | tail -6
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_final2.json 2> gpurun_out/r2_bench_final2.err; tail -1 gpurun_out/r2_bench_final2.err
python -c "
import json;d=json.loads(open('gpurun_out/r2_bench_final2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['cpu_baseline']['value'], d['memory']['max_reserved_gb'], d['step_roofline']['frac'], d['roofline']['frac'], d['clocks'])"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
