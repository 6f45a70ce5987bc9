DGNN_TRACE_SAMPLE=1 timeout 600 python tools/contention_probe.py 2>&1 | grep -v "^\[bench\]" | tail -20
