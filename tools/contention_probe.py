"""Host-side contention probe: dgnn_sample's enqueue time (DGNN_TRACE_SAMPLE=1 prints it) alone and
while a second host thread issues CUDA calls on another stream -- (a) small async copies, (b) tiny
kernel launches through torch, (c) pure Python work holding the GIL.  Prints the per-call traces
on stderr and a JSON summary of the wall times on stdout.

    DGNN_TRACE_SAMPLE=1 python tools/contention_probe.py
"""
import json
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2405_05231_b200 as dg
    from workload import CONFIGS, make_graph, make_seeds
    dev = torch.device("cuda", 0)
    cfg = CONFIGS["papers"]
    indptr, indices = make_graph(cfg["num_nodes"], cfg["num_edges"], cfg["degree"], cfg["skew"], 0, dev)
    seeds = make_seeds(cfg["num_nodes"], cfg["num_seeds"], 0, dev)
    ctx = dg.Ctx(device=dev)
    counts = torch.zeros(indptr.numel() - 1, dtype=torch.int32, device=dev)
    side = torch.cuda.Stream(dev)
    hb = dg.HostBuffer(64 << 20)
    d = torch.empty(64 << 20, dtype=torch.uint8, device=dev)
    x = torch.zeros(1024, device=dev)
    stop = threading.Event()

    def copies():
        with torch.cuda.stream(side):
            while not stop.is_set():
                for i in range(256):
                    d[i << 18:(i + 1) << 18].copy_(hb.tensor[i << 18:(i + 1) << 18], non_blocking=True)
                side.synchronize()

    def launches():
        with torch.cuda.stream(side):
            while not stop.is_set():
                for _ in range(256):
                    x.add_(1.0)
                side.synchronize()

    def python_only():
        while not stop.is_set():
            s = 0
            for i in range(100000):
                s += i

    out = {}
    for name, fn in [("alone", None), ("copies", copies), ("launches", launches), ("python", python_only)]:
        th = None
        if fn is not None:
            stop.clear()
            th = threading.Thread(target=fn, daemon=True)
            th.start()
            time.sleep(0.2)
        times = []
        for _ in range(3):
            counts.zero_()
            torch.cuda.synchronize()
            t = time.time()
            S = dg.dgnn_sample(ctx, indptr, indices, seeds, cfg["batch_size"], cfg["fanout"], 0x5EEDD15C, 0, counts)
            times.append(round((time.time() - t) * 1e3, 1))
            del S
        if th is not None:
            stop.set()
            th.join()
        out[name] = times
        print(name, times, file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
