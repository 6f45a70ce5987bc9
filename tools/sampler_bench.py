"""Sampler alone (a1-a3 + access counter) on a whole epoch, both dedup paths.

    python tools/sampler_bench.py [--config papers] [--reps 3]

Times dgnn_sample over the config's epoch with CUDA events on the ctx stream (nothing else on the
GPU), per dedup path (DGNN_SAMPLE_DEDUP unset = partitioned shared-memory buckets, "table" = the
per-batch global hash sets), prints the per-kernel-family split, and checks that both paths give
byte-identical samples and counts (the oracle parity of each path is in tests/).
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    ap.add_argument("--paths", default="part,table")
    args = ap.parse_args()
    import paper_2405_05231_b200 as dg
    from workload import CONFIGS, make_graph, make_seeds
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[args.config]
    t = time.time()
    indptr, indices = make_graph(cfg["num_nodes"], cfg["num_edges"], cfg["degree"], cfg["skew"], 0, dev)
    seeds = make_seeds(cfg["num_nodes"], cfg["num_seeds"], 0, dev)
    torch.cuda.synchronize()
    print(f"graph {args.config} in {time.time() - t:.1f}s", file=sys.stderr)
    N = indptr.numel() - 1
    res = {"config": args.config}
    keep = {}
    for path in args.paths.split(","):
        if path == "table":
            os.environ["DGNN_SAMPLE_DEDUP"] = "table"
        else:
            os.environ.pop("DGNN_SAMPLE_DEDUP", None)
        if path == "part-sort":  # bitonic order in every bucket instead of the counting order
            os.environ["DGNN_SAMPLE_ORDER"] = "sort"
        else:
            os.environ.pop("DGNN_SAMPLE_ORDER", None)
        ctx = dg.Ctx(device=dev)
        counts = torch.zeros(N, dtype=torch.int32, device=dev)
        times, stats = [], None
        for r in range(args.reps + 1):
            counts.zero_()
            ctx.reset_stats()
            ctx.set_timing(r == args.reps)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S = dg.dgnn_sample(ctx, indptr, indices, seeds, cfg["batch_size"], cfg["fanout"], 0x5EEDD15C, 0, counts)
            e1.record()
            torch.cuda.synchronize()
            if r > 0 and r < args.reps:
                times.append(e0.elapsed_time(e1))
            if r == args.reps:
                stats = {k: v for k, v in ctx.kernel_stats().items() if v["launches"]}
            if r < args.reps:
                del S
        ms = sorted(times)[len(times) // 2] if times else float("nan")
        res[path] = {"ms_per_epoch_median": round(ms, 2), "ms_all": [round(x, 2) for x in times],
                     "kernel_ms": {k: round(v["ms"], 2) for k, v in stats.items()},
                     "launches": {k: v["launches"] for k, v in stats.items()},
                     "nodes": int(S.total_nodes), "edges": int(S.total_edges)}
        keep[path] = (S.nodes.clone(), S.src_local.clone(), S.eptr.clone(), counts.clone())
        print(path, json.dumps(res[path]), file=sys.stderr)
        del S
        ctx.close()
    if len(keep) >= 2:
        a = next(iter(keep.values()))
        res["paths_identical"] = all(all(torch.equal(x, y) for x, y in zip(a, b)) for b in keep.values())
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
