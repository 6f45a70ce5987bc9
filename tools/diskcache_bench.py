"""Measure the segmented disk cache (Sec. 5.1) on a real offline layout of a config.

    python tools/diskcache_bench.py [--config papers] [--fractions 1.0,0.9,0.8,0.7]

Builds one offline layout (a1-a7) with the GPU path, then on its packed lists times
dgnn_disk_index_build, dgnn_disk_search (heuristic m = 1, budget = fraction x the
packed-only space), dgnn_disk_plan_build (k = 4) and dgnn_disk_cache_fill, and reports
Eq. 2 space / I/O pages of the chosen plan next to the packed-only layout and to the
identity (no-reorder) order.  Prints one JSON line.  No oracle is involved.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, stream):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    t = time.perf_counter()
    out = fn()
    b.record(stream)
    torch.cuda.synchronize()
    return out, a.elapsed_time(b), (time.perf_counter() - t) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers")
    ap.add_argument("--fractions", default="1.0,0.95,0.9,0.8,0.7")
    ap.add_argument("--k", type=int, default=4)
    args = ap.parse_args()
    import paper_2405_05231_b200 as dg
    from paper_2405_05231_b200 import _abi as A
    from bench import make_inputs
    dev = torch.device("cuda", 0)
    cfg, indptr, indices, seeds, feats, gpu_rows, host_rows = make_inputs(args.config, dev)
    ctx = dg.Ctx(device=0)
    L = dg.offline_layout(ctx, indptr, indices, feats, seeds, cfg["fanout"], cfg["batch_size"], gpu_rows, host_rows,
                          0x5EEDD15C, group_size=cfg.get("group_size", 0), stage="hbm")
    torch.cuda.synchronize()
    nb = L.num_batches
    row_bytes = L.row_bytes
    N = indptr.numel() - 1
    # the packed lists of the layout (DISK rows of each batch, local order): re-run a6
    tot = L.samples.total_nodes
    addr = torch.empty(tot, dtype=torch.int32, device=dev)
    pids = torch.empty(tot, dtype=torch.int32, device=dev)
    poff = torch.empty(nb + 1, dtype=torch.int64, device=dev)
    po = A.dgnn_classify(ctx, L.plan, L.samples, 0, nb, addr, pids, poff)
    R = int(po[-1])
    del addr
    s_ = ctx.stream
    idx, ms_index, _ = timed(lambda: dg.DiskIndex(ctx, pids[:R], poff, po, N), s_)
    packed_only = int(sum((np.diff(po) * row_bytes + 4095) // 4096))
    res = {"config": args.config, "batches": nb, "packed_rows": R, "row_bytes": row_bytes,
           "packed_only_pages": packed_only, "ms_index_build": round(ms_index, 2), "runs": []}
    sl = list(range(1, min(nb, 32) + 1))
    _, ms_space32, _ = timed(lambda: dg.dgnn_disk_space(ctx, idx, row_bytes, sl, 1), s_)
    res["ms_space_32_s_values"] = round(ms_space32, 2)
    for f in [float(x) for x in args.fractions.split(",")]:
        budget = int(f * packed_only)
        (s, pages), ms_search, host_search = timed(lambda: dg.dgnn_disk_search(ctx, idx, row_bytes, budget, 1), s_)
        run = {"fraction": f, "budget_pages": budget, "s": s, "search_ms": round(ms_search, 2),
               "search_host_ms": round(host_search, 2)}
        if s > 0:
            P, ms_plan, host_plan = timed(lambda: dg.dgnn_disk_plan_build(ctx, idx, row_bytes, s, 1, args.k, 7), s_)
            Pi = dg.dgnn_disk_plan_build(ctx, idx, row_bytes, s, 1, args.k, 7, reorder=False)
            # Algorithm 1 line 8 as printed (scalar MinHash over the k functions) at k and at 1
            lit = {kk: dg.dgnn_disk_plan_build(ctx, idx, row_bytes, s, 1, kk, 7, literal=True).io_pages
                   for kk in sorted({1, args.k})}
            cache = torch.empty(max(P.cache_pages, 1) * 4096, dtype=torch.uint8, device=dev)
            _, ms_fill, _ = timed(lambda: dg.dgnn_disk_cache_fill(ctx, P, feats, cache), s_)
            run.update(space_pages=P.space_pages, io_pages=P.io_pages, io_pages_identity=Pi.io_pages,
                       io_pages_literal={str(kk): v for kk, v in lit.items()},
                       cache_pages=P.cache_pages, chunk_pages=P.chunk_pages, cache_rows=P.n_cache,
                       packed_rows=P.n_packed, requests=P.n_req, plan_ms=round(ms_plan, 2),
                       plan_host_ms=round(host_plan, 2), fill_ms=round(ms_fill, 3),
                       fill_gbs=round(2 * P.n_cache * row_bytes / ms_fill / 1e6, 1) if ms_fill > 0 else None,
                       read_amplification=round(P.io_pages * 4096 / max(R * row_bytes, 1), 4))
            del P, Pi, cache
        res["runs"].append(run)
        print(json.dumps(run), file=sys.stderr, flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
