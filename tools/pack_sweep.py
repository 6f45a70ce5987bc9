"""Launch-configuration sweep of the a7 pack kernel on the papers-shaped epoch's own packed lists.

    python tools/pack_sweep.py [--config papers] [--reps 10]

Builds one offline layout (features in HBM), re-packs its packed lists with dgnn_pack under
DGNN_PACK_U (rows in flight per warp) x DGNN_PACK_BPS (CTAs per SM in the persistent grid), each
result compared byte for byte with the layout's own pack; prints one JSON line with the median
CUDA-event time and GB/s (algorithmic: rows x (2 x row_bytes + 4)) per setting.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import paper_2405_05231_b200 as dg
    from paper_2405_05231_b200 import _abi as A
    from bench import make_inputs
    dev = torch.device("cuda", 0)
    cfg, indptr, indices, seeds, feats, gpu_rows, host_rows = make_inputs(args.config, dev)
    ctx = dg.Ctx(device=0)
    L = dg.offline_layout(ctx, indptr, indices, feats, seeds, cfg["fanout"], cfg["batch_size"], gpu_rows, host_rows,
                          0x5EEDD15C, group_size=0, stage="hbm")
    torch.cuda.synchronize()
    nb, rb = L.num_batches, L.row_bytes
    tot = L.samples.total_nodes
    addr = torch.empty(tot, dtype=torch.int32, device=dev)
    pids = torch.empty(tot, dtype=torch.int32, device=dev)
    poff = torch.empty(nb + 1, dtype=torch.int64, device=dev)
    po = A.dgnn_classify(ctx, L.plan, L.samples, 0, nb, addr, pids, poff)
    R = int(po[-1])
    co = dg.dgnn_chunk_layout(po, rb)
    co_d = torch.as_tensor(co).to(dev)
    po_d = torch.as_tensor(po).to(dev)
    ref = L.arena_dev[:int(co[-1])].clone()
    del L, addr
    out = torch.empty(int(co[-1]), dtype=torch.uint8, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 2 x L2
    algo = R * (2 * rb + 4)
    res = {"config": args.config, "packed_rows": R, "row_bytes": rb, "algorithmic_bytes": algo, "runs": []}
    for u in (2, 4, 8):
        for bps in (2, 3, 4, 5, 6, 8):
            os.environ["DGNN_PACK_U"], os.environ["DGNN_PACK_BPS"] = str(u), str(bps)
            ts = []
            for r in range(args.reps + 2):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record(ctx.stream)
                dg.dgnn_pack(ctx, feats, pids[:R], po_d, co_d, R, int(co[-1]), out)
                b.record(ctx.stream)
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(a.elapsed_time(b))
            ok = bool(torch.equal(out, ref))
            ms = statistics.median(ts)
            res["runs"].append({"U": u, "bps": bps, "ms": round(ms, 4), "gbs": round(algo / ms / 1e6, 1), "equal": ok})
            out.zero_()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
