"""Individual vs batched packing (Sec. 5.2, Fig. 6) when the feature table is NOT in HBM.

    python tools/pack_streamed_bench.py [--config papers] [--budget-gb 8] [--file]

Builds one offline layout with the GPU path (features in HBM, as the bench does) to obtain the
epoch's packed lists, then re-packs them from a host-resident copy of the feature table:
  * individual: dgnn_pack reading every packed row on its own over PCIe (UVA), batch by batch
    (the paper's naive method);
  * batched: packing.pack_streamed -- partitions of C - 4 KiB x N bytes read once,
    sequentially (copy engine, or O_DIRECT pread with --file), rows routed on the GPU.
Both results are compared byte for byte with the HBM pack.  Prints one JSON line.
"""
import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="papers")
    ap.add_argument("--budget-gb", type=float, default=8.0)
    ap.add_argument("--file", action="store_true", help="batched packing reads an O_DIRECT feature file")
    args = ap.parse_args()
    import paper_2405_05231_b200 as dg
    from paper_2405_05231_b200 import _abi as A, packing
    from paper_2405_05231_b200.layout import HostBuffer
    from bench import make_inputs
    dev = torch.device("cuda", 0)
    cfg, indptr, indices, seeds, feats, gpu_rows, host_rows = make_inputs(args.config, dev)
    ctx = dg.Ctx(device=0)
    L = dg.offline_layout(ctx, indptr, indices, feats, seeds, cfg["fanout"], cfg["batch_size"], gpu_rows, host_rows,
                          0x5EEDD15C, group_size=0, stage="hbm")
    torch.cuda.synchronize()
    nb, rb, N = L.num_batches, L.row_bytes, feats.shape[0]
    tot = L.samples.total_nodes
    addr = torch.empty(tot, dtype=torch.int32, device=dev)
    pids = torch.empty(tot, dtype=torch.int32, device=dev)
    poff = torch.empty(nb + 1, dtype=torch.int64, device=dev)
    po = A.dgnn_classify(ctx, L.plan, L.samples, 0, nb, addr, pids, poff)
    del addr
    R = int(po[-1])
    co = dg.dgnn_chunk_layout(po, rb)
    co_d = torch.as_tensor(co).to(dev)
    ref = L.arena_dev[:int(co[-1])].clone()  # the HBM pack of the layout
    res = {"config": args.config, "batches": nb, "packed_rows": R, "row_bytes": rb,
           "table_gb": round(N * rb / 1e9, 2)}
    # host copy of the feature table
    hb = HostBuffer(N * rb)
    hb.tensor.copy_(feats.view(torch.uint8).reshape(-1))
    host_feats = hb.tensor.view(torch.float32).view(N, -1)
    del feats, L
    torch.cuda.empty_cache()
    out = torch.empty(int(co[-1]), dtype=torch.uint8, device=dev)

    def timed(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        t = time.perf_counter()
        r = fn()
        b.record(ctx.stream)
        torch.cuda.synchronize()
        return r, a.elapsed_time(b), (time.perf_counter() - t) * 1e3

    po_rel = torch.as_tensor(po).to(dev)
    _, ms_ind, _ = timed(lambda: dg.dgnn_pack(ctx, host_feats, pids[:R], po_rel, co_d, R, int(co[-1]), out))
    res["individual"] = {"ms": round(ms_ind, 1), "source_gb": round(R * rb / 1e9, 2),
                         "gbs": round(R * rb / ms_ind / 1e6, 1), "equal": bool(torch.equal(out, ref))}
    idx = dg.DiskIndex(ctx, pids[:R], poff, po, N)
    del pids
    part = packing.partition_rows(int(args.budget_gb * 2**30), nb, rb)
    src = hb
    if args.file:
        path = os.path.join(tempfile.mkdtemp(prefix="dgnn_feat_", dir=os.environ.get("DGNN_TMP", "/tmp")), "f.bin")
        size = packing.write_feature_file(path, host_feats)
        src = A.DiskFile(path, size, direct=True, create=False)
    out.zero_()
    rep, ms_bat, host_bat = timed(lambda: packing.pack_streamed(ctx, idx, src, N, rb, co_d, out, part))
    res["batched"] = {"ms": round(ms_bat, 1), "host_ms": round(host_bat, 1), "partition_rows": part,
                      "partitions_read": rep["parts"], "source_gb": round(rep["bytes"] / 1e9, 2),
                      "gbs": round(rep["bytes"] / ms_bat / 1e6, 1), "pages": rep["pages"],
                      "source": "O_DIRECT file" if args.file else "pinned host (copy engine)",
                      "equal": bool(torch.equal(out, ref))}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
