"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on the tiny config.

    compute-sanitizer --tool memcheck python tools/sanitize_tiny.py

Exercises every kernel family of the default path and the opt-in paths on the tiny config: both
a3 dedup paths, the layout with the pinned / HBM / O_DIRECT-file disk tiers, the assembly with
host windows on a second stream, bench.py's pipelined Runner (layout of pass e+1 next to the
assembly of pass e, 4 streams), the DGL-block variant, the trainer stub and the segmented disk
cache.  Exits non-zero on any CUDA or library error; the sanitizer reports its own findings.
"""
import os
import sys
import tempfile

# compute-sanitizer does not permit the driver's virtual-memory calls behind torch's expandable
# segments (cuMemCreate returns CUDA_ERROR_NOT_PERMITTED under the tool): plain cudaMalloc blocks
os.environ["PYTORCH_CUDA_ALLOC_CONF"] = "expandable_segments:False"
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    import paper_2405_05231_b200 as dg
    from workload import make_workload
    dev = torch.device("cuda", 0)
    w = make_workload("tiny")
    ip, ix, ft, sd = (t.to(dev) for t in (w.indptr, w.indices, w.features, w.seeds))
    fan, B = [10, 5], 256
    ctx = dg.Ctx(device=dev)
    for path in ("part", "table"):
        if path == "table":
            os.environ["DGNN_SAMPLE_DEDUP"] = "table"
        else:
            os.environ.pop("DGNN_SAMPLE_DEDUP", None)
        counts = torch.zeros(ip.numel() - 1, dtype=torch.int32, device=dev)
        dg.dgnn_sample(ctx, ip, ix, sd, B, fan, 7, 0, counts)
    os.environ.pop("DGNN_SAMPLE_DEDUP", None)
    gctx = dg.Ctx(device=dev, stream=torch.cuda.Stream(dev))
    with tempfile.TemporaryDirectory() as td:
        for stage in ("pinned", "hbm", "file"):
            L = dg.offline_layout(ctx, ip, ix, ft, sd, fan, B, 500, 1000, 7, group_size=3, stage=stage,
                                  file_path=os.path.join(td, "disk.bin"), direct_io=False)
            n = sum(1 for _ in L.assemble_epoch(host_window=3, gather_ctx=gctx))
            assert n == L.num_batches
            ctx.sync()
            gctx.sync()
            del L
        L = dg.offline_layout(ctx, ip, ix, ft, sd, fan, B, 500, 1000, 7, group_size=3, disk_budget_frac=0.9)
        for _ in L.train_epoch(host_window=2):
            pass
        ctx.sync()
        del L
    ctx.set_sample_mode(True)
    L = dg.offline_layout(ctx, ip, ix, ft, sd, fan, B, 500, 1000, 7, group_size=4)
    for _ in L.train_epoch():
        pass
    ctx.sync()
    ctx.set_sample_mode(False)
    del L
    inp = bench.make_inputs("tiny", dev)
    inp[0]["group_size"] = 2
    R = bench.Runner(dg, inp, 0, dev, pipelined=True)
    R.stage_piece = 64 << 10
    R.host_window = 3
    R.run(3)
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
