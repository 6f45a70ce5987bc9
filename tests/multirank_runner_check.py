"""Helper of test_gpu_bench_contract.py: bench.py's Runner at world size > 1, every output checked.

Launched with torch.distributed.run (one process per rank).  Each rank runs three pipelined passes
of the tiny config with the given split (weak: one epoch per rank; epoch: one epoch split into
contiguous batch blocks) and GPU-tier mode (replicated; peer: partitioned over the ranks and read
through CUDA IPC peer mappings; nccl: partitioned, remote rows through the all-to-all exchange),
and compares every assembled batch of every pass with the oracle's direct gather.  The counts
and tier map are checked against the oracle over all ranks' batches, with the capacities the
mode implies (partitioned: world x the config's GPU rows, reading c16).

    python -m torch.distributed.run --nproc-per-node 2 tests/multirank_runner_check.py SPLIT MODE
"""
import os
import sys

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    split, mode = sys.argv[1], sys.argv[2]
    shard = len(sys.argv) > 3 and sys.argv[3] == "shard"  # feature table partitioned by node range
    import torch.distributed as dist

    import bench
    import oracle
    import paper_2405_05231_b200 as dg
    from paper_2405_05231_b200.layout import batch_range
    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group(os.environ.get("DGNN_BENCH_BACKEND", "gloo"), rank=rank, world_size=ws)
    cfg, indptr, indices, seeds, feats, gpu_rows, host_rows = bench.make_inputs("tiny", dev, shard_features=shard,
                                                                                rank=rank, ws=ws)
    cfg["group_size"] = 3
    B = cfg["batch_size"]
    nb_epoch = (seeds.numel() + B - 1) // B
    all_seeds = seeds
    base = None
    if split == "epoch":
        lo, hi = batch_range(nb_epoch, rank, ws)
        seeds = seeds[lo * B:min(hi * B, all_seeds.numel())]
        base = lo
    if mode != "replicated":
        gpu_rows *= ws
    inp = (cfg, indptr, indices, seeds, feats, gpu_rows, host_rows)
    got = []

    R = bench.Runner(dg, inp, rank, dev, pipelined=True)

    def observe(e, b, out):  # every assembled batch of every pass
        while len(got) <= e:
            got.append({})
        with torch.cuda.stream(R.sB):
            got[e][b] = out.view(torch.uint8).reshape(out.shape[0], -1).clone()
    R.observe = observe
    R.bid_base = base
    R.host_window = 2
    R.stage_piece = 64 << 10
    R.setup_gpu_tier(mode, ws)
    R.run(3)
    torch.cuda.synchronize()
    ip, ix, sd = indptr.cpu().numpy(), indices.cpu().numpy(), all_seeds.cpu().numpy()
    if shard:
        from workload import feature_rows_np
        f = feature_rows_np(np.arange(cfg["num_nodes"]), cfg["dim"])
    else:
        f = feats.cpu().numpy()
    if split == "epoch":
        ref_all = oracle.sample(ip, ix, sd, B, list(cfg["fanout"]), bench.RNG_SEED)
        mine = ref_all[base:base + (seeds.numel() + B - 1) // B]
    else:
        ref_all = []
        for r in range(ws):
            ref_all += oracle.sample(ip, ix, sd, B, list(cfg["fanout"]), bench.RNG_SEED, batch_id_base=r * nb_epoch)
        mine = ref_all[rank * nb_epoch:(rank + 1) * nb_epoch]
    bad = []
    assert len(got) == 3
    for e, outs in enumerate(got):
        if sorted(outs) != list(range(len(mine))):
            bad.append(f"pass {e}: batches {sorted(outs)}")
        for b, s in enumerate(mine):
            if b in outs and not np.array_equal(outs[b].cpu().numpy(), oracle.assemble(f, s.nodes)):
                bad.append(f"pass {e} batch {b}")
    counts = oracle.count_frequencies(ref_all, len(ip) - 1)
    tier_map, _, _ = oracle.select_tiers(counts, gpu_rows, host_rows)
    L = R.layout(0)  # one more layout: its counts / plan against the oracle
    R.ctxA.sync()
    if not np.array_equal(L.counts.cpu().numpy().view(np.uint32), counts):
        bad.append("counts")
    if not np.array_equal(L.plan.tier_map.cpu().numpy().view(np.uint32), tier_map):
        bad.append("tier map")
    # (the extra layout's slot barrier is matched on every rank: all call layout(0) once more)
    print(f"rank {rank}: " + ("ok" if not bad else "FAIL " + "; ".join(bad[:10])), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
