"""Helper of test_gpu_papers_runner.py, run as its own process (the caching-allocator settings of
bench.py apply only before a process's first CUDA allocation).

Runs bench.py's pipelined Runner on the papers100M-shaped config for 1 + W + K passes -- the
driver's `--steps 20 --warmup 5` command -- and keeps the assembled rows of a few batches of the
last pass.  Prints one JSON line: allocator peaks against bench.py's HBM budget, and for every
kept batch whether its rows equal the oracle's sample gathered from the closed-form features.
"""
import json
import os
import sys

os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CHECK = [0, 1, 585, 1170, 1171]


def main():
    warmup, steps = int(sys.argv[1]), int(sys.argv[2])
    import bench
    import oracle
    import paper_2405_05231_b200 as dg
    from workload import feature_rows_np
    dev = torch.device("cuda", 0)
    inp = bench.make_inputs("papers", dev)
    cfg = inp[0]
    kept = {}
    passes = [0]

    total = 1 + max(warmup - 1, 2) + steps
    R = bench.Runner(dg, inp, 0, dev, pipelined=True)

    def observe(e, b, out):  # the rows of the checked batches of the last pass, as they are assembled
        passes[0] = max(passes[0], e + 1)
        if e == total - 1 and b in CHECK:
            with torch.cuda.stream(R.sB):
                kept[b] = out.view(torch.uint8).reshape(out.shape[0], -1).to("cpu", non_blocking=False)
    R.observe = observe
    R.run(1)
    R.run(max(warmup - 1, 2))
    R.run(steps)
    torch.cuda.synchronize()
    mem = bench.memory_report(dev, R)
    _, indptr, indices, seeds, feats, _, _ = inp
    del feats
    ref = oracle.sample(indptr.cpu().numpy(), indices.cpu().numpy(), seeds.cpu().numpy(), cfg["batch_size"],
                        list(cfg["fanout"]), bench.RNG_SEED, batches=CHECK, threads=8)
    ok = {}
    for r in ref:
        want = feature_rows_np(r.nodes, cfg["dim"]).view(np.uint8).reshape(len(r.nodes), -1)
        ok[str(r.bid)] = bool(r.bid in kept and np.array_equal(kept[r.bid].numpy(), want))
    print(json.dumps({"passes": passes[0], "memory": mem, "batches_equal": ok}))


if __name__ == "__main__":
    main()
