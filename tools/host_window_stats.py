"""How many host-tier rows would a window of W consecutive batches fetch if each
distinct row crossed PCIe once per window?  (design study for a9, papers-shaped)"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2405_05231_b200 as dg

dev = torch.device("cuda", 0)
inp = bench.make_inputs(sys.argv[1] if len(sys.argv) > 1 else "papers", dev)
R = bench.Runner(dg, inp, 0, dev, pipelined=False)
L = R.run(1, keep_last=True)
torch.cuda.synchronize()
no = L.samples.node_off_host
addr = L.addr[:L.samples.total_nodes]
nb = L.num_batches
out = {}
for W in (1, 2, 4, 8, 16, 32, 64, 128, 256, 586, nb):
    tot = 0
    acc = 0
    for b0 in range(0, nb, W):
        b1 = min(nb, b0 + W)
        a = addr[int(no[b0]):int(no[b1])]
        h = a[((a >> 30) & 3) == 1] & ((1 << 30) - 1)
        acc += h.numel()
        tot += torch.unique(h).numel()
    out[W] = {"accesses": acc, "distinct_per_window_sum": tot, "ratio": round(acc / max(tot, 1), 3)}
    print(W, out[W], flush=True)
json.dump(out, open("gpurun_out/host_window_stats.json", "w"))
