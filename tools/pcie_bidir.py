"""PCIe copy-engine bandwidth on this box: H2D alone, D2H alone, and both at once (separate streams),
from pinned host memory (dgnn_host_alloc) -- the floor of a step that moves H2D and D2H bytes
concurrently.  Prints one JSON line.

    python tools/pcie_bidir.py [--gib 2]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=2.0)
    args = ap.parse_args()
    import paper_2405_05231_b200 as dg
    n = int(args.gib * (1 << 30))
    dev = torch.device("cuda", 0)
    h1, h2 = dg.HostBuffer(n), dg.HostBuffer(n)
    d1 = torch.empty(n, dtype=torch.uint8, device=dev)
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fns):
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            evs = []
            for fn, st in fns:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                with torch.cuda.stream(st):
                    fn()
                b.record(st)
                evs.append((a, b))
            torch.cuda.synchronize()
            ms = max(a.elapsed_time(b) for a, b in evs)
            best = max(best, len(fns) * n / (ms / 1e3) / 1e9)
        return best

    h2d = lambda: d1.copy_(h1.tensor, non_blocking=True)
    d2h = lambda: h2.tensor.copy_(d2, non_blocking=True)
    out = {"bytes_per_copy": n,
           "h2d_gbs": round(timed([(h2d, s1)]), 2),
           "d2h_gbs": round(timed([(d2h, s2)]), 2),
           "both_total_gbs": round(timed([(h2d, s1), (d2h, s2)]), 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
