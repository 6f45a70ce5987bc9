"""bench.py's pipelined Runner produces the oracle's batches (run on a B200 with -m gpu).

The Runner overlaps pass e+1's layout with pass e's assembly, starts an assembly at the end of
its pass's classify step and lets each run wait only for the stage-out pieces holding its own
chunks (Runner._ready, Layout.wait_chunks).  Here the tiny configuration is split into four
packing groups staged out in small pieces, three passes run back to back, and every assembled
batch of every pass is compared byte for byte with the oracle's direct gather.
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("pipelined", [True, False])
def test_runner_passes_equal_the_oracle(pipelined):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import bench
    import paper_2405_05231_b200 as dg
    dev = torch.device("cuda", 0)
    inp = bench.make_inputs("tiny", dev)
    cfg = inp[0]
    cfg["group_size"] = 2  # 4 packing groups: packs and stage-outs interleave with the next assembly
    got = []

    class Checked(bench.Runner):
        def _assemble(self, L, ev_l):
            self.sB.wait_event(ev_l)
            outs = {}
            for b, out in L.assemble_epoch(ctx=self.ctxB, host_window=3, gather_ctx=self.ctxG, ws=self.asm_ws):
                with torch.cuda.stream(self.sB):
                    outs[b] = out.clone()
            got.append(outs)
            ev = torch.cuda.Event()
            ev.record(self.sB)
            return ev

    R = Checked(dg, inp, 0, dev, pipelined=pipelined)
    R.stage_piece = 64 << 10
    R.run(3)
    torch.cuda.synchronize()
    _, indptr, indices, seeds, feats, _, _ = inp
    ref = oracle.sample(indptr.cpu().numpy(), indices.cpu().numpy(), seeds.cpu().numpy(), cfg["batch_size"],
                        list(cfg["fanout"]), bench.RNG_SEED)
    f = feats.cpu().numpy()
    assert len(got) == 3
    for outs in got:
        assert sorted(outs) == list(range(len(ref)))
        for b, s in enumerate(ref):
            assert np.array_equal(outs[b].view(torch.uint8).reshape(outs[b].shape[0], -1).cpu().numpy(),
                                  oracle.assemble(f, s.nodes)), f"batch {b}"
