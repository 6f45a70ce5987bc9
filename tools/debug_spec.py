import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2405_05231_b200 as dg
from workload import make_workload
w = make_workload("tiny", num_nodes=1000, num_edges=10_000, num_seeds=800, batch_size=8, fanout=(5, 5))
ip, ix, sd = w.indptr.numpy(), w.indices.numpy(), w.seeds.numpy()
feats = w.features.numpy()
dev = torch.device("cuda", 0)
ctx = dg.Ctx(device=0)
L = dg.offline_layout(ctx, w.indptr.to(dev), w.indices.to(dev), w.features.to(dev), w.seeds.to(dev), [5, 5], 8, 50, 100, 0x5EEDD15C, group_size=16)
ctx.sync()
no = L.samples.node_off_host
addr = L.addr.cpu().numpy().view(np.uint32)
print("groups", L.assembly_groups(), "arena", L.stats["arena_bytes"], "batch_chunk[:3]", L.batch_chunk[:3])
for b, out in L.assemble_epoch():
    nodes = L.samples.nodes[no[b]:no[b+1]].cpu().numpy()
    exp = oracle.assemble(feats, nodes)
    got = out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy()
    bad = np.nonzero((got != exp).any(1))[0]
    if len(bad):
        a = addr[no[b]:no[b+1]]
        tiers = a[bad] >> 30
        print("batch", b, "bad rows", len(bad), "of", len(nodes), "tiers of bad", np.bincount(tiers, minlength=3), "tiers all", np.bincount(a >> 30, minlength=3))
        # which source row did we get?
        j = bad[0]
        m = np.nonzero((feats.view(np.uint8).reshape(1000, -1) == got[j]).all(1))[0]
        print("  row", j, "node", nodes[j], "addr tier", a[j] >> 30, "slot", a[j] & ((1<<30)-1), "got node", m)
        if b > 3: break
# single-batch API for comparison
out = torch.empty((no[1]-no[0], 128), dtype=torch.float32, device=dev)
L.assemble(0, out)
ctx.sync()
nodes = L.samples.nodes[no[0]:no[1]].cpu().numpy()
print("single-batch API ok:", np.array_equal(out.view(torch.uint8).reshape(out.shape[0], -1).cpu().numpy(), oracle.assemble(feats, nodes)))
