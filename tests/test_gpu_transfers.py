"""dgnn_upload (small host -> device tables carried in kernel parameters, 4000 bytes per launch;
above 256 KiB a copy-engine copy): the device bytes equal the host bytes for every size class,
including sizes that are not multiples of the chunk or of 4, and the upload is ordered on the
ctx stream before work enqueued after it."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nbytes", [0, 1, 3, 8, 3999, 4000, 4001, 12345, 64 << 10, (256 << 10) + 8])
def test_upload_bytes_equal(nbytes):
    import paper_2405_05231_b200 as dg
    ctx = dg.Ctx(device=0)
    rng = np.random.default_rng(nbytes)
    src = rng.integers(0, 256, nbytes, dtype=np.uint8)
    out = dg._abi.dgnn_upload(ctx, src, dtype=torch.uint8)
    src[:] = 0  # the call has consumed the host bytes by the time it returns
    torch.cuda.synchronize()
    assert out.numel() == nbytes
    assert np.array_equal(out.cpu().numpy(), rng_bytes(nbytes))


def rng_bytes(nbytes):
    return np.random.default_rng(nbytes).integers(0, 256, nbytes, dtype=np.uint8)


def test_upload_then_kernel_in_stream_order():
    """An upload followed by a library kernel reading the uploaded table on the same stream."""
    import paper_2405_05231_b200 as dg
    ctx = dg.Ctx(device=0)
    rows, rb = 5000, 64
    feats = torch.arange(rows * rb, dtype=torch.uint8, device="cuda").view(rows, rb)
    ids = np.random.default_rng(1).integers(0, rows, 3000).astype(np.int32)
    dev_ids = dg._abi.dgnn_upload(ctx, ids, dtype=torch.int32)
    out = torch.empty(len(ids), rb, dtype=torch.uint8, device="cuda")
    dg._abi.dgnn_gather_rows(ctx, feats, dev_ids, out)
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), feats.cpu()[torch.from_numpy(ids).long()])
