"""frob_inv_batched_host (include/frobinv.h): batched Frobenius inversion with pinned host
buffers, pipelined in chunks on two library-owned copy streams.  Results and info must equal
the device-resident frob_inv_batched bit for bit, with ragged last chunks and with one chunk."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,batch,chunk", [(32, 1000, 300), (128, 50, 16), (64, 7, 64), (5, 3, 1)])
def test_batched_host_equals_device(n, batch, chunk):
    import paper_2208_01239_b200 as fb
    zh = torch.from_numpy(synth.batch(n, batch, seed=2)).pin_memory()
    xh = torch.empty_like(zh).pin_memory()
    xh2, info = fb.inv_batched_host(zh, xh, chunk=chunk)
    assert xh2.data_ptr() == xh.data_ptr()
    x_dev, info_dev, _ = fb.inv_batched(zh.cuda())
    assert torch.equal(xh, x_dev.cpu())
    assert torch.equal(info, info_dev.cpu().to(torch.int32))
