"""CUDA-graph capture of the public API: everything frob_inv launches is asynchronous on the
caller's stream (include/frobinv.h: no host sync unless host_info is requested or AUTO has to
read pivot ratios), including the blocked LU's fork to its high / low priority streams and the
join back.  A captured call replayed must equal the direct call bit for bit (the split-K GEMM
reduction is ordered, the pipelines are deterministic)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["frob", "zinv"])
@pytest.mark.parametrize("n", [1024, 4700], ids=["lu2", "blocked_getrf"])
def test_graph_replay_bitwise(n, which):
    import paper_2208_01239_b200 as fb
    z = torch.from_numpy(synth.config2(n, seed=3)).cuda()
    call = (lambda o: fb.inv(z, branch="a", out=o)) if which == "frob" else (lambda o: fb.zinv(z, out=o))
    direct = torch.empty_like(z)
    call(direct)
    out = torch.empty_like(z)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call(out)  # warm-up on the capture stream (workspace, attributes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call(out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, direct)
    r = np.linalg.norm(z.cpu().numpy() @ out.cpu().numpy() - np.eye(n)) if n <= 1024 else 0.0
    assert r <= 1e-11 * n
