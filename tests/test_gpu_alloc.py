"""rpq_set_allocator: every device buffer of an evaluation comes from the
caller's allocator (here PyTorch's caching allocator); results stay exact."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2602_20748_b200")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if R.rpq_device_count() == 0:
        pytest.skip("no CUDA device")


def test_torch_caching_allocator():
    import torch
    torch.cuda.init()
    live = {}

    def alloc(n, s):
        p = torch.cuda.caching_allocator_alloc(n, stream=s)
        live[p] = n
        return p

    def free(p, s):
        live.pop(p)
        torch.cuda.caching_allocator_delete(p)

    g = synth.random_graph(3000, 12000, 3, seed=9)
    G = R.rpq_graph_load(g)
    a = R.rpq_compile(G, "(a|b)*c*")
    o = oracle.allpairs(g, "(a|b)*c*")
    want = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    want = want[np.lexsort((want[:, 1], want[:, 0]))]
    R.rpq_set_allocator(alloc, free)
    try:
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS)
        # what the result holds: its two pair columns and the per-source arrays
        assert sorted(live.values()) == sorted([4 * want.shape[0]] * 2 + [4 * 3000, 8 * 3000])
        assert np.array_equal(r.rows(), want)
        del r
        assert not live
    finally:
        R.rpq_set_allocator()
    assert np.array_equal(R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS).rows(), want)
