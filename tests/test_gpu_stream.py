"""GPU parity of the streamed all-pairs output: pieces
delivered to the host in (src, dst) order under a small device budget (many
source chunks, many pieces) must concatenate to the oracle's sorted pairs."""
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


@pytest.mark.parametrize("rx", ["(a|b)*c*", "a b* c", "c+"])
def test_stream_matches_oracle(rx):
    g = synth.random_graph(3000, 12000, 3, seed=5)
    G = R.rpq_graph_load(g)
    a = R.rpq_compile(G, rx)
    o = oracle.allpairs(g, rx)
    want = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    want = want[np.lexsort((want[:, 1], want[:, 0]))]
    # ~50 K pairs of device budget and 10 K-pair pieces: many chunks and pieces
    tot, got = R.rpq_eval_allpairs_stream(G, a, device_budget_bytes=400_000, piece_pairs=10_000)
    assert tot == want.shape[0]
    assert np.array_equal(got, want)
    # shards partition the chunks; the union is the whole result
    parts = [R.rpq_eval_allpairs_stream(G, a, device_budget_bytes=400_000, shard_index=i, shard_count=3)[1]
             for i in range(3)]
    u = np.concatenate(parts)
    assert np.array_equal(u[np.lexsort((u[:, 1], u[:, 0]))], want)


def test_stream_early_stop():
    g = synth.random_graph(2000, 8000, 3, seed=6)
    G = R.rpq_graph_load(g)
    a = R.rpq_compile(G, "(a|b)*c*")
    seen = []
    tot, _ = R.rpq_eval_allpairs_stream(G, a, sink=lambda s, d: seen.append(s.size) or True, piece_pairs=1000)
    assert len(seen) == 1 and tot == seen[0] == 1000
