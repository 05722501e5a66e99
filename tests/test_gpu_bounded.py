"""Length-bounded RPQs ("length constraints
can be naturally enforced by controlling traversal depth"): RPQ_BOUNDED with
max_hops = k returns the pairs joined by a path of <= k edges whose word is
in L(rho).  Checked against O1's depth-bounded BFS (itself pinned against O2
walks of length <= k and a chain closed form in tests/test_oracle.py):
pairs, per-source counts and PE, for automata with and without initial-state
rows (a* vs a b* c), several batch widths, hub rows and k = 0 .. 6."""
import numpy as np
import pytest

import oracle
import synth
from conftest import sorted_pairs

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2602_20748_b200")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if R.rpq_device_count() == 0:
        pytest.skip("no CUDA device")


def _hub_graph(nv, ne, seed, hub_edges=1500):
    g = synth.random_graph(nv, ne, 3, seed=seed)
    rng = np.random.default_rng(seed)
    hub_edges = min(hub_edges, nv)
    hd = rng.choice(nv, hub_edges, replace=False).astype(np.uint32)
    return synth.Graph(nv, np.concatenate([g.src, np.full(hub_edges, 7, np.uint32)]),
                       np.concatenate([g.dst, hd]), np.concatenate([g.label, np.ones(hub_edges, np.uint16)]),
                       g.label_names).check()


@pytest.mark.parametrize("nv,ne,seed", [(300, 900, 1), (3000, 9000, 2)])
@pytest.mark.parametrize("rx", ["a*", "a b* c", "(a|b)*c*", "c+"])
def test_bounded_pairs_pe(nv, ne, seed, rx):
    g = _hub_graph(nv, ne, seed)
    G = R.rpq_graph_load(g)
    og = oracle.OracleGraph(g)
    a = R.rpq_compile(G, rx)
    for k in [0, 1, 2, 3, 6]:
        o = oracle.eval_sources(og, rx, None, max_hops=k)
        want = sorted_pairs(o["src"], o["dst"])
        for B in [0, 64, 200]:
            r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=B, max_hops=k)
            assert np.array_equal(r.rows(), want), (rx, k, B)
            assert r.stats()["product_edges"] == int(o["pe"].sum()), (rx, k, B)
        c = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_PE, max_hops=k)
        assert c.count == len(want) and c.stats()["product_edges"] == int(o["pe"].sum()), (rx, k)
        ps = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PER_SOURCE | R.RPQ_SOURCE_PE, batch_sources=128, max_hops=k)
        s, cnt = ps.source_counts()
        pe = ps.source_pe()
        got_c = np.zeros(nv, np.uint64)
        got_pe = np.zeros(nv, np.uint64)
        got_c[s] = cnt
        got_pe[s] = pe
        assert np.array_equal(got_c, o["counts"]) and np.array_equal(got_pe, o["pe"]), (rx, k)


def test_bounded_chain_and_large_bound():
    """Chain of 300: a* bounded by k reaches exactly i..i+k; a bound beyond
    the diameter equals the unbounded query."""
    g = synth.chain_graph(299)
    G = R.rpq_graph_load(g)
    a = R.rpq_compile(G, "a*")
    for k in [0, 1, 7, 150]:
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, max_hops=k)
        assert r.count == sum(min(i + k, 299) - i + 1 for i in range(300)), k
    full = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS).rows()
    big = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS, max_hops=10_000).rows()
    assert np.array_equal(full, big)


def test_bounded_single_source_and_targets():
    g = _hub_graph(2000, 7000, 5)
    G = R.rpq_graph_load(g, in_edges=True)
    og = oracle.OracleGraph(g)
    a = R.rpq_compile(G, "(a|b)*c")
    srcs = synth.sample_sources(2000, 40, seed=3)
    o = oracle.eval_sources(og, "(a|b)*c", srcs, max_hops=3)
    r = R.rpq_eval_sources(G, a, srcs, mode=R.RPQ_PAIRS, max_hops=3)
    assert np.array_equal(r.rows(), sorted_pairs(o["src"], o["dst"]))
    # backwards from targets: same bound (path lengths are direction-free)
    full = oracle.allpairs(g, "(a|b)*c", max_hops=3)
    tg = srcs[:10]
    m = np.isin(full["dst"], tg)
    want = np.stack([full["src"][m], full["dst"][m]], 1).astype(np.uint32)
    want = want[np.lexsort((want[:, 0], want[:, 1]))]
    got = R.rpq_eval_targets(G, a, tg, mode=R.RPQ_PAIRS, max_hops=3).rows()
    assert np.array_equal(got, want)
