"""WavePlan plan variants:

* loop-cache (A2): R(loop+) materialised once as a derived label L, then
  "prefix L? suffix" -- the same pairs as the direct plan (checked against
  O1 on the original regex), and derived labels behave like loaded ones;
* reverse (A1) is covered by tests/test_gpu_targets.py.
"""
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


@pytest.mark.parametrize("ie", [False, True])
@pytest.mark.parametrize("prefix,loop,suffix", [("a", "b c", "d"), ("", "b c", "d"), ("a", "b c", ""),
                                                ("a|b", "c d?", "a"), ("", "a b", "")])
def test_loop_cache_equals_direct(prefix, loop, suffix, ie):
    g = synth.random_graph(3000, 12000, 4, seed=7)
    G = R.rpq_graph_load(g, in_edges=ie)
    rx = " ".join(x for x in [f"({prefix})" if prefix else "", f"({loop})*", f"({suffix})" if suffix else ""] if x)
    o = oracle.allpairs(g, rx)
    want = sorted_pairs(o["src"], o["dst"])
    direct = R.rpq_eval_allpairs(G, R.rpq_compile(G, rx), mode=R.RPQ_PAIRS).rows()
    cached = R.rpq_eval_loop_cached(G, prefix, loop, suffix, mode=R.RPQ_PAIRS).rows()
    assert np.array_equal(direct, want) and np.array_equal(cached, want), rx
    # the automaton compiled before the label was added still evaluates
    assert R.rpq_eval_allpairs(G, R.rpq_compile(G, rx), mode=R.RPQ_COUNT).count == len(want)


def test_derived_label_matches_loaded():
    """A label added from host pairs evaluates exactly like the same edges
    loaded with the graph (CSR, dedup, in-edges)."""
    g = synth.random_graph(2000, 8000, 3, seed=3)
    G = R.rpq_graph_load(g, in_edges=True)
    rng = np.random.default_rng(1)
    s = rng.integers(0, 2000, 5000).astype(np.uint32)
    d = rng.integers(0, 2000, 5000).astype(np.uint32)
    lid = R.rpq_graph_add_label(G, "x", s, d)
    assert lid == 3
    g2 = synth.Graph(2000, np.concatenate([g.src, s]), np.concatenate([g.dst, d]),
                     np.concatenate([g.label, np.full(5000, 3, np.uint16)]), g.label_names + ["x"]).check()
    for rx in ["x+", "a x* b", "(x|c)* a"]:
        o = oracle.allpairs(g2, rx)
        got = R.rpq_eval_allpairs(G, R.rpq_compile(G, rx), mode=R.RPQ_PAIRS | R.RPQ_STATS)
        assert np.array_equal(got.rows(), sorted_pairs(o["src"], o["dst"])), rx
        assert got.stats()["product_edges"] == int(o["pe"].sum()), rx
        t = R.rpq_eval_targets(G, R.rpq_compile(G, rx), np.arange(0, 2000, 7, dtype=np.uint32), mode=R.RPQ_COUNT)
        m = np.isin(o["dst"], np.arange(0, 2000, 7))
        assert t.count == int(m.sum()), rx
    with pytest.raises(R.RPQError):
        R.rpq_graph_add_label(G, "x", s, d)            # duplicate name
    with pytest.raises(R.RPQError):
        R.rpq_graph_add_label(G, "y", np.array([5000], np.uint32), np.array([0], np.uint32))


@pytest.mark.parametrize("ie", [False, True])
@pytest.mark.parametrize("alpha,mid,beta", [("a*", "b", "c*"), ("(a|c)+", "d", "a b*"), ("a", "b", "c")])
def test_start_in_the_middle_equals_direct(alpha, mid, beta, ie):
    """WavePlan A3/A4: R(alpha mid beta) explored from the middle
    edges outwards, enumerated then deduplicated -- the same pairs as O1."""
    g = synth.random_graph(1500, 4500, 4, seed=11)
    G = R.rpq_graph_load(g, in_edges=ie)
    rx = f"({alpha}) ({mid}) ({beta})"
    o = oracle.allpairs(g, rx)
    got = R.rpq_eval_middle(G, alpha, mid, beta)
    assert np.array_equal(got.rows(), sorted_pairs(o["src"], o["dst"])), rx
    assert got.count == len(o["src"])


def test_crpq_projection():
    """crpq_eval_project: distinct projections of the CRPQ tuples, sorted."""
    g = synth.random_graph(300, 1200, 3, seed=2)
    G = R.rpq_graph_load(g, in_edges=True)
    atoms = [("x", "a", "y"), ("y", "b*", "z"), ("x", "c", "z")]
    full = R.crpq(G, ["x", "y", "z"], atoms).rows()
    for proj in (["x", "z"], ["z"], ["y", "x"]):
        idx = [["x", "y", "z"].index(v) for v in proj]
        want = np.unique(full[:, idx], axis=0) if len(full) else np.zeros((0, len(idx)), np.uint32)
        got = R.crpq(G, ["x", "y", "z"], atoms, project=proj).rows()
        assert np.array_equal(got, want), proj
        got_w = R.crpq(G, ["x", "y", "z"], atoms, project=proj, mode=R.RPQ_WCOJ).rows()
        assert np.array_equal(got_w, want), proj
