"""GPU parity of the direction-optimising (bottom-up) levels (SURVEY §8(f)
N1) against the oracle: RPQ_PULL=2 forces bottom-up dense levels on directed
graphs (in-edge CSR); the default (1) takes them for symmetric labels only.
PE (computed after the fact) must equal the oracle's own count."""
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


def sorted_rows(o):
    rows = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    return rows[np.lexsort((rows[:, 1], rows[:, 0]))]


@pytest.mark.parametrize("mode", ["2", "1"])
@pytest.mark.parametrize("nv,ne,seed", [(300, 1500, 1), (4000, 24000, 2)])
def test_pull_random_graphs(mode, nv, ne, seed, monkeypatch):
    monkeypatch.setenv("RPQ_PULL", mode)
    g = synth.random_graph(nv, ne, 3, seed=seed)
    G = R.rpq_graph_load(g, in_edges=True)
    for rx in ["(a|b)*c*", "a b* c", "c+", "a*", "(a|b|c)*", "((a|b)c)+"]:
        a = R.rpq_compile(G, rx)
        o = oracle.allpairs(g, rx)
        for B in (0, 2048):   # 2048: several batches, 32-word chunks
            r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=B)
            assert np.array_equal(r.rows(), sorted_rows(o)), (rx, B)
            st = r.stats()
            assert st["product_edges"] == int(o["pe"].sum()), (rx, B)
            if mode == "2" and st["batch_sources"] >= 2048 and st["levels"] > 1:
                assert st["pull_levels"] > 0, (rx, B)
        assert R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT).count == o["src"].size, rx


@pytest.mark.parametrize("mode", ["2", "1"])
def test_pull_ldbc_closed_forms(mode, monkeypatch):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    monkeypatch.setenv("RPQ_PULL", mode)
    g = synth.ldbc_graph(0.01)
    G = R.rpq_graph_load(g, in_edges=True)
    base, cnt = g.meta["base"], g.meta["count"]
    P = cnt["Person"]
    m = g.label == g.label_names.index("knows")
    A = sp.csr_matrix((np.ones(int(m.sum())), (g.src[m] - base["Person"], g.dst[m] - base["Person"])), shape=(P, P))
    _, comp = connected_components(A, directed=False)
    sizes = np.bincount(comp)
    per = np.where(sizes[comp] >= 2, sizes[comp], 0).astype(np.uint64)
    k = R.rpq_compile(G, "knows+")
    r = R.rpq_eval_allpairs(G, k, mode=R.RPQ_PER_SOURCE | R.RPQ_STATS)
    s, c = r.source_counts()
    got = np.zeros(g.num_vertices, np.uint64)
    got[s] = c
    want = np.zeros(g.num_vertices, np.uint64)
    want[base["Person"]:base["Person"] + P] = per
    assert np.array_equal(got, want)
    assert R.rpq_eval_allpairs(G, k, mode=R.RPQ_COUNT).count == int(per.sum())


def test_pull_reverse_targets(monkeypatch):
    """Bottom-up levels of a target-side evaluation use the forward CSR."""
    monkeypatch.setenv("RPQ_PULL", "2")
    g = synth.random_graph(3000, 15000, 3, seed=7)
    G = R.rpq_graph_load(g, in_edges=True)
    targets = np.arange(3000, dtype=np.uint32)
    for rx in ["(a|b)*c*", "a b* c"]:
        a = R.rpq_compile(G, rx)
        o = oracle.allpairs(g, rx)
        rows = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
        rows = rows[np.lexsort((rows[:, 0], rows[:, 1]))]
        r = R.rpq_eval_targets(G, a, targets, mode=R.RPQ_PAIRS)
        assert np.array_equal(r.rows(), rows), rx


@pytest.mark.parametrize("nv,npairs,seed", [(500, 3000, 3), (6000, 40000, 4)])
def test_pull_symmetric_default(nv, npairs, seed, monkeypatch):
    """Undirected (symmetric) labels: the default mode runs dense levels
    bottom-up, without the in-edge CSR (the CSR is its own transpose)."""
    monkeypatch.delenv("RPQ_PULL", raising=False)
    g = synth.symmetric_graph(nv, npairs, seed=seed)
    G = R.rpq_graph_load(g)
    lab = g.label_names[0]
    for rx in [f"{lab}+", f"{lab}*", f"{lab} {lab}"]:
        a = R.rpq_compile(G, rx)
        o = oracle.allpairs(g, rx)
        for B in (0, 2048):
            r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=B)
            assert np.array_equal(r.rows(), sorted_rows(o)), (rx, B)
            st = r.stats()
            assert st["product_edges"] == int(o["pe"].sum()), (rx, B)
        if rx.endswith("+") and nv >= 2048:   # 32-word chunks (>= 2048 sources per batch)
            assert R.rpq_eval_allpairs(G, a, mode=R.RPQ_STATS).stats()["pull_levels"] > 0


@pytest.mark.parametrize("pull", ["0", "2"])
def test_host_driven_level_loop(pull, monkeypatch):
    """RPQ_HOST_LOOP=1 (the fallback when the conditional CUDA graph cannot be
    built, and the mode ncu profiles) gives the same pairs and PE."""
    monkeypatch.setenv("RPQ_HOST_LOOP", "1")
    monkeypatch.setenv("RPQ_PULL", pull)
    g = synth.rmat_graph(14, seed=3)          # skewed degrees: rows > HUB_EDGES (742 edges)
    G = R.rpq_graph_load(g, in_edges=True)
    for rx in ["(a|b)*c*", "a b* c"]:
        a = R.rpq_compile(G, rx)
        o = oracle.allpairs(g, rx)
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=2048)
        assert np.array_equal(r.rows(), sorted_rows(o)), rx
        assert r.stats()["product_edges"] == int(o["pe"].sum()), rx
