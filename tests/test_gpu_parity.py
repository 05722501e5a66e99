"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle O1.

Integer set semantics: results must be bit-exact (sorted distinct pairs,
per-source counts, totals).  PE (product edges traversed on the minimal trim
DFA) must equal the oracle's own count.  Inputs are seeded synthetic graphs
(synth/), never produced by the CUDA path.
"""
import numpy as np
import pytest

import oracle
import synth
from conftest import golden_int_tuples

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2602_20748_b200")

SHAPES = ["abc*", "ab", "ab*c", "a*", "c*", "c+", "(a|b)*c", "(a|b)*c*", "a?b*", "abcc",
          "(a|b)b*", "a*b*", "ab*c*", "(a|b|c)*", "(ab)*", "a(b|c)?", "((a|b)c)+"]


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if R.rpq_device_count() == 0:
        pytest.skip("no CUDA device")


def oracle_rows(g, rx, sources=None):
    og = oracle.OracleGraph(g)
    r = oracle.eval_sources(og, rx, sources)
    rows = np.stack([r["src"], r["dst"]], axis=1).astype(np.uint32) if r["src"].size else np.zeros((0, 2), np.uint32)
    order = np.lexsort((rows[:, 1], rows[:, 0])) if rows.size else np.zeros(0, np.int64)
    return rows[order], r


def gpu_eval(G, rx, mode, **kw):
    a = R.rpq_compile(G, rx)
    return R.rpq_eval_allpairs(G, a, mode=mode, **kw)


def assert_pairs_equal(got, want, ctx=""):
    assert got.shape == want.shape, (ctx, got.shape, want.shape)
    assert np.array_equal(got, want), ctx


def test_toy_abcstar_13_pairs(toy):
    """P:84 footnote 1."""
    G = R.rpq_graph_load(toy)
    r = gpu_eval(G, "abc*", R.RPQ_PAIRS | R.RPQ_STATS)
    rows = [tuple(x) for x in r.rows().tolist()]
    assert rows == golden_int_tuples("q1_abcstar_pairs.txt")
    assert r.count == 13
    assert r.stats()["product_edges"] == 22


def test_toy_all_shapes(toy):
    G = R.rpq_graph_load(toy)
    for rx in SHAPES:
        want, o = oracle_rows(toy, rx)
        r = gpu_eval(G, rx, R.RPQ_PAIRS | R.RPQ_STATS)
        assert_pairs_equal(r.rows(), want, rx)
        assert r.stats()["product_edges"] == int(o["pe"].sum()), rx
        c = gpu_eval(G, rx, R.RPQ_COUNT)
        assert c.count == want.shape[0], rx


def test_single_source_v7(toy):
    G = R.rpq_graph_load(toy)
    a = R.rpq_compile(G, "abc*")
    r = R.rpq_eval_single_source(G, a, 7, mode=R.RPQ_PAIRS)
    assert [tuple(x) for x in r.rows().tolist()] == [(7, 2), (7, 3)]
    r = R.rpq_eval_single_source(G, a, 5, mode=R.RPQ_PAIRS)     # non-productive
    assert r.count == 0
    a2 = R.rpq_compile(G, "a*")
    r = R.rpq_eval_single_source(G, a2, 5, mode=R.RPQ_PAIRS)    # epsilon only (R1)
    assert [tuple(x) for x in r.rows().tolist()] == [(5, 5)]


@pytest.mark.parametrize("nv,ne,seed", [(300, 1200, 1), (3000, 12000, 2), (20000, 60000, 3)])
def test_random_graphs_pairs_counts_pe(nv, ne, seed):
    g = synth.random_graph(nv, ne, 4, seed=seed)
    G = R.rpq_graph_load(g)
    for rx in ["a*", "(a|b)*c", "a b* c", "abc*", "(a|b)*c*", "c+", "a?b*", "((a|b)c)+"]:
        want, o = oracle_rows(g, rx)
        r = gpu_eval(G, rx, R.RPQ_PAIRS | R.RPQ_PER_SOURCE | R.RPQ_STATS)
        assert_pairs_equal(r.rows(), want, rx)
        s, c = r.source_counts()
        nz = o["counts"] > 0
        assert np.array_equal(s, o["sources"][nz]) and np.array_equal(c, o["counts"][nz]), rx
        assert r.stats()["product_edges"] == int(o["pe"].sum()), rx
        assert gpu_eval(G, rx, R.RPQ_COUNT).count == want.shape[0], rx


@pytest.mark.parametrize("B,cw", [(64, 1), (64, 0), (128, 2), (200, 4), (1000, 8), (2048, 16), (4096, 32), (0, 0),
                                  (0, 1)])
def test_batch_and_chunk_invariance(B, cw):
    """Batch width B and chunk width must not change the result."""
    g = synth.random_graph(5000, 20000, 3, seed=7)
    G = R.rpq_graph_load(g)
    for rx in ["(a|b)*c*", "ab*c"]:
        want, o = oracle_rows(g, rx)
        r = gpu_eval(G, rx, R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=B, chunk_words=cw)
        assert_pairs_equal(r.rows(), want, (rx, B, cw))
        assert r.stats()["product_edges"] == int(o["pe"].sum())
        assert gpu_eval(G, rx, R.RPQ_COUNT, batch_sources=B, chunk_words=cw).count == want.shape[0]


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_shard_union_equals_whole(shards):
    """Fake multi-GPU on one device: shards are a pure function of (index,
    count); their disjoint union is the 1-shard result."""
    g = synth.random_graph(4000, 16000, 3, seed=8)
    G = R.rpq_graph_load(g)
    want, _ = oracle_rows(g, "(a|b)*c*")
    parts, total = [], 0
    for i in range(shards):
        r = gpu_eval(G, "(a|b)*c*", R.RPQ_PAIRS, batch_sources=256, shard_index=i, shard_count=shards)
        parts.append(r.rows())
        total += gpu_eval(G, "(a|b)*c*", R.RPQ_COUNT, batch_sources=256, shard_index=i, shard_count=shards).count
    got = np.concatenate(parts)
    got = got[np.lexsort((got[:, 1], got[:, 0]))]
    assert_pairs_equal(got, want)
    assert total == want.shape[0]


def test_eval_sources_and_single_source():
    """single-source(s) = all-pairs filtered to s."""
    g = synth.random_graph(3000, 15000, 3, seed=9)
    G = R.rpq_graph_load(g)
    a = R.rpq_compile(G, "(a|b)*c*")
    want, _ = oracle_rows(g, "(a|b)*c*")
    rng = np.random.default_rng(0)
    srcs = rng.choice(3000, 100, replace=False).astype(np.uint32)
    r = R.rpq_eval_sources(G, a, srcs, mode=R.RPQ_PAIRS)
    keep = np.isin(want[:, 0], srcs)
    assert_pairs_equal(r.rows(), want[keep])
    for s in srcs[:5]:
        r1 = R.rpq_eval_single_source(G, a, int(s), mode=R.RPQ_PAIRS)
        assert_pairs_equal(r1.rows(), want[want[:, 0] == s])
    with pytest.raises(R.RPQError):
        R.rpq_eval_sources(G, a, np.array([1, 1], np.uint32))
    with pytest.raises(R.RPQError):
        R.rpq_eval_single_source(G, a, 3000)
    r0 = R.rpq_eval_sources(G, a, np.zeros(0, np.uint32), mode=R.RPQ_PAIRS)
    assert r0.count == 0


def test_relabel_invariance():
    g = synth.random_graph(2000, 9000, 3, seed=10)
    perm = np.random.default_rng(1).permutation(2000).astype(np.uint32)
    g2 = synth.relabel(g, perm)
    a = gpu_eval(R.rpq_graph_load(g), "a b* c", R.RPQ_PAIRS).rows()
    b = gpu_eval(R.rpq_graph_load(g2), "a b* c", R.RPQ_PAIRS).rows()
    mapped = np.stack([perm[a[:, 0]], perm[a[:, 1]]], axis=1)
    mapped = mapped[np.lexsort((mapped[:, 1], mapped[:, 0]))]
    assert_pairs_equal(b, mapped)


def test_chain_hop_coverage():
    """No hop limit (tab:max_hop lesson)."""
    for L in [64, 300]:
        g = synth.chain_graph(L)
        G = R.rpq_graph_load(g)
        n = L + 1
        assert gpu_eval(G, "a*", R.RPQ_COUNT).count == n * (n + 1) // 2
        assert gpu_eval(G, "a+", R.RPQ_COUNT).count == n * (n - 1) // 2
        assert gpu_eval(G, "a+", R.RPQ_COUNT, batch_sources=64).count == n * (n - 1) // 2


def test_hub_vertices_split():
    """Rows longer than the hub segment are split across warps; results
    must not change (degree-skewed RMAT-like hubs)."""
    rng = np.random.default_rng(5)
    nv = 20000
    hub_src = np.zeros(6000, np.uint32)
    hub_dst = rng.integers(0, nv, 6000).astype(np.uint32)
    src = np.concatenate([hub_src, rng.integers(0, nv, 30000).astype(np.uint32), np.arange(1, 50, dtype=np.uint32)])
    dst = np.concatenate([hub_dst, rng.integers(0, nv, 30000).astype(np.uint32), np.zeros(49, np.uint32)])
    lab = rng.integers(0, 2, src.size).astype(np.uint16)
    g = synth.Graph(nv, src, dst, lab, ["a", "b"]).check()
    G = R.rpq_graph_load(g)
    for rx in ["(a|b)*", "a b*", "(ab)+"]:
        want, o = oracle_rows(g, rx)
        for B, cw in [(0, 0), (64, 1), (512, 8)]:
            r = gpu_eval(G, rx, R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=B, chunk_words=cw)
            assert_pairs_equal(r.rows(), want, (rx, B, cw))
            assert r.stats()["product_edges"] == int(o["pe"].sum())


def test_degenerate_cases():
    # no edges carry the query's labels; epsilon-only results (R1)
    g = synth.Graph(10, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32), np.array([0, 0], np.uint16),
                    ["a", "b"]).check()
    G = R.rpq_graph_load(g)
    assert gpu_eval(G, "b", R.RPQ_COUNT).count == 0
    assert gpu_eval(G, "b*", R.RPQ_COUNT).count == 10
    r = gpu_eval(G, "b*", R.RPQ_PAIRS)
    assert [tuple(x) for x in r.rows().tolist()] == [(v, v) for v in range(10)]
    r = gpu_eval(G, "a*", R.RPQ_PAIRS | R.RPQ_PER_SOURCE)
    want, _ = oracle_rows(g, "a*")
    assert_pairs_equal(r.rows(), want)
    # graph with a single vertex and a self-loop (R5)
    g1 = synth.Graph(1, np.array([0], np.uint32), np.array([0], np.uint32), np.array([0], np.uint16), ["a"]).check()
    G1 = R.rpq_graph_load(g1)
    assert gpu_eval(G1, "a+", R.RPQ_COUNT).count == 1
    # duplicate edges collapse (R4)
    g2 = synth.Graph(3, np.array([0, 0, 0], np.uint32), np.array([1, 1, 2], np.uint32), np.zeros(3, np.uint16),
                     ["a"]).check()
    G2 = R.rpq_graph_load(g2)
    assert R.rpq_graph_info(G2)["num_edges"] == 2
    with pytest.raises(R.RPQError):
        R.rpq_graph_load(synth.Graph(2, np.array([0], np.uint32), np.array([5], np.uint32), np.zeros(1, np.uint16),
                                     ["a"]))


def test_cfg2_full_size_sampled():
    """BASELINE cfg2 (100K vertices, 1M distinct edges, 4 labels) in the
    bench launch configuration: full all-pairs per-source counts on the GPU,
    checked exactly against the oracle on a seeded sample of sources; exact
    pair sets on a smaller sample; total == sum of per-source counts."""
    g = synth.uniform_graph()
    G = R.rpq_graph_load(g)
    og = oracle.OracleGraph(g)
    sample = synth.sample_sources(g.num_vertices, 256, seed=123)
    for rx in ["a*", "(a|b)*c", "a b* c"]:
        a = R.rpq_compile(G, rx)
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PER_SOURCE | R.RPQ_STATS)
        s, c = r.source_counts()
        full = np.zeros(g.num_vertices, np.uint64)
        full[s] = c
        o = oracle.eval_sources(og, rx, sample, pairs=False)
        assert np.array_equal(full[sample], o["counts"]), rx
        tot = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT)
        assert tot.count == int(c.sum()), rx
        small = sample[:16]
        rp = R.rpq_eval_sources(G, a, small, mode=R.RPQ_PAIRS)
        op = oracle.eval_sources(og, rx, small)
        want = np.stack([op["src"], op["dst"]], 1).astype(np.uint32)
        want = want[np.lexsort((want[:, 1], want[:, 0]))]
        assert_pairs_equal(rp.rows(), want, rx)


def _reply_depths(g):
    base, cnt = g.meta["base"], g.meta["count"]
    parent = g.meta["reply_parent"]
    C = cnt["Comment"]
    depth = np.zeros(C, np.int64)
    pc = parent - base["Comment"]
    is_c = (parent >= base["Comment"]) & (parent < base["Comment"] + C)
    for i in range(C):
        depth[i] = 1 + (depth[pc[i]] if is_c[i] else 0)
    return depth


@pytest.mark.parametrize("B", [0, 1024, 4096])
def test_ldbc_closed_forms(B):
    """cfg3 shapes: replyOf* on the reply forest = |V| + sum of comment depths
    (per source: its ancestor chain + itself); knows+ on symmetric knows =
    component size per person (SURVEY §8(c) closed forms).  Small batches
    exercise the touched-set clearing / sparse counting paths."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    g = synth.ldbc_graph(0.002)
    G = R.rpq_graph_load(g)
    base, cnt = g.meta["base"], g.meta["count"]
    depth = _reply_depths(g)
    a = R.rpq_compile(G, "replyOf*")
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, batch_sources=B)
    assert r.count == g.num_vertices + int(depth.sum())
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PER_SOURCE, batch_sources=B)
    s, c = r.source_counts()
    full = np.ones(g.num_vertices, np.uint64)            # epsilon pair of every vertex (R1)
    full[base["Comment"]:base["Comment"] + cnt["Comment"]] += depth.astype(np.uint64)
    assert np.array_equal(s, np.arange(g.num_vertices)) and np.array_equal(c, full)
    P = cnt["Person"]
    m = g.label == 0
    A = sp.csr_matrix((np.ones(int(m.sum())), (g.src[m] - base["Person"], g.dst[m] - base["Person"])), shape=(P, P))
    _, comp = connected_components(A, directed=False)
    sizes = np.bincount(comp)
    per = np.where(sizes[comp] >= 2, sizes[comp], 0).astype(np.uint64)
    k = R.rpq_compile(G, "knows+")
    r = R.rpq_eval_allpairs(G, k, mode=R.RPQ_PER_SOURCE, batch_sources=min(B, 256) if B else 0)
    s, c = r.source_counts()
    want = np.zeros(g.num_vertices, np.uint64)
    want[base["Person"]:base["Person"] + P] = per
    got = np.zeros(g.num_vertices, np.uint64)
    got[s] = c
    assert np.array_equal(got, want)
    assert R.rpq_eval_allpairs(G, k, mode=R.RPQ_COUNT, batch_sources=B).count == int(per.sum())


@pytest.mark.parametrize("engine", ["sparse", "dense"])
def test_engines_agree(engine, monkeypatch):
    """The sparse (warp per source, shared-memory visited set) and dense
    (bit-parallel) engines give identical counts, per-source counts and PE;
    forcing the sparse engine on a dense query exercises the overflow
    fallback to the dense engine."""
    monkeypatch.setenv("RPQ_ENGINE", engine)
    g = synth.random_graph(3000, 9000, 3, seed=21)
    G = R.rpq_graph_load(g)
    for rx in ["a b* c", "(a|b)*c*", "abc", "c?a"]:
        want, o = oracle_rows(g, rx)
        r = gpu_eval(G, rx, R.RPQ_PER_SOURCE | R.RPQ_STATS)
        s, c = r.source_counts()
        nz = o["counts"] > 0
        assert np.array_equal(s, o["sources"][nz]) and np.array_equal(c, o["counts"][nz]), (engine, rx)
        assert r.stats()["product_edges"] == int(o["pe"].sum()), (engine, rx)
        assert_pairs_equal(gpu_eval(G, rx, R.RPQ_PAIRS).rows(), want, (engine, rx))
        parts = [gpu_eval(G, rx, R.RPQ_PAIRS, batch_sources=700, shard_index=i, shard_count=2).rows()
                 for i in range(2)]
        got = np.concatenate(parts)
        got = got[np.lexsort((got[:, 1], got[:, 0]))]
        assert_pairs_equal(got, want, (engine, rx, "sharded"))
        for sc in [1, 3]:
            tot = sum(gpu_eval(G, rx, R.RPQ_COUNT, batch_sources=512, shard_index=i, shard_count=sc).count
                      for i in range(sc))
            assert tot == want.shape[0], (engine, rx, sc)
    # LDBC replyOf* (sparse reach) and knows+ (dense reach) under auto choice
    monkeypatch.delenv("RPQ_ENGINE")
    lg = synth.ldbc_graph(0.002)
    LG = R.rpq_graph_load(lg)
    depth = _reply_depths(lg)
    r = gpu_eval(LG, "replyOf*", R.RPQ_COUNT | R.RPQ_STATS)
    assert r.count == lg.num_vertices + int(depth.sum())


def test_sparse_batches_dense_engine(monkeypatch):
    """Many small batches with small reach take the touched-set clear/count
    path of the dense engine; automata whose final state has no outgoing
    transition must still count every result bit (they fall back to dense
    clearing/counting)."""
    monkeypatch.setenv("RPQ_ENGINE", "dense")
    g = synth.random_graph(40000, 24000, 3, seed=22)
    G = R.rpq_graph_load(g)
    for rx in ["ab*c", "c?a", "abc", "(a|b)*c*", "a+", "b"]:
        want, _ = oracle_rows(g, rx)
        for B in [64, 256]:
            assert gpu_eval(G, rx, R.RPQ_COUNT, batch_sources=B).count == want.shape[0], (rx, B)
        r = gpu_eval(G, rx, R.RPQ_PAIRS, batch_sources=128)
        assert_pairs_equal(r.rows(), want, rx)


@pytest.mark.parametrize("tma", ["1", "2", "3"])
@pytest.mark.parametrize("B", [0, 4096])
def test_tma_bulk_copy_expand(B, tma, monkeypatch):
    """RPQ_TMA (bit 0: k_level, bit 1: k_level_hub): the target-row segments
    of multi-chunk groups arrive by cp.async.bulk into a per-warp shared-memory
    ring (mbarrier completion); pairs and PE must equal the oracle's
    (multi-chunk rows: B = 0 puts all 20 K sources in one batch, 10 chunks
    per row; vertices 0 and 7 have 1,500 / 900 out-edges, so their rows are
    split into HUB_EDGES segments for the hub kernel)."""
    monkeypatch.setenv("RPQ_TMA", tma)
    monkeypatch.setenv("RPQ_ENGINE", "dense")
    rng = np.random.default_rng(12)
    g = synth.random_graph(20000, 70000, 3, seed=12)
    hs = np.concatenate([np.zeros(1500, np.uint32), np.full(900, 7, np.uint32)])
    hd = rng.integers(0, 20000, hs.size).astype(np.uint32)
    hl = np.concatenate([np.zeros(1500, np.uint16), np.ones(900, np.uint16)])
    g = synth.Graph(20000, np.concatenate([g.src, hs]), np.concatenate([g.dst, hd]), np.concatenate([g.label, hl]),
                    g.label_names).check()
    G = R.rpq_graph_load(g)
    for rx in ["a*", "(a|b)*c", "a b* c"]:
        want, o = oracle_rows(g, rx)
        r = gpu_eval(G, rx, R.RPQ_PAIRS | R.RPQ_STATS, batch_sources=B)
        assert_pairs_equal(r.rows(), want, (rx, B, tma))
        assert r.stats()["product_edges"] == int(o["pe"].sum()), (rx, tma)


def test_sparse_write_pass_redo(monkeypatch):
    """If the sparse engine's PAIRS write pass overflows where its counting
    pass fitted, the whole query is re-run on the dense engine.  The hook
    RPQ_TEST_SPARSE_REDO forces that path: pairs and PE must still equal the
    oracle's (sparse-reach and dense-reach queries)."""
    monkeypatch.setenv("RPQ_ENGINE", "sparse")
    monkeypatch.setenv("RPQ_TEST_SPARSE_REDO", "1")
    g = synth.random_graph(3000, 6000, 3, seed=31)
    G = R.rpq_graph_load(g)
    for rx in ["a b c", "c?a", "(a|b)*c*"]:
        want, o = oracle_rows(g, rx)
        r = gpu_eval(G, rx, R.RPQ_PAIRS | R.RPQ_STATS)
        assert_pairs_equal(r.rows(), want, rx)
        assert r.stats()["product_edges"] == int(o["pe"].sum()), rx


def test_edgeless_graph_and_empty_vertex_set():
    """|E| = 0: every query returns exactly its epsilon pairs (R1), and
    nothing else; |V| = 0 is rejected with EINVAL."""
    g = synth.Graph(1000, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint16), ["a", "b"]).check()
    G = R.rpq_graph_load(g)
    for rx, n in [("a*", 1000), ("a+", 0), ("(a|b)*b?", 1000), ("ab", 0)]:
        assert gpu_eval(G, rx, R.RPQ_COUNT).count == n, rx
        r = gpu_eval(G, rx, R.RPQ_PAIRS)
        assert r.count == n and (n == 0 or np.array_equal(r.rows(), np.stack([np.arange(n)] * 2, 1))), rx
    with pytest.raises(R.RPQError):
        R.rpq_graph_load(synth.Graph(0, np.zeros(0, np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint16),
                                     ["a"]))


def test_many_state_automata_multi_chunk():
    """Automata with 6-9 minimal-DFA states over 10 chunks per row (all 20 K
    sources in one batch): pairs and PE equal O1's."""
    g = synth.random_graph(20000, 60000, 4, seed=41)
    G = R.rpq_graph_load(g)
    for rx in ["a b c d a", "(a|b)(b|c)(c|d)d*a", "a(b a)*c(d|a)+", "((a b)|(c d))+ a?"]:
        a = R.rpq_compile(G, rx)
        want, o = oracle_rows(g, rx)
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS | R.RPQ_STATS)
        assert_pairs_equal(r.rows(), want, rx)
        assert r.stats()["product_edges"] == int(o["pe"].sum()), rx
