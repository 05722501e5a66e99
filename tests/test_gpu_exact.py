"""Exact parity at BASELINE's bench sizes ("Exact result for
cfg2"; the cfg5 4,096-source rule), in the launch
configuration bench.py times (all-pairs, automatic batch width):

* cfg2: per-source result counts AND per-source product edges (PE, the
  numerator of the metric) of ALL 100,000 sources against O1, per query;
  the COUNT total and its fused PE (RPQ_PE) against O1's sums; the pair sets
  of 2,048 seeded sources sliced out of the device-resident all-pairs PAIRS
  result (bench.py's pairs_mode) against O1's.
* cfg5 (R-MAT scale 24): the first batch at bench width (B from rpq_plan),
  per-source counts and PE of seeded sources of that batch against O1; and
  1,024 seeded sources over all of V (rpq_eval_sources, chunks of 128):
  pair sets, counts and PE against O1.

Expected values come from oracle/ only.  Tolerance: none (integer sets)."""
import os

import numpy as np
import pytest

import oracle
import synth
from conftest import device_rows, sorted_pairs

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2602_20748_b200")
THREADS = os.cpu_count() or 1
CFG2_QUERIES = ["a*", "(a|b)*c", "a b* c"]


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if R.rpq_device_count() == 0:
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def cfg2():
    g = synth.uniform_graph()                   # bench.py default workload
    return g, R.rpq_graph_load(g), oracle.OracleGraph(g)


@pytest.mark.parametrize("rx", CFG2_QUERIES)
def test_cfg2_all_sources_counts_and_pe(cfg2, rx):
    g, G, og = cfg2
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PER_SOURCE | R.RPQ_SOURCE_PE)
    s, c = r.source_counts()
    pe = r.source_pe()
    got_c = np.zeros(g.num_vertices, np.uint64)
    got_pe = np.zeros(g.num_vertices, np.uint64)
    got_c[s] = c
    got_pe[s] = pe
    o = oracle.eval_sources(og, rx, None, pairs=False, threads=THREADS)
    assert np.array_equal(got_c, o["counts"]), rx
    assert np.array_equal(got_pe, o["pe"]), rx
    # the bench's COUNT call, PE fused into its count pass
    t = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_PE)
    assert t.count == int(o["counts"].sum())
    assert t.stats()["product_edges"] == int(o["pe"].sum())


@pytest.mark.parametrize("rx", CFG2_QUERIES)
def test_cfg2_pairs_of_2048_sources(cfg2, rx):
    g, G, og = cfg2
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS)          # 64-74 GB, device-resident
    s, c = r.source_counts()
    start = np.zeros(g.num_vertices + 1, np.uint64)
    cnt = np.zeros(g.num_vertices, np.uint64)
    cnt[s] = c
    start[1:] = np.cumsum(cnt)
    assert int(start[-1]) == r.count
    sample = synth.sample_sources(g.num_vertices, 2048, seed=2048)
    o = oracle.eval_sources(og, rx, sample, threads=THREADS)
    want = sorted_pairs(o["src"], o["dst"])
    got = np.concatenate([device_rows(r, int(start[v]), int(cnt[v])) for v in sample])
    assert np.array_equal(got, want), rx


@pytest.fixture(scope="module")
def rmat():
    g = synth.rmat_graph(24, seed=24)           # bench.py north_star / --workload cfg5
    return g, R.rpq_graph_load(g), oracle.OracleGraph(g)


def test_rmat24_first_batch_at_bench_width(rmat):
    g, G, og = rmat
    rx = "(a|b)*c*"
    a = R.rpq_compile(G, rx)
    pl = R.rpq_plan(G, a, mode=R.RPQ_COUNT)
    B, nb = pl["batch_sources"], pl["num_batches"]
    assert nb > 1 and B % 64 == 0
    # batch 0 exactly (shard 0 of nb shards), per-source counts + PE
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PER_SOURCE | R.RPQ_SOURCE_PE, batch_sources=B, shard_index=0,
                            shard_count=int(nb))
    lo, hi = r.batches()[0][:2]
    s, c = r.source_counts()
    pe = r.source_pe()
    assert s.size and int(s[0]) >= int(lo) and int(s[-1]) < int(hi)
    pick = synth.sample_sources(s.size, 192, seed=240)
    o = oracle.eval_sources(og, rx, s[pick].astype(np.uint32), pairs=False, threads=THREADS)
    assert np.array_equal(o["counts"], c[pick])
    assert np.array_equal(o["pe"], pe[pick])


def test_rmat24_1024_sources_pairs_counts_pe(rmat):
    g, G, og = rmat
    rx = "(a|b)*c*"
    a = R.rpq_compile(G, rx)
    sample = synth.sample_sources(g.num_vertices, 1024, seed=1024)
    for k in range(0, sample.size, 128):
        part = sample[k:k + 128]
        r = R.rpq_eval_sources(G, a, part, mode=R.RPQ_PAIRS | R.RPQ_PER_SOURCE | R.RPQ_SOURCE_PE)
        o = oracle.eval_sources(og, rx, part, threads=THREADS)
        s, c = r.source_counts()
        pe = r.source_pe()
        got_c = dict(zip(s.tolist(), c.tolist()))
        got_pe = dict(zip(s.tolist(), pe.tolist()))
        assert [got_c.get(v, 0) for v in part.tolist()] == o["counts"].tolist()
        assert [got_pe.get(v, 0) for v in part.tolist()] == o["pe"].tolist()
        # O1 emits each source's targets ascending, sources in the given
        # (ascending) order: already (src, dst)-sorted, no host sort needed
        want = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
        assert np.array_equal(r.rows(), want)


@pytest.mark.parametrize("rx", ["(a|b)*c*", "a b* c"])
def test_pairs_multi_tile_parts(rx):
    """All-pairs PAIRS where the extraction tasks span several 512-vertex
    tiles (40 K sources x 40 K vertices: 157 word groups x parts of 4 tiles),
    so per-source runs continue across tiles through the sector-aligned carry;
    (a|b)*c* has two final states (their rows are OR-ed).  Every source's
    count against O1, the pair lists of 512 seeded sources element by element,
    and the (src, dst) order across run boundaries."""
    g = synth.uniform_graph(40_000, 300_000, 3, seed=7)
    G = R.rpq_graph_load(g)
    og = oracle.OracleGraph(g)
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS)
    s, c = r.source_counts()
    cnt = np.zeros(g.num_vertices, np.uint64)
    cnt[s] = c
    o_all = oracle.eval_sources(og, rx, None, pairs=False, threads=THREADS)
    assert np.array_equal(cnt, o_all["counts"]), rx
    start = np.zeros(g.num_vertices + 1, np.uint64)
    start[1:] = np.cumsum(cnt)
    assert int(start[-1]) == r.count
    sample = synth.sample_sources(g.num_vertices, 512, seed=77)
    o = oracle.eval_sources(og, rx, sample, threads=THREADS)
    want = sorted_pairs(o["src"], o["dst"])
    got = np.concatenate([device_rows(r, int(start[v]), int(cnt[v])) for v in sample])
    assert np.array_equal(got, want), rx
    # source-major order across run boundaries: windows around sampled starts
    for v in sample[:64]:
        lo = max(0, int(start[v]) - 8)
        w = device_rows(r, lo, min(16, r.count - lo))
        key = w[:, 0].astype(np.uint64) << np.uint64(32) | w[:, 1].astype(np.uint64)
        assert bool(np.all(key[1:] > key[:-1])), (rx, v)
