"""GPU parity for the reverse direction: single-target /
target-set evaluation = the reversed automaton over the in-edge CSR.
Expected values: the oracle's all-pairs result (O1) filtered by target, and
the paper's Q1 footnote restricted to targets v2/v3."""
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


def oracle_by_target(g, rx, targets):
    o = oracle.allpairs(g, rx)
    rows = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    rows = rows[np.isin(rows[:, 1], np.asarray(targets, np.uint32))]
    return rows[np.lexsort((rows[:, 0], rows[:, 1]))]      # sorted by (t, x)


def test_toy_single_target():
    toy = synth.toy_graph()
    G = R.rpq_graph_load(toy, in_edges=True)
    a = R.rpq_compile(G, "abc*")
    # P:84 footnote 1: the pairs of abc* with target v2 and v3
    assert R.rpq_eval_single_target(G, a, 2, mode=R.RPQ_PAIRS).rows().tolist() == [[2, 2], [7, 2]]
    assert R.rpq_eval_single_target(G, a, 3, mode=R.RPQ_PAIRS).rows().tolist() == [[2, 3], [7, 3]]
    assert R.rpq_eval_single_target(G, a, 0, mode=R.RPQ_PAIRS).count == 0


@pytest.mark.parametrize("rx", ["abc*", "a*", "(a|b)*c", "(a|b)*c*", "c+", "ab*c", "a?b*"])
def test_toy_all_targets(rx):
    toy = synth.toy_graph()
    G = R.rpq_graph_load(toy, in_edges=True)
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_targets(G, a, list(range(toy.num_vertices)), mode=R.RPQ_PAIRS)
    assert np.array_equal(r.rows(), oracle_by_target(toy, rx, range(toy.num_vertices))), rx


@pytest.mark.parametrize("nv,ne,seed", [(300, 1200, 1), (5000, 20000, 2)])
def test_random_graph_targets(nv, ne, seed):
    g = synth.random_graph(nv, ne, 3, seed=seed)
    G = R.rpq_graph_load(g, in_edges=True)
    targets = synth.sample_sources(nv, 97, seed=seed + 10)
    for rx in ["(a|b)*c*", "a b* c", "c+", "a*"]:
        a = R.rpq_compile(G, rx)
        want = oracle_by_target(g, rx, targets)
        r = R.rpq_eval_targets(G, a, targets[::-1].copy(), mode=R.RPQ_PAIRS)
        assert np.array_equal(r.rows(), want), rx
        assert R.rpq_eval_targets(G, a, targets, mode=R.RPQ_COUNT).count == want.shape[0], rx
        t, c = R.rpq_eval_targets(G, a, targets, mode=R.RPQ_PER_SOURCE).source_counts()
        ut, uc = np.unique(want[:, 1], return_counts=True)
        assert np.array_equal(t, ut) and np.array_equal(c, uc.astype(np.uint64)), rx
        # small batches: several batches of targets, dense engine
        r2 = R.rpq_eval_targets(G, a, targets, mode=R.RPQ_PAIRS, batch_sources=64)
        assert np.array_equal(r2.rows(), want), rx


def test_targets_need_in_edges():
    toy = synth.toy_graph()
    G = R.rpq_graph_load(toy)
    with pytest.raises(R.RPQError) as e:
        R.rpq_eval_single_target(G, R.rpq_compile(G, "abc*"), 2)
    assert e.value.status == R.RPQ_EUNSUPPORTED
    G2 = R.rpq_graph_load(toy, in_edges=True)
    with pytest.raises(R.RPQError) as e:
        R.rpq_eval_single_target(G2, R.rpq_compile(G2, "abc*"), 14)
    assert e.value.status == R.RPQ_EINVAL
