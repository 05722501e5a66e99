"""Worst-case-optimal CRPQ joins ("the WCOJ-based CQ
method"; cyclic CQ shapes with distinct filters).  crpq_eval
with RPQ_WCOJ binds one variable at a time and intersects the sorted value
lists of every atom into it.  The CQ1-CQ5 drawings are image-only, so the
shapes here are the cyclic / acyclic families they are built from (LSQB
triangles, 4-cycles, diamonds with a distinct filter, stars, paths, self
atoms, constants).  Expected tuples: the brute-force CRPQ oracle (every
assignment checked against O1 atom relations) on small graphs, the
hash-join oracle on larger ones; also equal to the binary-join plan."""
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


def rows(res):
    return [tuple(r) for r in res.rows().tolist()]


SHAPES = [
    # triangle (cyclic), a closure edge
    (["x", "y", "z"], [("x", "a", "y"), ("y", "b", "z"), ("z", "c*", "x")], {}, []),
    # triangle with a distinct filter and a label
    (["x", "y", "z"], [("x", "a|b", "y"), ("y", "(a|c)+", "z"), ("x", "c", "z")], {"x": "P"}, [("x", "z")]),
    # 4-cycle
    (["w", "x", "y", "z"], [("w", "a", "x"), ("x", "b*", "y"), ("y", "a", "z"), ("z", "c", "w")], {}, [("w", "y")]),
    # diamond (two paths x -> w) with a distinct filter on the middle vertices (CQ4/CQ5-style)
    (["x", "y", "z", "w"], [("x", "a", "y"), ("x", "b", "z"), ("y", "c*", "w"), ("z", "c*", "w")], {"w": "Q"},
     [("y", "z")]),
    # star and path (acyclic)
    (["x", "y", "z"], [("x", "a", "y"), ("x", "b*", "z")], {}, []),
    (["x", "y", "z", "w"], [("x", "a|b", "y"), ("y", "c", "z"), ("z", "(a|b)*", "w")], {"w": "Q"}, [("x", "w")]),
    # self atom + edge into it
    (["x", "y"], [("x", "c+", "x"), ("y", "a", "x")], {}, []),
]


@pytest.mark.parametrize("ie", [False, True])
@pytest.mark.parametrize("seed", range(6))
def test_wcoj_vs_bruteforce(seed, ie):
    rng = np.random.default_rng(100 + seed)
    g = synth.random_small(rng, max_v=8, max_e=20, num_labels=3, min_v=3)
    g.vertex_label = rng.integers(0, 2, g.num_vertices).astype(np.uint16)
    g.vertex_label_names = ["P", "Q"]
    G = R.rpq_graph_load(g, in_edges=ie)
    for vars_, atoms, lab, dist in SHAPES:
        want = oracle.crpq_bruteforce(g, oracle.CRPQ(vars_, atoms, var_label=lab, distinct=dist))
        got = rows(R.crpq(G, vars_, atoms, var_label=lab, distinct=dist, mode=R.RPQ_WCOJ))
        assert got == want, (seed, vars_, atoms)


@pytest.mark.parametrize("seed", range(3))
def test_wcoj_vs_hash_join_larger(seed):
    g = synth.random_graph(400, 1600, 3, seed=seed)
    rng = np.random.default_rng(seed)
    g.vertex_label = rng.integers(0, 2, g.num_vertices).astype(np.uint16)
    g.vertex_label_names = ["P", "Q"]
    G = R.rpq_graph_load(g, in_edges=True)
    og = oracle.OracleGraph(g)
    for vars_, atoms, lab, dist in SHAPES:
        q = oracle.CRPQ(vars_, atoms, var_label=lab, distinct=dist)
        # the hash-join oracle needs each atom to share a variable with earlier ones
        want = oracle.crpq_join(g, q, og)
        got_w = rows(R.crpq(G, vars_, atoms, var_label=lab, distinct=dist, mode=R.RPQ_WCOJ))
        got_b = rows(R.crpq(G, vars_, atoms, var_label=lab, distinct=dist))
        assert got_w == want and got_b == want, (seed, vars_, atoms)


def test_wcoj_paper_q2(toy):
    """Q2 -> 4 tuples; distinct(u2, u4) -> 2 (also through WCOJ)."""
    G = R.rpq_graph_load(toy, in_edges=True)
    atoms = [("u3", "ab", "u2"), ("u3", "ab", "u4"), ("u2", "c*", "u4")]
    lab = {"u2": "D", "u3": "A", "u4": "D"}
    r = R.crpq(G, ["u2", "u3", "u4"], atoms, var_label=lab, mode=R.RPQ_WCOJ)
    assert rows(r) == [(10, 0, 10), (10, 0, 12), (12, 0, 10), (12, 0, 12)]
    r = R.crpq(G, ["u2", "u3", "u4"], atoms, var_label=lab, distinct=[("u2", "u4")], mode=R.RPQ_WCOJ)
    assert rows(r) == [(10, 0, 12), (12, 0, 10)]
