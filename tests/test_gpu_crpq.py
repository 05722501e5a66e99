"""GPU parity for crpq_eval (Definition 2) against the oracle."""
import numpy as np
import pytest

import oracle
import synth
from conftest import golden_int_tuples

pytestmark = pytest.mark.gpu
R = pytest.importorskip("paper_2602_20748_b200")


@pytest.fixture(scope="module", autouse=True)
def need_gpu():
    if R.rpq_device_count() == 0:
        pytest.skip("no CUDA device")


def rows(res):
    return [tuple(r) for r in res.rows().tolist()]


@pytest.mark.parametrize("ie", [False, True])
def test_q2_paper_tuples(toy, ie):
    """Q2 -> 4 tuples; with distinct(u2,u4) -> 2."""
    G = R.rpq_graph_load(toy, in_edges=ie)
    atoms = [("u3", "ab", "u2"), ("u3", "ab", "u4"), ("u2", "c*", "u4")]
    lab = {"u2": "D", "u3": "A", "u4": "D"}
    r = R.crpq(G, ["u2", "u3", "u4"], atoms, var_label=lab)
    assert rows(r) == golden_int_tuples("q2_tuples.txt")
    r = R.crpq(G, ["u2", "u3", "u4"], atoms, var_label=lab, distinct=[("u2", "u4")])
    assert rows(r) == [(10, 0, 12), (12, 0, 10)]


@pytest.mark.parametrize("ie", [False, True])
def test_constant_and_self_atom(toy, ie):
    G = R.rpq_graph_load(toy, in_edges=ie)
    # x -c+-> x on the toy graph: vertices on c-cycles
    r = R.crpq(G, ["x"], [("x", "c+", "x")])
    want = oracle.crpq_bruteforce(toy, oracle.CRPQ(["x"], [("x", "c+", "x")]))
    assert rows(r) == want
    # constant target (t = v12), free source
    q = oracle.CRPQ(["m", "t"], [("m", "ab", "t")], var_const={"t": 12})
    r = R.crpq(G, ["m", "t"], [("m", "ab", "t")], var_const={"t": 12})
    assert rows(r) == oracle.crpq_bruteforce(toy, q)


@pytest.mark.parametrize("ie", [False, True])
@pytest.mark.parametrize("seed", range(8))
def test_random_crpqs_vs_bruteforce(seed, ie):
    rng = np.random.default_rng(seed)
    g = synth.random_small(rng, max_v=7, max_e=16, num_labels=3, min_v=3)
    g.vertex_label = rng.integers(0, 2, g.num_vertices).astype(np.uint16)
    g.vertex_label_names = ["P", "Q"]
    G = R.rpq_graph_load(g, in_edges=ie)
    shapes = [
        (["x", "y", "z"], [("x", "a b*", "y"), ("y", "c*", "z"), ("x", "(a|c)+", "z")], {"x": "P"}, [("x", "z")]),
        (["x", "y", "z"], [("x", "a", "y"), ("x", "b*", "z")], {}, []),                          # star
        (["x", "y", "z", "w"], [("x", "a|b", "y"), ("y", "c", "z"), ("z", "(a|b)*", "w")], {"w": "Q"}, [("x", "w")]),
        (["x", "y"], [("y", "a+", "x")], {}, []),                                                # only y-side join later
        (["x", "y", "z"], [("y", "a", "x"), ("z", "b", "x")], {"z": "P"}, []),                   # x bound via y
    ]
    for vars_, atoms, lab, dist in shapes:
        q = oracle.CRPQ(vars_, atoms, var_label=lab, distinct=dist)
        want = oracle.crpq_bruteforce(g, q)
        got = rows(R.crpq(G, vars_, atoms, var_label=lab, distinct=dist))
        assert got == want, (seed, atoms)


def test_crpq_errors(toy):
    G = R.rpq_graph_load(toy)
    with pytest.raises(R.RPQError) as e:      # disconnected pattern (R18)
        R.crpq(G, ["a", "b", "c", "d"], [("a", "a", "b"), ("c", "b", "d")])
    assert e.value.status == R.RPQ_EUNSUPPORTED
    nfa = R.rpq_compile(G, "a")
    with pytest.raises(R.RPQError) as e:      # variable in no atom
        R.crpq_eval(G, [-1, -1, -1], [-1, -1, -1], [(0, nfa, 1)])
    assert e.value.status == R.RPQ_EUNSUPPORTED


@pytest.mark.parametrize("ie", [False, True])
def test_cfg4_ldbc_crpq_small(ie):
    """BASELINE cfg4 shape: m -hasTag-> t:Sports, m -hasCreator-> u,
    m -replyOf*-> p:Post.  Against the oracle's hash join of O1 relations and
    the closed form (one tuple per Sports-tagged message: one creator, one
    root post)."""
    g = synth.ldbc_graph(0.002)
    G = R.rpq_graph_load(g, in_edges=ie)
    sports = g.meta["sports"]
    vars_ = ["m", "t", "u", "p"]
    atoms = [("m", "hasTag", "t"), ("m", "hasCreator", "u"), ("m", "replyOf*", "p")]
    got = rows(R.crpq(G, vars_, atoms, var_label={"p": "Post"}, var_const={"t": sports}))
    q = oracle.CRPQ(vars_, atoms, var_label={"p": "Post"}, var_const={"t": sports})
    assert got == oracle.crpq_join(g, q)
    tagged = set(g.src[(g.label == g.label_names.index("hasTag")) & (g.dst == sports)].tolist())
    assert len(got) == len(tagged) and {t[0] for t in got} == tagged
