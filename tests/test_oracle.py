"""Pins for the CPU oracle (O1), independent of the oracle itself.

Each test pins O1 to something other than its own code: values the paper
prints (tests/golden/, each with its PAPER.md citation), brute force over
walks (O2, Definition 1), relational algebra (O3), closed forms
(scipy connected components, forest depths) and the language of Python `re`.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth
from conftest import golden_int_tuples, read_golden

# tab:queries shapes and the BASELINE.json regexes
QUERY_SHAPES = ["a*", "a?b*", "ab*", "abcd" , "abc*", "ab*c", "(a|b)b*", "a*b*",
                "ab*c*", "(a|b|c)*", "(a|b)*c", "a b* c", "(a|b)*c*", "a+", "c+",
                "(ab)*", "a(b|c)?", "((a|b)c)+", "a**", "(a*)+", "a?+"]


def _edges(g):
    return set(zip(g.src.tolist(), g.label.tolist(), g.dst.tolist()))


def test_toy_graph_matches_tab_LGF(toy):
    names = toy.label_names
    want = {(int(s), names.index(l), int(d)) for (s, l, d) in read_golden("toy_graph_edges.txt")}
    assert _edges(toy) == want
    assert len(want) == 19                       # P:361-377 (not 15)


def test_q1_abcstar_13_pairs(toy):
    """Footnote 1 of P:84: Q1 = abc* returns exactly these 13 pairs."""
    r = oracle.allpairs(toy, "abc*")
    assert sorted(oracle.pair_set(r)) == golden_int_tuples("q1_abcstar_pairs.txt")
    r_nfa = oracle.allpairs(toy, "abc*", use_dfa=False)
    assert oracle.pair_set(r_nfa) == oracle.pair_set(r)


def test_relation_a(toy):
    """the relation for edge label a."""
    assert sorted(oracle.pair_set(oracle.allpairs(toy, "a"))) == golden_int_tuples("relation_a.txt")


def test_witness_paths(toy):
    """(v2,v2), (v0,v7), (v0,v11) are witnessed by ab, abc, abccc;
    P:400: (v0,v9) by the 4-hop word abcc (v0->v3->v12->v13->v9)."""
    assert (2, 2) in oracle.pair_set(oracle.allpairs(toy, "ab"))
    assert (0, 7) in oracle.pair_set(oracle.allpairs(toy, "abc"))
    assert (0, 11) in oracle.pair_set(oracle.allpairs(toy, "abccc"))
    assert (0, 9) in oracle.pair_set(oracle.allpairs(toy, "abcc"))
    assert (0, 9) not in oracle.pair_set(oracle.allpairs(toy, "abc"))


def test_single_source_v7(toy):
    og = oracle.OracleGraph(toy)
    r = oracle.eval_sources(og, "abc*", np.array([7], np.uint32))
    assert list(zip(r["src"].tolist(), r["dst"].tolist())) == [(7, 2), (7, 3)]


def test_q2_crpq_paper_tuples(toy):
    """Q2 on (u2,u3,u4) -> 4 tuples (pattern reading R8)."""
    q = oracle.CRPQ(["u2", "u3", "u4"],
                    [("u3", "ab", "u2"), ("u3", "ab", "u4"), ("u2", "c*", "u4")],
                    var_label={"u2": "D", "u3": "A", "u4": "D"})
    want = golden_int_tuples("q2_tuples.txt")
    assert oracle.crpq_bruteforce(toy, q) == want
    assert oracle.crpq_join(toy, q) == want
    qd = oracle.CRPQ(q.vars, q.atoms, q.var_label, distinct=[("u2", "u4")])
    assert oracle.crpq_bruteforce(toy, qd) == [(10, 0, 12), (12, 0, 10)]


def test_ab_atom_restricted(toy):
    """P'_0 = result of ab from A-labelled to D-labelled vertices."""
    q = oracle.CRPQ(["x", "y"], [("x", "ab", "y")], var_label={"x": "A", "y": "D"})
    assert oracle.crpq_bruteforce(toy, q) == golden_int_tuples("rpq_ab_atom.txt")


def test_paper_dfa_state_counts():
    """abc* has 3 states q0,q1,q2 with a c-loop on q2;
    abcd has |Q|=5.  Others: textbook minimal DFAs."""
    names = ["a", "b", "c", "d", "knows"]
    want = {"abc*": 3, "abcd": 5, "a*": 1, "knows+": 2, "(a|b)*c": 2, "(a|b)*c*": 2,
            "ab*c": 3, "a b* c": 3}
    for rx, n in want.items():
        assert oracle.Automaton(rx, names).info()["states"] == n, rx
    A = oracle.Automaton("abc*", names)
    assert sorted(A.dfa_transitions()) == [(0, 0, 1), (1, 1, 2), (2, 2, 2)]
    assert A.dfa_finals() == [2]


def test_paper_dialect_plus_is_alternation():
    """tab:queries writes alternation as infix + (P:1042-1043), reading R2."""
    g = synth.random_graph(40, 120, 3, seed=5)
    a = oracle.pair_set(oracle.allpairs(g, "(a+b)*c", paper_dialect=True))
    b = oracle.pair_set(oracle.allpairs(g, "(a|b)*c"))
    assert a == b


def test_syntax_errors():
    names = ["a", "b", "c"]
    for bad in ["", "()", "(a", "a|", "*a", "a)", "|a"]:
        with pytest.raises(oracle.OracleError) as e:
            oracle.Automaton(bad, names)
        assert e.value.status == oracle.OG_ESYNTAX, bad
    with pytest.raises(oracle.OracleError) as e:
        oracle.Automaton("ax", names)
    assert e.value.status == oracle.OG_ELABEL and e.value.offset == 1


@pytest.mark.parametrize("rx", QUERY_SHAPES)
def test_language_vs_python_re(rx):
    """Both automata accept exactly the words Python's re.fullmatch accepts,
    for every word of length <= 6 over 4 labels (SPEC S:100 idea)."""
    import re
    names = ["a", "b", "c", "d"]
    if "**" in rx or "*)+" in rx or "?+" in rx:
        pytest.skip("stacked postfix operators: Python re disagrees syntactically")
    pat = re.compile(oracle.to_python_re(rx, names))
    A = oracle.Automaton(rx, names)
    for n in range(0, 7):
        for w in itertools.product(range(4), repeat=n):
            want = bool(pat.fullmatch("".join(chr(0xE000 + x) for x in w)))
            assert A.accepts(w, dfa=True) == want, (rx, w)
            assert A.accepts(w, dfa=False) == want, (rx, w)


def test_stacked_postfix_idempotent():
    """Reading R19: a** = a*, (a*)+ = a*, a?+ = a*."""
    g = synth.random_graph(30, 90, 3, seed=9)
    base = oracle.pair_set(oracle.allpairs(g, "a*"))
    for rx in ["a**", "(a*)+", "(a?)+", "(a+)*"]:
        assert oracle.pair_set(oracle.allpairs(g, rx)) == base, rx


def test_brute_force_definition1():
    """O1 (both automata) == O2 (walk enumeration + Python re) on tiny random
    graphs, every tab:queries shape."""
    rng = np.random.default_rng(1234)
    shapes = [s for s in QUERY_SHAPES if not ("**" in s or "*)+" in s or "?+" in s)]
    n = 0
    for trial in range(14):
        g = synth.random_small(rng, max_v=5, max_e=7, num_labels=4)
        for rx in shapes:
            try:
                want = oracle.brute_force(g, rx)
            except oracle.OracleError:
                continue
            assert oracle.pair_set(oracle.allpairs(g, rx)) == want, (rx, trial)
            assert oracle.pair_set(oracle.allpairs(g, rx, use_dfa=False)) == want, (rx, trial)
            n += 1
    assert n > 200


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_algebra_alpha_operator(seed):
    """O1 == O3 (relational algebra with the alpha-operator) on
    random graphs with a few hundred vertices."""
    g = synth.random_graph(200 + 50 * seed, 500 + 100 * seed, 4, seed=seed)
    for rx in QUERY_SHAPES:
        assert oracle.pair_set(oracle.allpairs(g, rx)) == oracle.algebra(g, rx), rx


def test_union_concat_star_invariants():
    """Definition 1 gives R(r1|r2) = R(r1) u R(r2), R(r1 r2) = R(r1) o R(r2),
    R(r*) = R(r+) u Id_V (reading R1), R(r?) = R(r) u Id_V."""
    g = synth.random_graph(120, 400, 3, seed=77)
    R = lambda rx: oracle.pair_set(oracle.allpairs(g, rx))
    ident = {(v, v) for v in range(g.num_vertices)}

    def compose(A, B):
        by = {}
        for x, y in B:
            by.setdefault(x, set()).add(y)
        return {(x, z) for x, y in A for z in by.get(y, ())}
    for r1, r2 in [("a", "b"), ("ab*", "c"), ("(a|b)*", "c+")]:
        assert R(f"({r1})|({r2})") == R(r1) | R(r2)
        assert R(f"({r1})({r2})") == compose(R(r1), R(r2))
        assert R(r1) <= R(f"({r1})|({r2})")             # monotone under union
    for r in ["a", "ab", "a|bc"]:
        assert R(f"({r})*") == R(f"({r})+") | ident
        assert R(f"({r})?") == R(r) | ident
        assert ident <= R(f"({r})*")


def test_closed_form_reply_forest():
    """replyOf* on a forest: per source the ancestor chain, |R| = |V| + sum of
    depths (SURVEY.md §8(c) closed form)."""
    g, parent = synth.reply_forest(3000, seed=3)
    r = oracle.allpairs(g, "replyOf*")
    depth = np.zeros(g.num_vertices, dtype=np.int64)
    for i in range(g.num_vertices):
        depth[i] = 0 if parent[i] < 0 else depth[parent[i]] + 1
    assert int(r["counts"].sum()) == g.num_vertices + int(depth.sum())
    for s in [0, 17, 2999]:
        chain, v = [s], s
        while parent[v] >= 0:
            v = int(parent[v]); chain.append(v)
        got = r["dst"][r["src"] == s].tolist()
        assert got == sorted(chain)


def test_closed_form_knows_plus_components():
    """knows+ on a symmetric graph without self-loops: pairs = union of CxC
    over connected components with |C| >= 2 (scipy connected_components)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    g = synth.symmetric_graph(4000, 2600, seed=4)
    r = oracle.allpairs(g, "knows+", pairs=False)
    A = sp.csr_matrix((np.ones(g.num_edges), (g.src, g.dst)), shape=(g.num_vertices,) * 2)
    _, comp = connected_components(A, directed=False)
    sizes = np.bincount(comp)
    per_v = np.where(sizes[comp] >= 2, sizes[comp], 0)
    assert np.array_equal(r["counts"].astype(np.int64), per_v)


def test_chain_hop_coverage():
    """No hop limit (the correctness lesson of tab:max_hop):
    on a 64-edge chain, a* returns all i<=j pairs, a+ all i<j."""
    g = synth.chain_graph(64)
    n = 65
    assert int(oracle.allpairs(g, "a*", pairs=False)["counts"].sum()) == n * (n + 1) // 2
    assert int(oracle.allpairs(g, "a+", pairs=False)["counts"].sum()) == n * (n - 1) // 2


def test_pe_toy_and_hand_derivation():
    """PE (product edges traversed, reading R12) pinned by a hand derivation
    from the abc* automaton of P:258-259 (q0 -a-> q1 -b-> q2, c loop on q2):
      PE = sum_s deg_a(s) + sum_{(s,u) in R(a)} deg_b(u)
           + sum_{(s,u) in R(abc*)} deg_c(u),
    with the relations computed by O3 (algebra).  Toy graph: 22."""
    def degs(g, li):                      # out-degree over DISTINCT triples (R4)
        t = {(u, w) for u, l, w in zip(g.src.tolist(), g.label.tolist(), g.dst.tolist()) if l == li}
        return np.bincount(np.array([u for u, _ in t], dtype=np.int64), minlength=g.num_vertices)
    for g in [synth.toy_graph(), synth.random_graph(150, 600, 3, seed=11)]:
        da, db, dc = degs(g, 0), degs(g, 1), degs(g, 2)
        want = int(da.sum()) + sum(int(db[u]) for _, u in oracle.algebra(g, "a")) \
            + sum(int(dc[u]) for _, u in oracle.algebra(g, "abc*"))
        assert int(oracle.allpairs(g, "abc*")["pe"].sum()) == want
        if g.num_vertices == 14:
            assert want == 22
    # single-state a*: PE = sum over (s,u) in R(a*) of deg_a(u)
    g = synth.random_graph(150, 400, 2, seed=12)
    da = degs(g, 0)
    want = sum(int(da[u]) for _, u in oracle.algebra(g, "a*"))
    assert int(oracle.allpairs(g, "a*")["pe"].sum()) == want


def test_crpq_join_vs_bruteforce():
    """Hash-join CRPQ oracle == enumeration of all assignments (Def. 2)."""
    rng = np.random.default_rng(99)
    for trial in range(12):
        g = synth.random_small(rng, max_v=6, max_e=14, num_labels=3, min_v=2)
        g.vertex_label = rng.integers(0, 2, g.num_vertices).astype(np.uint16)
        g.vertex_label_names = ["P", "Q"]
        q = oracle.CRPQ(["x", "y", "z"], [("x", "a b*", "y"), ("y", "c*", "z"), ("x", "(a|c)+", "z")],
                        var_label={"x": "P"}, distinct=[("x", "z")] if trial % 2 else [])
        assert oracle.crpq_join(g, q) == oracle.crpq_bruteforce(g, q)


def test_uniform_generator_shape():
    g = synth.uniform_graph(2000, 20000, 4, seed=2)
    keys = set(zip(g.src.tolist(), g.label.tolist(), g.dst.tolist()))
    assert len(keys) == 20000 == g.num_edges


def test_longest_match_label_vocabulary():
    """Reading R3 pinned on a prefix-ambiguous vocabulary {reply, replyOf}:
    O1 (C parser), O2 (its own scanner) and O3 all read 'replyOf*' as the
    closure of the single label replyOf, and 'reply' as the other label.
    Expected sets written out from Definition 1 on this 4-edge graph."""
    names = ["reply", "replyOf"]
    # 0 -replyOf-> 1 -replyOf-> 2 ; 0 -reply-> 3 ; 3 -replyOf-> 0
    g = synth.Graph(4, np.array([0, 1, 0, 3], np.uint32), np.array([1, 2, 3, 0], np.uint32),
                    np.array([1, 1, 0, 1], np.uint16), names).check()
    ident = {(v, v) for v in range(4)}
    want = {
        "replyOf*": ident | {(0, 1), (0, 2), (1, 2), (3, 0), (3, 1), (3, 2)},
        "reply": {(0, 3)},
        "reply replyOf": {(0, 0)},
        "reply.replyOf+": {(0, 0), (0, 1), (0, 2)},
        "(replyOf|reply)+": {(a, b) for a in (0, 3) for b in range(4)} | {(0, 1), (0, 2), (1, 2)},
    }
    for rx, w in want.items():
        assert oracle.pair_set(oracle.allpairs(g, rx)) == w, ("O1", rx)
        assert oracle.brute_force(g, rx) == w, ("O2", rx)
        assert oracle.algebra(g, rx) == w, ("O3", rx)


def test_length_bounded_vs_brute_force():
    """Length-bounded RPQs: O1 with max_hops = k equals O2 with
    walks of length <= k (Definition 1 restricted to |path| <= k), in both
    automaton modes, on tiny random graphs; k >= O2's bound = unbounded."""
    rng = np.random.default_rng(17)
    for it in range(60):
        g = synth.random_small(rng, max_v=5, max_e=9)
        for rx in ["a*", "(a|b)*c", "a b* c", "c+", "(a|b)*c*", "a?b"]:
            for k in range(0, 5):
                want = oracle.brute_force(g, rx, max_len=k)
                for dfa in (True, False):
                    got = oracle.pair_set(oracle.allpairs(g, rx, use_dfa=dfa, max_hops=k))
                    assert got == want, (it, rx, k, dfa)
            big = oracle.allpairs(g, rx, max_hops=10_000)
            full = oracle.allpairs(g, rx)
            assert oracle.pair_set(big) == oracle.pair_set(full)
            assert np.array_equal(big["pe"], full["pe"])


def test_length_bounded_chain_closed_form():
    """a* on the chain 0 -a-> 1 -a-> ... -a-> n-1 with bound k: source i
    reaches i..min(i+k, n-1); the expanded product vertices are those at
    depth < k, each with one out-edge except vertex n-1, so
    PE(i) = |{v : i <= v <= min(i+k-1, n-2)}|."""
    n = 40
    g = synth.chain_graph(n - 1)              # n vertices, n - 1 edges
    for k in [0, 1, 2, 5, 39, 50]:
        r = oracle.allpairs(g, "a*", max_hops=k)
        want_pairs = {(i, j) for i in range(n) for j in range(i, min(i + k, n - 1) + 1)}
        assert oracle.pair_set(r) == want_pairs, k
        want_pe = [max(0, min(i + k - 1, n - 2) - i + 1) for i in range(n)]
        assert r["pe"].tolist() == want_pe, k
