"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/rpq.h declares, and its host-side compiler (rpq_compile_labels)
produces the same minimal trim DFA as the independent oracle compiler and the
language of Python `re`.  No GPU compute is called here."""
import itertools
import os
import re

import numpy as np
import pytest

import oracle
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rpq.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*([a-z_0-9]+)\s*\(", txt, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("rpq_", "crpq_"))))


def test_library_exports_every_header_symbol():
    import ctypes
    import paper_2602_20748_b200 as R
    lib = ctypes.CDLL(R.LIB_PATH)
    fns = header_functions()
    assert len(fns) >= 20
    for f in fns:
        assert hasattr(lib, f), f
    assert set(fns) == set(R.EXPORTED)


def test_library_is_sm100a():
    import subprocess
    import paper_2602_20748_b200 as R
    out = subprocess.run(["cuobjdump", "--list-elf", R.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_graph_load_fails_loudly():
    import paper_2602_20748_b200 as R
    if R.rpq_device_count() > 0:
        pytest.skip("GPU present")
    import synth
    with pytest.raises(R.RPQError) as e:
        R.rpq_graph_load(synth.toy_graph())
    assert e.value.status == R.RPQ_ECUDA


def test_no_gpu_trim_memory_einval():
    import paper_2602_20748_b200 as R
    if R.rpq_device_count() > 0:
        pytest.skip("GPU present")
    with pytest.raises(R.RPQError) as e:
        R.rpq_trim_memory(0)
    assert e.value.status == R.RPQ_EINVAL


NAMES = ["a", "b", "c", "d", "knows", "replyOf"]
REGEXES = ["abc*", "abcd", "a*", "knows+", "(a|b)*c", "(a|b)*c*", "ab*c", "a b* c", "a?b*",
           "ab*", "(a|b)b*", "a*b*", "ab*c*", "(a|b|c)*", "(ab)*", "a(b|c)?", "((a|b)c)+",
           "a**", "(a*)+", "replyOf*", "(a|b)*(c|d)(a|b)*", "a(b|c)*d+"]


@pytest.mark.parametrize("rx", REGEXES)
def test_compiler_matches_oracle_min_dfa(rx):
    """The minimal trim DFA is unique; both sides number states canonically
    (BFS from the initial state, labels ascending), so the transition lists
    must be identical (independent constructions: Glushkov + Hopcroft here,
    Thompson + Moore in the oracle)."""
    import paper_2602_20748_b200 as R
    a = R.rpq_compile_labels(NAMES, rx)
    info = a.info()
    assert info["is_dfa"]
    trans, finals = a.transitions()
    o = oracle.Automaton(rx, NAMES)
    assert sorted(trans) == sorted(o.dfa_transitions())
    assert finals == o.dfa_finals()
    assert info["accepts_empty"] == o.info()["accepts_empty"]


def test_paper_state_counts():
    """abc*: 3 states; abcd: |Q| = 5."""
    import paper_2602_20748_b200 as R
    assert R.rpq_compile_labels(NAMES, "abc*").info()["states"] == 3
    assert R.rpq_compile_labels(NAMES, "abcd").info()["states"] == 5
    tr, fin = R.rpq_compile_labels(NAMES, "abc*").transitions()
    assert sorted(tr) == [(0, 0, 1), (1, 1, 2), (2, 2, 2)] and fin == [2]


@pytest.mark.parametrize("rx", ["abc*", "(a|b)*c", "a?b*", "((a|b)c)+", "a(b|c)?", "(ab)*"])
def test_compiler_language_vs_python_re(rx):
    import paper_2602_20748_b200 as R
    pat = re.compile(oracle.to_python_re(rx, NAMES[:4]))
    for flags in (0, R.RPQ_NO_MINIMIZE):
        a = R.rpq_compile_labels(NAMES[:4], rx, flags)
        assert a.info()["is_dfa"] == (flags == 0)
        for n in range(6):
            for w in itertools.product(range(4), repeat=n):
                want = bool(pat.fullmatch("".join(chr(0xE000 + x) for x in w)))
                assert a.accepts(list(w)) == want, (rx, w, flags)


def test_compiler_errors():
    import paper_2602_20748_b200 as R
    for bad in ["", "()", "(a", "a|", "*a", "a)", "|a"]:
        with pytest.raises(R.RPQError) as e:
            R.rpq_compile_labels(NAMES, bad)
        assert e.value.status == R.RPQ_ESYNTAX, bad
    with pytest.raises(R.RPQError) as e:
        R.rpq_compile_labels(["a", "b"], "ab x")
    assert e.value.status == R.RPQ_ELABEL and e.value.offset == 3


def test_paper_dialect():
    import paper_2602_20748_b200 as R
    a = R.rpq_compile_labels(NAMES, "(a+b)*c", R.RPQ_SYNTAX_PAPER)
    b = R.rpq_compile_labels(NAMES, "(a|b)*c")
    assert a.transitions() == b.transitions()


def test_longest_match_tokenisation():
    """Reading R3: identifiers such as replyOf and knows are single labels."""
    import paper_2602_20748_b200 as R
    tr, fin = R.rpq_compile_labels(["reply", "replyOf", "knows"], "replyOf*").transitions()
    assert tr == [(0, 1, 0)] and fin == [0]


@pytest.mark.parametrize("rx", ["abc*", "(a|b)*c", "a?b*", "((a|b)c)+", "a(b|c)?", "(ab)*", "a b* c", "c*",
                                "(a|b)*(c|d)(a|b)*", "a(b|c)*d+"])
def test_nfa_reverse_language(rx):
    """rpq_nfa_reverse accepts exactly the reversed words (all words of length
    <= 6 against Python re on the reversed word), and reversing twice gives
    back the same canonical minimal DFA."""
    import paper_2602_20748_b200 as R
    pat = re.compile(oracle.to_python_re(rx, NAMES[:4]))
    a = R.rpq_compile_labels(NAMES[:4], rx)
    r = R.rpq_nfa_reverse(a)
    assert r.info()["accepts_empty"] == a.info()["accepts_empty"]
    for n in range(7):
        for w in itertools.product(range(4), repeat=n):
            want = bool(pat.fullmatch("".join(chr(0xE000 + x) for x in reversed(w))))
            assert r.accepts(list(w)) == want, (rx, w)
    assert R.rpq_nfa_reverse(r).transitions() == a.transitions()


def test_nfa_reverse_matches_reversed_regex():
    """abc* reversed is c*ba; (a|b)*c reversed is c(a|b)*: identical minimal DFAs."""
    import paper_2602_20748_b200 as R
    for rx, rrx in [("abc*", "c*ba"), ("(a|b)*c", "c(a|b)*"), ("a b* c", "c b* a")]:
        assert R.rpq_nfa_reverse(R.rpq_compile_labels(NAMES, rx)).transitions() == \
            R.rpq_compile_labels(NAMES, rrx).transitions()
