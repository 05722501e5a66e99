"""CPU oracles for RPQ / CRPQ evaluation -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  Nothing here is imported
by, or imports, the CUDA product path (paper_2602_20748_b200/).

Three oracles that share no code with the product path or with each other
(citations are PAPER.md = /root/reference/PAPER.md lines):

  O1  ``OracleGraph`` / ``Automaton`` / ``eval_sources`` -- ctypes wrapper of
      oracle/rpq_oracle.c: per-source product-graph BFS with a visited set
      over (vertex, state); Thompson epsilon-NFA or its minimal
      trim DFA; also counts product edges traversed (PE, reading R12).
  O2  ``brute_force`` -- Definition 1 literally: enumerate walks
      up to a length bound and test each label word with Python ``re``.
  O3  ``algebra`` -- the algebra-based approach: relations per
      label, join for concatenation, union for alternation, the alpha-operator
      fixpoint for closure; Id_V added for star/optional (reading R1).

CRPQ (Definition 2): ``crpq_bruteforce`` enumerates every
assignment on tiny graphs; ``crpq_join`` hash-joins O1 atom relations.

Parity status: O1 is pinned by tests/test_oracle.py against the paper's worked
example (P:84 footnote 1), against O2 and O3, and against closed
forms; PE is pinned against a hand derivation from the abc* automaton of
P:258-259 (see tests).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import itertools
import os
import re
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "rpq_oracle.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle/rpq_oracle.c (plain C, gcc) into oracle/liboracle.so."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-Wall", "-shared", "-fPIC", "-pthread",
                               "-o", _SO, _SRC])
    return _SO


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    L = ctypes.CDLL(_SO)
    P = ctypes.POINTER
    u32p, u64p = P(ctypes.c_uint32), P(ctypes.c_uint64)
    L.og_graph_new.restype = ctypes.c_void_p
    L.og_graph_new.argtypes = [ctypes.c_uint32, ctypes.c_uint64, u32p, u32p,
                               P(ctypes.c_uint16), ctypes.c_uint32]
    L.og_graph_free.argtypes = [ctypes.c_void_p]
    L.og_graph_num_edges.restype = ctypes.c_uint64
    L.og_graph_num_edges.argtypes = [ctypes.c_void_p]
    L.og_compile.restype = ctypes.c_void_p
    L.og_compile.argtypes = [ctypes.c_char_p, P(ctypes.c_char_p), ctypes.c_uint32,
                             ctypes.c_int, P(ctypes.c_int), P(ctypes.c_size_t)]
    L.og_automaton_free.argtypes = [ctypes.c_void_p]
    ip = P(ctypes.c_int)
    L.og_automaton_info.argtypes = [ctypes.c_void_p, ctypes.c_int, ip, ip, ip, ip]
    L.og_dfa_transitions.restype = ctypes.c_int
    L.og_dfa_transitions.argtypes = [ctypes.c_void_p, ip, ip, ip, ctypes.c_int]
    L.og_dfa_is_final.restype = ctypes.c_int
    L.og_dfa_is_final.argtypes = [ctypes.c_void_p, ctypes.c_int]
    L.og_accepts.restype = ctypes.c_int
    L.og_accepts.argtypes = [ctypes.c_void_p, ctypes.c_int, ip, ctypes.c_int]
    L.og_eval.restype = ctypes.c_int
    L.og_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, u32p,
                          ctypes.c_uint64, ctypes.c_int, ctypes.c_int, u64p, u64p,
                          P(u32p), P(u32p), u64p]
    L.og_eval_bounded.restype = ctypes.c_int
    L.og_eval_bounded.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, u32p,
                                  ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, u64p, u64p,
                                  P(u32p), P(u32p), u64p]
    L.og_free.argtypes = [ctypes.c_void_p]
    _lib = L
    return L


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class OracleError(RuntimeError):
    def __init__(self, status, offset=0, msg=""):
        super().__init__(f"oracle status {status} at offset {offset} {msg}")
        self.status, self.offset = status, offset


OG_ESYNTAX, OG_ELABEL = -2, -3


class OracleGraph:
    """Edge-labelled graph G=(V,E,L) of P:182-183 (E deduplicated, R4)."""

    def __init__(self, graph):
        L = _load()
        self.g = graph
        self.nv = int(graph.num_vertices)
        self.label_names = list(graph.label_names)
        src = np.ascontiguousarray(graph.src, dtype=np.uint32)
        dst = np.ascontiguousarray(graph.dst, dtype=np.uint32)
        lab = np.ascontiguousarray(graph.label, dtype=np.uint16)
        self.h = L.og_graph_new(self.nv, src.size, _ptr(src, ctypes.c_uint32),
                                _ptr(dst, ctypes.c_uint32), _ptr(lab, ctypes.c_uint16),
                                len(self.label_names))
        if not self.h:
            raise OracleError(-1, msg="bad graph")
        self.num_edges = int(L.og_graph_num_edges(self.h))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.og_graph_free(self.h)
            self.h = None


class Automaton:
    """Thompson NFA + minimal trim DFA of a regex over a label vocabulary."""

    def __init__(self, regex: str, label_names: Sequence[str], paper_dialect: bool = False):
        L = _load()
        names = (ctypes.c_char_p * max(1, len(label_names)))(*[n.encode() for n in label_names])
        st = ctypes.c_int(0)
        off = ctypes.c_size_t(0)
        self.h = L.og_compile(regex.encode(), names, len(label_names), int(paper_dialect),
                              ctypes.byref(st), ctypes.byref(off))
        if not self.h:
            raise OracleError(st.value, off.value, regex)
        self.regex = regex

    def info(self, dfa: bool = True) -> dict:
        a = [ctypes.c_int(0) for _ in range(4)]
        _lib.og_automaton_info(self.h, int(dfa), *[ctypes.byref(x) for x in a])
        return {"states": a[0].value, "transitions": a[1].value,
                "accepts_empty": bool(a[2].value), "finals": a[3].value}

    def dfa_transitions(self) -> List[Tuple[int, int, int]]:
        n = _lib.og_dfa_transitions(self.h, None, None, None, 0)
        f = (ctypes.c_int * max(n, 1))(); l = (ctypes.c_int * max(n, 1))(); t = (ctypes.c_int * max(n, 1))()
        _lib.og_dfa_transitions(self.h, f, l, t, n)
        return [(f[i], l[i], t[i]) for i in range(n)]

    def dfa_finals(self) -> List[int]:
        n = self.info(True)["states"]
        return [d for d in range(n) if _lib.og_dfa_is_final(self.h, d)]

    def accepts(self, word: Sequence[int], dfa: bool = True) -> bool:
        w = (ctypes.c_int * max(1, len(word)))(*word)
        return bool(_lib.og_accepts(self.h, int(dfa), w, len(word)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.og_automaton_free(self.h)
            self.h = None


def eval_sources(og: OracleGraph, regex: str, sources=None, *, pairs: bool = True,
                 use_dfa: bool = True, threads: int = 0, paper_dialect: bool = False,
                 max_hops: Optional[int] = None):
    """O1: single-source RPQ for each source (all of V when sources is None).
    max_hops = k: only paths of length <= k (BFS depth bound).

    Returns dict(counts=u64[n], pe=u64[n], src=u32[], dst=u32[]) with pairs
    sorted by (source order given, target ascending)."""
    L = _load()
    A = Automaton(regex, og.label_names, paper_dialect)
    if sources is None:
        sources = np.arange(og.nv, dtype=np.uint32)
    sources = np.ascontiguousarray(sources, dtype=np.uint32)
    n = sources.size
    counts = np.zeros(n, dtype=np.uint64)
    pe = np.zeros(n, dtype=np.uint64)
    ps = ctypes.POINTER(ctypes.c_uint32)()
    pd = ctypes.POINTER(ctypes.c_uint32)()
    npairs = ctypes.c_uint64(0)
    threads = threads or os.cpu_count() or 1
    st = L.og_eval_bounded(og.h, A.h, int(use_dfa), _ptr(sources, ctypes.c_uint32), n, threads,
                           int(pairs), -1 if max_hops is None else int(max_hops),
                           _ptr(counts, ctypes.c_uint64), _ptr(pe, ctypes.c_uint64),
                           ctypes.byref(ps), ctypes.byref(pd), ctypes.byref(npairs))
    if st != 0:
        raise OracleError(st)
    out = {"counts": counts, "pe": pe, "sources": sources}
    if pairs:
        m = npairs.value
        if m:
            out["src"] = np.ctypeslib.as_array(ps, (m,)).copy()
            out["dst"] = np.ctypeslib.as_array(pd, (m,)).copy()
        else:
            out["src"] = np.zeros(0, np.uint32)
            out["dst"] = np.zeros(0, np.uint32)
        L.og_free(ps)
        L.og_free(pd)
    return out


def allpairs(graph, regex: str, *, use_dfa: bool = True, threads: int = 0,
             paper_dialect: bool = False, pairs: bool = True, max_hops: Optional[int] = None):
    """O1 all-pairs RPQ (x ranges over all of V, reading R11)."""
    og = OracleGraph(graph)
    return eval_sources(og, regex, None, pairs=pairs, use_dfa=use_dfa, threads=threads,
                        paper_dialect=paper_dialect, max_hops=max_hops)


def pair_set(res) -> set:
    return set(zip(res["src"].tolist(), res["dst"].tolist()))


# ==========================================================================
# O3's tokeniser (reading R3: longest match; '.', '/' and whitespace are
# optional concatenation; R2 dialects).  O2 has its own (below): the three
# oracles share no code.
# ==========================================================================
_OPS = "()|*+?"


def tokenize(regex: str, names: Sequence[str]) -> List[Tuple[str, object]]:
    toks, i = [], 0
    while i < len(regex):
        c = regex[i]
        if c in " \t\n./":
            i += 1
            continue
        if c in _OPS:
            toks.append(("op", c)); i += 1
            continue
        best, bl = -1, 0
        for k, n in enumerate(names):
            if n and regex.startswith(n, i) and len(n) > bl:
                best, bl = k, len(n)
        if best < 0:
            raise OracleError(OG_ELABEL, i, regex)
        toks.append(("lab", best)); i += bl
    return toks


# ==========================================================================
# O2: brute force over walks (Definition 1)
# ==========================================================================
def _o2_label_pattern(names: Sequence[str]):
    """O2's own scanner (reading R3): one Python ``re`` alternation of the
    label names, longest names first, so that ``re`` performs the longest
    match at every position (e.g. 'replyOf' before 'reply')."""
    order = sorted((k for k, n in enumerate(names) if n), key=lambda k: -len(names[k]))
    return order, re.compile("|".join(re.escape(names[k]) for k in order)) if order else None


def to_python_re(regex: str, names: Sequence[str], paper_dialect: bool = False) -> str:
    """Map each label to one private-use character; Python's own ``re``
    parser then parses the expression (no parser of ours is involved)."""
    order, pat = _o2_label_pattern(names)
    out, i = [], 0
    while i < len(regex):
        c = regex[i]
        if c.isspace() or c in "./":
            i += 1
        elif c in "()|*?":
            out.append(c)
            i += 1
        elif c == "+":
            out.append("|" if paper_dialect else "+")
            i += 1
        else:
            m = pat.match(regex, i) if pat else None
            if not m:
                raise OracleError(OG_ELABEL, i, regex)
            out.append(chr(0xE000 + list(names).index(m.group(0))))
            i = m.end()
    return "".join(out)


def _o2_num_labels(regex: str, names: Sequence[str]) -> int:
    """Label occurrences in rho (O2's walk-length bound)."""
    return sum(1 for ch in to_python_re(regex, names) if ord(ch) >= 0xE000)


def brute_force(graph, regex: str, paper_dialect: bool = False,
                max_len: Optional[int] = None) -> set:
    """{(x,y)}: some walk x..y of length <= max_len has a label word in L(rho).

    The default bound |V| * (#label occurrences in rho + 1) is >= the number
    of product states of the position automaton, so every pair has a witness
    within it (pigeonhole on a shortest product path)."""
    pat = re.compile(to_python_re(regex, graph.label_names, paper_dialect))
    nv = graph.num_vertices
    occ = _o2_num_labels(regex, graph.label_names)
    if max_len is None:
        max_len = nv * (occ + 1)
    adj: Dict[int, List[Tuple[int, str]]] = {v: [] for v in range(nv)}
    for u, w, l in set(zip(graph.src.tolist(), graph.dst.tolist(), graph.label.tolist())):
        adj[u].append((w, chr(0xE000 + l)))
    res = set()
    for x in range(nv):
        frontier = {(x, "")}
        seen = set(frontier)
        for _k in range(max_len + 1):
            for (v, word) in frontier:
                if pat.fullmatch(word):
                    res.add((x, v))
            nxt = set()
            for (v, word) in frontier:
                for (w, ch) in adj[v]:
                    t = (w, word + ch)
                    if t not in seen:
                        seen.add(t); nxt.add(t)
            frontier = nxt
            if len(seen) > 2_000_000:
                raise OracleError(-4, msg="brute force too large; use a smaller graph")
            if not frontier:
                break
    return res


# ==========================================================================
# O3: relational algebra (the algebra-based approach)
# ==========================================================================
def _parse_ast(regex: str, names: Sequence[str], paper_dialect: bool):
    toks = tokenize(regex, names)
    pos = [0]

    def peek():
        return toks[pos[0]] if pos[0] < len(toks) else (None, None)

    def alt():
        r = cat()
        while peek() == ("op", "|") or (paper_dialect and peek() == ("op", "+")):
            pos[0] += 1
            r = ("alt", r, cat())
        return r

    def cat():
        r = post()
        while peek()[0] == "lab" or peek() == ("op", "("):
            r = ("cat", r, post())
        return r

    def post():
        r = atom()
        while True:
            t = peek()
            if t == ("op", "*"):
                r = ("star", r)
            elif t == ("op", "?"):
                r = ("opt", r)
            elif t == ("op", "+") and not paper_dialect:
                r = ("plus", r)
            else:
                break
            pos[0] += 1
        return r

    def atom():
        t = peek()
        if t == ("op", "("):
            pos[0] += 1
            r = alt()
            if peek() != ("op", ")"):
                raise OracleError(OG_ESYNTAX, pos[0], regex)
            pos[0] += 1
            return r
        if t[0] == "lab":
            pos[0] += 1
            return ("lab", t[1])
        raise OracleError(OG_ESYNTAX, pos[0], regex)

    r = alt()
    if pos[0] != len(toks):
        raise OracleError(OG_ESYNTAX, pos[0], regex)
    return r


def algebra(graph, regex: str, paper_dialect: bool = False) -> set:
    """R(l) = E_l; R(ab) = R(a) o R(b); R(a|b) = R(a) u R(b);
    R(a+) = alpha-operator fixpoint (start from R(a), repeatedly join with
    R(a) and union until no new pair); R(a*) = Id_V u R(a+);
    R(a?) = Id_V u R(a)."""
    import scipy.sparse as sp
    nv = graph.num_vertices
    ident = sp.identity(nv, dtype=bool, format="csr")

    def rel(lbl):
        m = graph.label == lbl
        return sp.csr_matrix((np.ones(int(m.sum()), dtype=bool),
                              (graph.src[m].astype(np.int64), graph.dst[m].astype(np.int64))),
                             shape=(nv, nv), dtype=bool)

    def boolify(x):
        x = x.tocsr()
        x.data = np.ones_like(x.data, dtype=bool)
        x.eliminate_zeros()
        return x.astype(bool)

    def closure_plus(R):
        X = R.copy()
        while True:
            Xn = boolify(X + boolify(X.astype(np.int64) @ R.astype(np.int64)))
            if Xn.nnz == X.nnz:
                return Xn
            X = Xn

    def ev(n):
        k = n[0]
        if k == "lab":
            return rel(n[1])
        if k == "cat":
            return boolify(ev(n[1]).astype(np.int64) @ ev(n[2]).astype(np.int64))
        if k == "alt":
            return boolify(ev(n[1]) + ev(n[2]))
        if k == "plus":
            return closure_plus(ev(n[1]))
        if k == "star":
            return boolify(ident + closure_plus(ev(n[1])))
        if k == "opt":
            return boolify(ident + ev(n[1]))
        raise ValueError(k)

    R = ev(_parse_ast(regex, graph.label_names, paper_dialect)).tocoo()
    return set(zip(R.row.tolist(), R.col.tolist()))


# ==========================================================================
# CRPQ oracles (Definition 2)
# ==========================================================================
class CRPQ:
    """vars: names; var_label: vertex-label name or None (reading R7);
    var_const: vertex id or None; atoms: (x, regex, y) with var names;
    distinct: list of (var, var) filters."""

    def __init__(self, vars, atoms, var_label=None, var_const=None, distinct=()):
        self.vars = list(vars)
        self.atoms = list(atoms)
        self.var_label = dict(var_label or {})
        self.var_const = dict(var_const or {})
        self.distinct = list(distinct)


def _atom_relation(og: OracleGraph, regex: str, sources=None) -> set:
    r = eval_sources(og, regex, sources, pairs=True)
    return set(zip(r["src"].tolist(), r["dst"].tolist()))


def _candidates(graph, q: CRPQ, v):
    if q.var_const.get(v) is not None:
        cands = [int(q.var_const[v])]
    else:
        cands = list(range(graph.num_vertices))
    lab = q.var_label.get(v)
    if lab is not None:
        li = graph.vertex_label_names.index(lab)
        cands = [c for c in cands if int(graph.vertex_label[c]) == li]
    return cands


def crpq_bruteforce(graph, q: CRPQ) -> List[tuple]:
    """Enumerate every assignment f: V_q -> V and keep those satisfying (1)
    vertex labels, constants, (2) every atom, and the distinct filters."""
    og = OracleGraph(graph)
    rels = {i: _atom_relation(og, rx) for i, (_, rx, _) in enumerate(q.atoms)}
    cands = [_candidates(graph, q, v) for v in q.vars]
    idx = {v: i for i, v in enumerate(q.vars)}
    out = []
    for f in itertools.product(*cands):
        if any((f[idx[x]], f[idx[y]]) not in rels[i] for i, (x, _, y) in enumerate(q.atoms)):
            continue
        if any(f[idx[a]] == f[idx[b]] for a, b in q.distinct):
            continue
        out.append(tuple(f))
    return sorted(set(out))


def crpq_join(graph, q: CRPQ, og: Optional[OracleGraph] = None) -> List[tuple]:
    """Hash-join of O1 atom relations in the given atom order (each atom must
    share a variable with the earlier ones); then label/constant/distinct
    filters.  Tuples sorted lexicographically in variable order."""
    og = og or OracleGraph(graph)
    idx = {v: i for i, v in enumerate(q.vars)}
    allowed = {v: set(_candidates(graph, q, v)) for v in q.vars}
    table: Optional[List[dict]] = None
    for (x, rx, y) in q.atoms:
        x_bound = table is not None and (not table or x in table[0])
        srcs = sorted({t[x] for t in table}) if x_bound else sorted(allowed[x])
        srcs = np.array([s for s in srcs if s in allowed[x]], dtype=np.uint32)
        rel = _atom_relation(og, rx, srcs) if srcs.size else set()
        rel = {(a, b) for (a, b) in rel if b in allowed[y] and (x != y or a == b)}
        if table is None:
            table = [{x: a, y: b} for (a, b) in rel]
            continue
        if not table:
            break
        bound = set(table[0])
        nt = []
        if x in bound:
            by_src: Dict[int, List[int]] = {}
            for a, b in rel:
                by_src.setdefault(a, []).append(b)
            for t in table:
                for b in by_src.get(t[x], []):
                    if y in bound:
                        if t[y] == b:
                            nt.append(dict(t))
                    else:
                        u = dict(t); u[y] = b; nt.append(u)
        elif y in bound:
            by_dst: Dict[int, List[int]] = {}
            for a, b in rel:
                by_dst.setdefault(b, []).append(a)
            for t in table:
                for a in by_dst.get(t[y], []):
                    u = dict(t); u[x] = a; nt.append(u)
        else:
            raise ValueError("atom shares no variable with earlier atoms")
        table = nt
    table = table or []
    out = set()
    for t in table:
        if any(t[a] == t[b] for a, b in q.distinct):
            continue
        out.add(tuple(t[v] for v in q.vars))
    return sorted(out)
