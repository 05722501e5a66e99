"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the RPQ method: it only draws edge-labelled
graphs (u32 src, u32 dst, u16 label triples + label names) whose shapes follow
the paper's workloads (BASELINE.json `configs`).  Both sides
dedup (u, label, w) themselves (reading R4 in DESIGN.md); generators may emit
duplicates.

Recipes (DESIGN.md §"Input recipe" states them in prose):
  toy_graph()       tab:LGF, PAPER.md P:357-379 (19 edges, labels a/b/c) with
                    vertex labels A/B/C/D of reading R9.
  uniform_graph()   cfg2: |V|=100,000, exactly 1,000,000 distinct i.i.d.
                    uniform (u, w, label) triples over 4 labels, seed 2.
  rmat_graph()      cfg5: Graph500 R-MAT (0.57,0.19,0.19,0.05), scale s,
                    edge factor 16, seeded vertex permutation, uniform labels.
  ldbc_graph()      cfg3: LDBC-SNB-shaped social graph (SF10 counts from
                    P:1015-1016, the rest Datagen-like and stated in DESIGN.md).
  random_small()    tiny random graphs for brute-force pins.
  reply_forest()    replyOf-style forest (one parent edge per non-root).
  symmetric_graph() undirected graph stored both ways (knows-style).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np


@dataclass
class Graph:
    num_vertices: int
    src: np.ndarray            # uint32 [E]
    dst: np.ndarray            # uint32 [E]
    label: np.ndarray          # uint16 [E]
    label_names: List[str]
    vertex_label: Optional[np.ndarray] = None      # uint16 [V] or None
    vertex_label_names: List[str] = field(default_factory=list)
    meta: dict = field(default_factory=dict)

    @property
    def num_edges(self) -> int:
        return int(self.src.shape[0])

    def check(self) -> "Graph":
        assert self.src.dtype == np.uint32 and self.dst.dtype == np.uint32
        assert self.label.dtype == np.uint16
        assert self.src.shape == self.dst.shape == self.label.shape
        if self.num_edges:
            assert int(self.src.max()) < self.num_vertices
            assert int(self.dst.max()) < self.num_vertices
            assert int(self.label.max()) < len(self.label_names)
        return self


def _mk(nv, src, dst, lab, names, vlab=None, vnames=(), **meta) -> Graph:
    return Graph(int(nv), np.ascontiguousarray(src, dtype=np.uint32),
                 np.ascontiguousarray(dst, dtype=np.uint32),
                 np.ascontiguousarray(lab, dtype=np.uint16), list(names),
                 None if vlab is None else np.ascontiguousarray(vlab, dtype=np.uint16),
                 list(vnames), dict(meta)).check()


# --------------------------------------------------------------------------
# cfg1: the paper's worked example
# --------------------------------------------------------------------------
# tab:LGF: slices S0..S11, vertex v_i has id i.
TOY_EDGES = {
    "a": [(0, 1), (0, 3), (2, 5), (0, 6), (7, 5)],
    "b": [(1, 4), (1, 10), (3, 12), (5, 2), (6, 1)],
    "c": [(2, 3), (3, 2), (4, 7), (10, 8), (13, 9), (10, 11), (11, 12),
          (12, 13), (13, 10)],
}
# Reading R9: A={v0..v3}, B={v4,v5}, C={v6..v9}, D={v10..v13}.
TOY_VERTEX_LABELS = ["A"] * 4 + ["B"] * 2 + ["C"] * 4 + ["D"] * 4


def toy_graph() -> Graph:
    names = ["a", "b", "c"]
    src, dst, lab = [], [], []
    for li, n in enumerate(names):
        for (u, w) in TOY_EDGES[n]:
            src.append(u); dst.append(w); lab.append(li)
    vnames = ["A", "B", "C", "D"]
    vlab = [vnames.index(x) for x in TOY_VERTEX_LABELS]
    return _mk(14, src, dst, lab, names, vlab, vnames, name="toy")


# --------------------------------------------------------------------------
# cfg2: uniform random labelled graph
# --------------------------------------------------------------------------
def uniform_graph(num_vertices: int = 100_000, num_edges: int = 1_000_000,
                  num_labels: int = 4, seed: int = 2) -> Graph:
    """Draw (u, w, l) i.i.d. uniform, keep the first `num_edges` DISTINCT
    triples in draw order (self-loops kept, reading R5)."""
    rng = np.random.default_rng(seed)
    names = [chr(ord("a") + i) for i in range(num_labels)] if num_labels <= 26 \
        else [f"l{i}" for i in range(num_labels)]
    need = num_edges
    keys_seen = np.empty(0, dtype=np.uint64)
    order_keys = []
    draw = int(num_edges * 1.05) + 1024
    while need > 0:
        u = rng.integers(0, num_vertices, draw, dtype=np.uint64)
        w = rng.integers(0, num_vertices, draw, dtype=np.uint64)
        l = rng.integers(0, num_labels, draw, dtype=np.uint64)
        key = (l * np.uint64(num_vertices) + u) * np.uint64(num_vertices) + w
        _, first = np.unique(key, return_index=True)
        first.sort()
        key = key[first]                       # distinct within draw, draw order
        if keys_seen.size:
            key = key[~np.isin(key, keys_seen)]
        key = key[:need]
        order_keys.append(key)
        keys_seen = np.concatenate([keys_seen, key])
        need -= key.size
        draw = max(need * 2, 1024)
    key = np.concatenate(order_keys)
    w = key % np.uint64(num_vertices)
    rest = key // np.uint64(num_vertices)
    u = rest % np.uint64(num_vertices)
    l = rest // np.uint64(num_vertices)
    return _mk(num_vertices, u, w, l, names, name="uniform", seed=seed)


# --------------------------------------------------------------------------
# cfg5: R-MAT
# --------------------------------------------------------------------------
def rmat_graph(scale: int = 24, edge_factor: int = 16, num_labels: int = 8,
               seed: int = 24, abcd=(0.57, 0.19, 0.19, 0.05),
               chunk: int = 1 << 22) -> Graph:
    """Graph500-style R-MAT: 2**scale vertices, edge_factor * 2**scale edge
    samples, per-bit quadrant choice with probabilities (A,B,C,D), then a
    seeded random vertex permutation; labels uniform over `num_labels`."""
    rng = np.random.default_rng(seed)
    nv = 1 << scale
    ne = edge_factor * nv
    a, b, c, _ = abcd
    src = np.empty(ne, dtype=np.uint32)
    dst = np.empty(ne, dtype=np.uint32)
    for s0 in range(0, ne, chunk):
        n = min(chunk, ne - s0)
        u = np.zeros(n, dtype=np.uint32)
        w = np.zeros(n, dtype=np.uint32)
        for bit in range(scale):
            r = rng.random(n, dtype=np.float32)
            ubit = r >= (a + b)                       # quadrants C or D
            wbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)   # B or D
            u |= ubit.astype(np.uint32) << np.uint32(bit)
            w |= wbit.astype(np.uint32) << np.uint32(bit)
        src[s0:s0 + n] = u
        dst[s0:s0 + n] = w
    perm = rng.permutation(nv).astype(np.uint32)
    src = perm[src]
    dst = perm[dst]
    lab = rng.integers(0, num_labels, ne, dtype=np.uint16)
    names = [chr(ord("a") + i) for i in range(num_labels)]
    return _mk(nv, src, dst, lab, names, name="rmat", scale=scale, seed=seed)


# --------------------------------------------------------------------------
# small graphs for pins
# --------------------------------------------------------------------------
def random_small(rng: np.random.Generator, max_v: int = 6, max_e: int = 10,
                 num_labels: int = 3, min_v: int = 1) -> Graph:
    nv = int(rng.integers(min_v, max_v + 1))
    ne = int(rng.integers(0, max_e + 1))
    src = rng.integers(0, nv, ne)
    dst = rng.integers(0, nv, ne)
    lab = rng.integers(0, num_labels, ne)
    names = [chr(ord("a") + i) for i in range(num_labels)]
    return _mk(nv, src, dst, lab, names, name="random_small")


def random_graph(num_vertices: int, num_edges: int, num_labels: int,
                 seed: int) -> Graph:
    rng = np.random.default_rng(seed)
    src = rng.integers(0, num_vertices, num_edges)
    dst = rng.integers(0, num_vertices, num_edges)
    lab = rng.integers(0, num_labels, num_edges)
    names = [chr(ord("a") + i) for i in range(num_labels)]
    return _mk(num_vertices, src, dst, lab, names, name="random", seed=seed)


def reply_forest(num_vertices: int, seed: int, root_prob: float = 0.2,
                 window: int = 64, label_name: str = "replyOf"):
    """Vertex i>0 is a root with prob root_prob, else has exactly one parent
    edge i -replyOf-> p with p drawn from the previous `window` vertices.
    Returns (graph, parent) with parent[i] = -1 for roots."""
    rng = np.random.default_rng(seed)
    parent = np.full(num_vertices, -1, dtype=np.int64)
    for i in range(1, num_vertices):
        if rng.random() >= root_prob:
            parent[i] = int(rng.integers(max(0, i - window), i))
    child = np.nonzero(parent >= 0)[0]
    g = _mk(num_vertices, child, parent[child], np.zeros(child.size), [label_name],
            name="reply_forest")
    return g, parent


def symmetric_graph(num_vertices: int, num_pairs: int, seed: int,
                    label_name: str = "knows") -> Graph:
    """Undirected pairs {u,w}, u != w, stored both ways (reading R16)."""
    rng = np.random.default_rng(seed)
    u = rng.integers(0, num_vertices, num_pairs)
    w = rng.integers(0, num_vertices, num_pairs)
    keep = u != w
    u, w = u[keep], w[keep]
    src = np.concatenate([u, w])
    dst = np.concatenate([w, u])
    return _mk(num_vertices, src, dst, np.zeros(src.size), [label_name],
               name="symmetric")


def chain_graph(length: int, label_name: str = "a") -> Graph:
    """v0 -a-> v1 -a-> ... -a-> v_length (hop-coverage pin)."""
    src = np.arange(length)
    return _mk(length + 1, src, src + 1, np.zeros(length), [label_name],
               name="chain")


def relabel(g: Graph, perm: np.ndarray) -> Graph:
    """Apply a vertex permutation pi (new id = perm[old id])."""
    perm = np.asarray(perm, dtype=np.uint32)
    vl = None
    if g.vertex_label is not None:
        vl = np.empty_like(g.vertex_label)
        vl[perm] = g.vertex_label
    return _mk(g.num_vertices, perm[g.src], perm[g.dst], g.label, g.label_names,
               vl, g.vertex_label_names, name=g.meta.get("name", "") + "+relabel")


def sample_sources(num_vertices: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    n = min(n, num_vertices)
    return np.sort(rng.choice(num_vertices, n, replace=False)).astype(np.uint32)


# --------------------------------------------------------------------------
# cfg3 / cfg4: LDBC-SNB-shaped social graph
# --------------------------------------------------------------------------
LDBC_VERTEX_LABELS = ["Person", "Forum", "Post", "Comment", "Tag", "TagClass", "City", "Country",
                      "Continent", "University", "Company", "Filler"]
LDBC_EDGE_LABELS = ["knows", "replyOf", "hasCreator", "hasTag", "containerOf", "isLocatedIn", "hasMember",
                    "hasModerator", "hasInterest", "studyAt", "workAt", "isPartOf", "isSubclassOf", "hasType",
                    "likes"]
# SF10 sizes: |V| = 35.5 M and |E| = 219.4 M, 12 vertex / 15 edge labels
# (P:1015-1016); the split below is Datagen-like and assumed.
LDBC_SF10_COUNTS = {"Person": 65_000, "Forum": 600_000, "Post": 7_000_000, "Tag": 16_080, "TagClass": 71,
                    "City": 1_343, "Country": 111, "Continent": 6, "University": 6_380, "Company": 1_575,
                    "Filler": 9_434}
LDBC_SF10_V, LDBC_SF10_E = 35_500_000, 219_400_000


def _zipf_pick(rng, n, size, a=0.5):
    """Indices in [0, n) with P(i) ~ (i+1)^-a (Chung-Lu style weights)."""
    w = (np.arange(1, n + 1, dtype=np.float64)) ** (-a)
    c = np.cumsum(w)
    c /= c[-1]
    return np.minimum(np.searchsorted(c, rng.random(size)), n - 1).astype(np.int64)


def ldbc_graph(scale: float = 1.0, seed: int = 10, sports_frac: float = 0.005) -> Graph:
    """LDBC-SNB-shaped graph; scale=1.0 is SF10 size (35.5 M vertices,
    219.4 M edges).  Vertex ids are label-contiguous in LDBC_VERTEX_LABELS
    order (Post and Comment adjacent = the message range).  Edges:
      knows      2 M undirected pairs x scale among persons, Zipf(0.5) weights,
                 80 % inside one of 100 contiguous communities, stored both ways;
      replyOf    one per comment: a random Post (p = 0.45) else an earlier
                 comment within 4096 positions (a forest);
      hasCreator one per message (Zipf person); hasTag one per message (+1 for
                 15 %), tag 0 = "Sports" with prob sports_frac, else Zipf;
      containerOf one per post; isLocatedIn one per person and message;
      hasMember/hasModerator/hasInterest/studyAt/workAt/isPartOf/isSubclassOf/
      hasType as filler; likes = person -> message, the remainder up to
      219.4 M x scale edges."""
    rng = np.random.default_rng(seed)
    cnt = {k: max(1, int(round(v * scale))) for k, v in LDBC_SF10_COUNTS.items()}
    for k in ["Tag", "TagClass", "City", "Country", "Continent"]:
        cnt[k] = max(cnt[k], min(LDBC_SF10_COUNTS[k], 8))
    nv_target = max(int(round(LDBC_SF10_V * scale)), sum(cnt.values()) + 10)
    cnt["Comment"] = nv_target - sum(cnt.values())
    base, off = {}, 0
    for k in LDBC_VERTEX_LABELS:
        base[k] = off
        off += cnt[k]
    nv = off
    E = {k: i for i, k in enumerate(LDBC_EDGE_LABELS)}
    S, D, L = [], [], []

    def add(u, w, lab):
        S.append(np.asarray(u, dtype=np.uint32))
        D.append(np.asarray(w, dtype=np.uint32))
        L.append(np.full(len(u), E[lab], dtype=np.uint16))

    P, F, Po, C, T = cnt["Person"], cnt["Forum"], cnt["Post"], cnt["Comment"], cnt["Tag"]
    # knows
    npairs = max(1, int(2_000_000 * scale))
    u = _zipf_pick(rng, P, npairs)
    ncomm = 100
    csize = max(1, P // ncomm)
    intra = rng.random(npairs) < 0.8
    comm0 = (u // csize) * csize
    v_in = comm0 + (csize * rng.random(npairs) ** 2).astype(np.int64)
    v_in = np.minimum(v_in, P - 1)
    v_out = _zipf_pick(rng, P, npairs)
    v = np.where(intra, v_in, v_out)
    keep = u != v
    u, v = u[keep] + base["Person"], v[keep] + base["Person"]
    add(np.concatenate([u, v]), np.concatenate([v, u]), "knows")
    # replyOf: comment i -> post or earlier comment
    i = np.arange(C, dtype=np.int64)
    to_post = (rng.random(C) < 0.45) | (i == 0)
    back = 1 + (rng.random(C) * np.minimum(np.maximum(i, 1), 4096)).astype(np.int64)
    parent_c = np.maximum(i - back, 0)
    parent = np.where(to_post, base["Post"] + rng.integers(0, Po, C), base["Comment"] + parent_c)
    add(base["Comment"] + i, parent, "replyOf")
    nmsg = Po + C
    msg = base["Post"] + np.arange(nmsg, dtype=np.int64)
    add(msg, base["Person"] + _zipf_pick(rng, P, nmsg), "hasCreator")
    first = np.where(rng.random(nmsg) < sports_frac, 0, 1 + _zipf_pick(rng, max(1, T - 1), nmsg) % max(1, T - 1))
    first = np.minimum(first, T - 1)
    second_m = msg[rng.random(nmsg) < 0.15]
    add(np.concatenate([msg, second_m]),
        base["Tag"] + np.concatenate([first, 1 + _zipf_pick(rng, max(1, T - 1), second_m.size) % max(1, T - 1)]),
        "hasTag")
    add(base["Forum"] + rng.integers(0, F, Po), base["Post"] + np.arange(Po), "containerOf")
    ppl = base["Person"] + np.arange(P)
    add(np.concatenate([ppl, msg]),
        np.concatenate([base["City"] + rng.integers(0, cnt["City"], P),
                        base["Country"] + rng.integers(0, cnt["Country"], nmsg)]), "isLocatedIn")
    nmem = max(1, int(10_000_000 * scale))
    add(base["Forum"] + rng.integers(0, F, nmem), base["Person"] + _zipf_pick(rng, P, nmem), "hasMember")
    add(base["Forum"] + np.arange(F), base["Person"] + _zipf_pick(rng, P, F), "hasModerator")
    nint = P * 10
    add(base["Person"] + rng.integers(0, P, nint), base["Tag"] + _zipf_pick(rng, T, nint), "hasInterest")
    add(ppl, base["University"] + rng.integers(0, cnt["University"], P), "studyAt")
    add(ppl, base["Company"] + rng.integers(0, cnt["Company"], P), "workAt")
    add(np.concatenate([base["City"] + np.arange(cnt["City"]), base["Country"] + np.arange(cnt["Country"])]),
        np.concatenate([base["Country"] + rng.integers(0, cnt["Country"], cnt["City"]),
                        base["Continent"] + rng.integers(0, cnt["Continent"], cnt["Country"])]), "isPartOf")
    tc = base["TagClass"] + np.arange(1, cnt["TagClass"])
    add(tc, base["TagClass"] + rng.integers(0, np.maximum(1, tc - base["TagClass"])), "isSubclassOf")
    add(base["Tag"] + np.arange(T), base["TagClass"] + rng.integers(0, cnt["TagClass"], T), "hasType")
    fixed = sum(x.size for x in S)
    nlikes = max(0, int(round(LDBC_SF10_E * scale)) - fixed)
    add(base["Person"] + _zipf_pick(rng, P, nlikes), base["Post"] + rng.integers(0, nmsg, nlikes), "likes")
    src = np.concatenate(S)
    dst = np.concatenate(D)
    lab = np.concatenate(L)
    vlab = np.zeros(nv, dtype=np.uint16)
    for k, name in enumerate(LDBC_VERTEX_LABELS):
        vlab[base[name]:base[name] + cnt[name]] = k
    g = _mk(nv, src, dst, lab, LDBC_EDGE_LABELS, vlab, LDBC_VERTEX_LABELS, name="ldbc", scale=scale, seed=seed)
    g.meta.update({"base": base, "count": cnt, "reply_parent": parent, "sports": base["Tag"]})
    return g
