"""Python binding of the RPQ / CRPQ C-ABI (include/rpq.h) -- marshalling only.

Every step of evaluation runs in librpq.so (hand-written sm_100a kernels);
this module only converts arguments and wraps handles.  The function names are
the C names.  There is no CPU fallback: if librpq.so is missing the import
fails, and GPU calls return RPQ_ECUDA (raised as RPQError) without a device.

PAPER.md citations (P:n): Definition 1, Definition 2
(P:204-210), automata-based evaluation.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RPQ_LIB_PATH selects an alternative build of the same library (kernel
# tuning experiments); the default is the in-tree librpq.so
LIB_PATH = os.environ.get("RPQ_LIB_PATH") or os.path.join(_HERE, "librpq.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `make` (or __graft_entry__.build()); "
                      "the CUDA library is required, there is no fallback")
_lib = ctypes.CDLL(LIB_PATH)

# ---- constants (include/rpq.h) ---------------------------------------------
RPQ_OK, RPQ_EINVAL, RPQ_ESYNTAX, RPQ_ELABEL = 0, -1, -2, -3
RPQ_ENOMEM, RPQ_ECUDA, RPQ_ECAPACITY, RPQ_EUNSUPPORTED = -4, -5, -6, -7
RPQ_SYNTAX_PAPER, RPQ_NO_MINIMIZE = 1, 2
RPQ_MAX_STATES, RPQ_MAX_TRANSITIONS, RPQ_MAX_QUERY_LABELS = 64, 256, 32
RPQ_COUNT, RPQ_PAIRS, RPQ_PER_SOURCE, RPQ_STATS, RPQ_TIME_KERNELS = 1, 2, 4, 8, 16
RPQ_PE, RPQ_SOURCE_PE, RPQ_BOUNDED, RPQ_WCOJ = 32, 64, 128, 256
RPQ_GRAPH_IN_EDGES = 1
RPQ_MAX_COLS = 16

_STATUS_NAMES = {0: "RPQ_OK", -1: "RPQ_EINVAL", -2: "RPQ_ESYNTAX", -3: "RPQ_ELABEL",
                 -4: "RPQ_ENOMEM", -5: "RPQ_ECUDA", -6: "RPQ_ECAPACITY", -7: "RPQ_EUNSUPPORTED"}


class RPQError(RuntimeError):
    def __init__(self, status: int, msg: str, offset: int = 0):
        super().__init__(f"{_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.offset = offset


# ---- ctypes structures (must mirror include/rpq.h) ---------------------------
c_u32p = ctypes.POINTER(ctypes.c_uint32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)


class rpq_graph_desc(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_uint32), ("num_edges", ctypes.c_uint64),
                ("src", c_u32p), ("dst", c_u32p), ("label", ctypes.POINTER(ctypes.c_uint16)),
                ("num_labels", ctypes.c_uint32), ("label_names", ctypes.POINTER(ctypes.c_char_p)),
                ("vertex_label", ctypes.POINTER(ctypes.c_uint16)), ("num_vertex_labels", ctypes.c_uint32),
                ("vertex_label_names", ctypes.POINTER(ctypes.c_char_p)), ("device", ctypes.c_int),
                ("flags", ctypes.c_uint32), ("cuda_stream", ctypes.c_void_p)]


class rpq_eval_opts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_uint32), ("batch_sources", ctypes.c_uint32),
                ("hbm_budget_bytes", ctypes.c_uint64), ("shard_index", ctypes.c_uint32),
                ("shard_count", ctypes.c_uint32), ("cuda_stream", ctypes.c_void_p),
                ("chunk_words", ctypes.c_uint32), ("reserved", ctypes.c_uint32),
                ("max_hops", ctypes.c_uint32), ("pad0", ctypes.c_uint32)]


class rpq_plan_info(ctypes.Structure):
    _fields_ = [("productive_sources", ctypes.c_uint64), ("batch_sources", ctypes.c_uint32),
                ("chunk_words", ctypes.c_uint32), ("num_batches", ctypes.c_uint64),
                ("state_words", ctypes.c_uint64)]


class rpq_batch_info(ctypes.Structure):
    _fields_ = [("cand_lo", ctypes.c_uint64), ("cand_hi", ctypes.c_uint64),
                ("offset", ctypes.c_uint64), ("count", ctypes.c_uint64)]


class crpq_query(ctypes.Structure):
    _fields_ = [("num_vars", ctypes.c_uint32), ("var_label", ctypes.POINTER(ctypes.c_int32)),
                ("var_const", ctypes.POINTER(ctypes.c_int64)), ("num_atoms", ctypes.c_uint32),
                ("atom_x", c_u32p), ("atom_y", c_u32p), ("atom_nfa", ctypes.POINTER(ctypes.c_void_p)),
                ("num_distinct", ctypes.c_uint32), ("distinct_pairs", c_u32p)]


class rpq_stats(ctypes.Structure):
    _fields_ = [("count", ctypes.c_uint64), ("product_edges", ctypes.c_uint64),
                ("word_items", ctypes.c_uint64), ("word_edge_ops", ctypes.c_uint64),
                ("items", ctypes.c_uint64), ("item_edges", ctypes.c_uint64),
                ("item_transitions", ctypes.c_uint64), ("activations", ctypes.c_uint64),
                ("next_reds", ctypes.c_uint64), ("levels", ctypes.c_uint32),
                ("batches", ctypes.c_uint32), ("batch_sources", ctypes.c_uint32),
                ("chunk_words", ctypes.c_uint32), ("productive_sources", ctypes.c_uint64),
                ("state_words", ctypes.c_uint64), ("expand_launches", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("expand_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("pull_levels", ctypes.c_uint64),
                ("pull_loads", ctypes.c_uint64), ("pull_words", ctypes.c_uint64),
                ("adv_words", ctypes.c_uint64), ("adv_zero_sectors", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


# ---- prototypes ----------------------------------------------------------------
_P = ctypes.POINTER
_vp = ctypes.c_void_p
_st = ctypes.c_int


def _proto(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


EXPORTED = [
    "rpq_graph_load", "rpq_graph_free", "rpq_graph_info", "rpq_graph_label_csr",
    "rpq_compile", "rpq_compile_labels", "rpq_nfa_free", "rpq_nfa_info", "rpq_nfa_transitions",
    "rpq_nfa_accepts", "rpq_eval_allpairs", "rpq_eval_single_source", "rpq_eval_sources",
    "crpq_eval", "rpq_result_count", "rpq_result_device_view", "rpq_result_copy_host",
    "rpq_result_source_counts", "rpq_result_stats", "rpq_result_free", "rpq_last_error",
    "rpq_device_count", "rpq_version", "rpq_shard_plan", "rpq_trim_memory",
    "rpq_nfa_reverse", "rpq_eval_targets", "rpq_eval_single_target", "rpq_eval_allpairs_stream",
    "rpq_set_allocator", "rpq_plan", "rpq_result_batches", "rpq_result_source_pe",
    "rpq_graph_add_label", "rpq_cache_closure", "rpq_eval_loop_cached", "crpq_eval_project", "rpq_eval_middle",
]

_c = {}
_c["rpq_graph_load"] = _proto("rpq_graph_load", _st, [_P(rpq_graph_desc), _P(_vp)])
_c["rpq_graph_free"] = _proto("rpq_graph_free", None, [_vp])
_c["rpq_graph_info"] = _proto("rpq_graph_info", _st, [_vp, c_u32p, c_u64p, c_u32p])
_c["rpq_graph_label_csr"] = _proto("rpq_graph_label_csr", _st, [_vp, ctypes.c_uint32, _P(_vp), _P(_vp), c_u64p])
_c["rpq_compile"] = _proto("rpq_compile", _st, [_vp, ctypes.c_char_p, ctypes.c_uint32, _P(_vp), _P(ctypes.c_size_t)])
_c["rpq_compile_labels"] = _proto("rpq_compile_labels", _st, [_P(ctypes.c_char_p), ctypes.c_uint32, ctypes.c_char_p,
                                                              ctypes.c_uint32, _P(_vp), _P(ctypes.c_size_t)])
_c["rpq_nfa_free"] = _proto("rpq_nfa_free", None, [_vp])
_c["rpq_nfa_info"] = _proto("rpq_nfa_info", _st, [_vp, c_u32p, c_u32p, c_u32p, _P(ctypes.c_int), _P(ctypes.c_int)])
_c["rpq_nfa_transitions"] = _proto("rpq_nfa_transitions", _st, [_vp, c_u32p, c_u32p, c_u32p, ctypes.c_uint32,
                                                                c_u32p, c_u64p])
_c["rpq_nfa_accepts"] = _proto("rpq_nfa_accepts", _st, [_vp, c_u32p, ctypes.c_uint32, _P(ctypes.c_int)])
_c["rpq_nfa_reverse"] = _proto("rpq_nfa_reverse", _st, [_vp, _P(_vp)])
_c["rpq_eval_allpairs"] = _proto("rpq_eval_allpairs", _st, [_vp, _vp, _P(rpq_eval_opts), _P(_vp)])
_c["rpq_eval_single_source"] = _proto("rpq_eval_single_source", _st, [_vp, _vp, ctypes.c_uint32,
                                                                      _P(rpq_eval_opts), _P(_vp)])
RPQ_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
RPQ_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
_c["rpq_set_allocator"] = _proto("rpq_set_allocator", _st, [RPQ_ALLOC_FN, RPQ_FREE_FN, ctypes.c_void_p])
RPQ_PAIRS_SINK = ctypes.CFUNCTYPE(ctypes.c_int, c_u32p, c_u32p, ctypes.c_uint64, ctypes.c_void_p)
_c["rpq_eval_allpairs_stream"] = _proto("rpq_eval_allpairs_stream", _st,
                                        [_vp, _vp, _P(rpq_eval_opts), ctypes.c_uint64, ctypes.c_uint64,
                                         RPQ_PAIRS_SINK, ctypes.c_void_p, _P(ctypes.c_uint64)])
_c["rpq_eval_targets"] = _proto("rpq_eval_targets", _st, [_vp, _vp, c_u32p, ctypes.c_uint64,
                                                          _P(rpq_eval_opts), _P(_vp)])
_c["rpq_eval_single_target"] = _proto("rpq_eval_single_target", _st, [_vp, _vp, ctypes.c_uint32,
                                                                      _P(rpq_eval_opts), _P(_vp)])
_c["rpq_eval_sources"] = _proto("rpq_eval_sources", _st, [_vp, _vp, c_u32p, ctypes.c_uint64,
                                                          _P(rpq_eval_opts), _P(_vp)])
_c["crpq_eval"] = _proto("crpq_eval", _st, [_vp, _P(crpq_query), _P(rpq_eval_opts), _P(_vp)])
_c["rpq_result_count"] = _proto("rpq_result_count", ctypes.c_uint64, [_vp])
_c["rpq_result_device_view"] = _proto("rpq_result_device_view", _st, [_vp, _P(_vp), c_u32p, c_u64p])
_c["rpq_result_copy_host"] = _proto("rpq_result_copy_host", _st, [_vp, _P(c_u32p), ctypes.c_uint64, c_u64p])
_c["rpq_result_source_counts"] = _proto("rpq_result_source_counts", _st, [_vp, c_u32p, c_u64p, ctypes.c_uint64,
                                                                          c_u64p])
_c["rpq_result_stats"] = _proto("rpq_result_stats", _st, [_vp, _P(rpq_stats)])
_c["rpq_result_free"] = _proto("rpq_result_free", None, [_vp])
_c["rpq_result_batches"] = _proto("rpq_result_batches", _st, [_vp, _P(rpq_batch_info), ctypes.c_uint64, c_u64p])
_c["rpq_plan"] = _proto("rpq_plan", _st, [_vp, _vp, _P(rpq_eval_opts), _P(rpq_plan_info)])
_c["rpq_graph_add_label"] = _proto("rpq_graph_add_label", _st, [_vp, ctypes.c_char_p, _vp, _vp, ctypes.c_uint64,
                                                                ctypes.c_int, _vp, c_u32p])
_c["crpq_eval_project"] = _proto("crpq_eval_project", _st, [_vp, _P(crpq_query), c_u32p, ctypes.c_uint32,
                                                            _P(rpq_eval_opts), _P(_vp)])
_c["rpq_eval_middle"] = _proto("rpq_eval_middle", _st, [_vp, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                                        _P(rpq_eval_opts), _P(_vp)])
_c["rpq_eval_loop_cached"] = _proto("rpq_eval_loop_cached", _st, [_vp, ctypes.c_char_p, ctypes.c_char_p,
                                                                  ctypes.c_char_p, _P(rpq_eval_opts), _P(_vp)])
_c["rpq_cache_closure"] = _proto("rpq_cache_closure", _st, [_vp, _vp, ctypes.c_char_p, _P(rpq_eval_opts), c_u32p])
_c["rpq_result_source_pe"] = _proto("rpq_result_source_pe", _st, [_vp, c_u64p, ctypes.c_uint64, c_u64p])
_c["rpq_last_error"] = _proto("rpq_last_error", ctypes.c_char_p, [])
_c["rpq_device_count"] = _proto("rpq_device_count", _st, [_P(ctypes.c_int)])
_c["rpq_version"] = _proto("rpq_version", ctypes.c_char_p, [])
_c["rpq_trim_memory"] = _proto("rpq_trim_memory", _st, [ctypes.c_int])
_c["rpq_shard_plan"] = _proto("rpq_shard_plan", _st, [c_u32p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                                      ctypes.c_uint32, c_u32p])


def _check(st: int, offset: int = 0):
    if st != RPQ_OK:
        raise RPQError(st, _c["rpq_last_error"]().decode(errors="replace"), offset)


def _arr(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _names(names):
    return (ctypes.c_char_p * max(1, len(names)))(*[n.encode() for n in names])


# ---- handles -----------------------------------------------------------------
class Graph:
    """Handle of an rpq_graph (per-label device CSR)."""

    def __init__(self, handle, label_names, vertex_label_names, num_vertices):
        self.h = handle
        self.label_names = list(label_names)
        self.vertex_label_names = list(vertex_label_names)
        self.num_vertices = num_vertices

    def __del__(self):
        if getattr(self, "h", None) and _c:
            _c["rpq_graph_free"](self.h)
            self.h = None


class Nfa:
    """Handle of an rpq_nfa (minimal trim DFA or Glushkov NFA)."""

    def __init__(self, handle):
        self.h = handle

    def info(self) -> dict:
        nq, nt, nf = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        ae, dfa = ctypes.c_int(), ctypes.c_int()
        _check(_c["rpq_nfa_info"](self.h, ctypes.byref(nq), ctypes.byref(nt), ctypes.byref(nf),
                                  ctypes.byref(ae), ctypes.byref(dfa)))
        return {"states": nq.value, "transitions": nt.value, "finals": nf.value,
                "accepts_empty": bool(ae.value), "is_dfa": bool(dfa.value)}

    def transitions(self):
        n = ctypes.c_uint32()
        fm = ctypes.c_uint64()
        _check(_c["rpq_nfa_transitions"](self.h, None, None, None, 0, ctypes.byref(n), ctypes.byref(fm)))
        k = n.value
        f, l, t = (np.zeros(max(k, 1), np.uint32) for _ in range(3))
        _check(_c["rpq_nfa_transitions"](self.h, _ptr(f, ctypes.c_uint32), _ptr(l, ctypes.c_uint32),
                                         _ptr(t, ctypes.c_uint32), k, ctypes.byref(n), ctypes.byref(fm)))
        finals = [q for q in range(64) if (fm.value >> q) & 1]
        return list(zip(f[:k].tolist(), l[:k].tolist(), t[:k].tolist())), finals

    def accepts(self, word: Sequence[int]) -> bool:
        w = _arr(word if len(word) else [0], np.uint32)
        acc = ctypes.c_int()
        _check(_c["rpq_nfa_accepts"](self.h, _ptr(w, ctypes.c_uint32), len(word), ctypes.byref(acc)))
        return bool(acc.value)

    def __del__(self):
        if getattr(self, "h", None) and _c:
            _c["rpq_nfa_free"](self.h)
            self.h = None


class Result:
    """Handle of an rpq_result (device-resident rows, counts, stats)."""

    def __init__(self, handle):
        self.h = handle

    @property
    def count(self) -> int:
        return int(_c["rpq_result_count"](self.h))

    def stats(self) -> dict:
        s = rpq_stats()
        _check(_c["rpq_result_stats"](self.h, ctypes.byref(s)))
        return s.as_dict()

    def device_view(self):
        cols = (ctypes.c_void_p * RPQ_MAX_COLS)()
        nc, n = ctypes.c_uint32(), ctypes.c_uint64()
        _check(_c["rpq_result_device_view"](self.h, cols, ctypes.byref(nc), ctypes.byref(n)))
        return [cols[i] for i in range(nc.value)], n.value

    def rows(self) -> np.ndarray:
        """Host copy of the rows as an (n, ncols) uint32 array."""
        ptrs, n = self.device_view()
        nc = len(ptrs)
        bufs = [np.zeros(max(n, 1), np.uint32) for _ in range(nc)]
        arr = (c_u32p * max(nc, 1))(*[_ptr(b, ctypes.c_uint32) for b in bufs])
        got = ctypes.c_uint64()
        _check(_c["rpq_result_copy_host"](self.h, arr, n, ctypes.byref(got)))
        return np.stack([b[:n] for b in bufs], axis=1) if nc else np.zeros((0, 0), np.uint32)

    def source_counts(self):
        n = ctypes.c_uint64()
        st = _c["rpq_result_source_counts"](self.h, None, None, 0, ctypes.byref(n))
        if st not in (RPQ_OK, RPQ_ECAPACITY):
            _check(st)
        k = n.value
        s = np.zeros(max(k, 1), np.uint32)
        c = np.zeros(max(k, 1), np.uint64)
        _check(_c["rpq_result_source_counts"](self.h, _ptr(s, ctypes.c_uint32), _ptr(c, ctypes.c_uint64), k,
                                              ctypes.byref(n)))
        return s[:k], c[:k]

    def source_pe(self) -> np.ndarray:
        """Per-source PE (RPQ_PER_SOURCE | RPQ_SOURCE_PE), aligned with source_counts()."""
        n = ctypes.c_uint64()
        st = _c["rpq_result_source_pe"](self.h, None, 0, ctypes.byref(n))
        if st not in (RPQ_OK, RPQ_ECAPACITY):
            _check(st)
        k = n.value
        pe = np.zeros(max(k, 1), np.uint64)
        _check(_c["rpq_result_source_pe"](self.h, _ptr(pe, ctypes.c_uint64), k, ctypes.byref(n)))
        return pe[:k]

    def batches(self) -> np.ndarray:
        """(k, 4) uint64 rows (cand_lo, cand_hi, offset, count) of this
        shard's batches (PAIRS results; see rpq_result_batches)."""
        n = ctypes.c_uint64()
        st = _c["rpq_result_batches"](self.h, None, 0, ctypes.byref(n))
        if st not in (RPQ_OK, RPQ_ECAPACITY):
            _check(st)
        k = n.value
        buf = (rpq_batch_info * max(k, 1))()
        _check(_c["rpq_result_batches"](self.h, buf, k, ctypes.byref(n)))
        return np.array([[b.cand_lo, b.cand_hi, b.offset, b.count] for b in buf[:k]], np.uint64).reshape(k, 4)

    def __del__(self):
        if getattr(self, "h", None) and _c:
            _c["rpq_result_free"](self.h)
            self.h = None


# ---- the C-ABI calls -----------------------------------------------------------
def rpq_device_count() -> int:
    n = ctypes.c_int()
    _check(_c["rpq_device_count"](ctypes.byref(n)))
    return n.value


def rpq_version() -> str:
    return _c["rpq_version"]().decode()


# every allocator ever installed stays referenced: graphs and results free
# their buffers through the allocator that allocated them, which may have
# been replaced (or removed) since
_allocator_refs = []


def rpq_set_allocator(alloc=None, free=None) -> None:
    """alloc(nbytes, stream) -> device pointer (int), free(ptr, stream);
    both None restores the library's stream-ordered pool.  Example (PyTorch's
    caching allocator): alloc=lambda n, s: torch.cuda.caching_allocator_alloc(n, stream=s),
    free=lambda p, s: torch.cuda.caching_allocator_delete(p)."""
    if alloc is None and free is None:
        _check(_c["rpq_set_allocator"](RPQ_ALLOC_FN(), RPQ_FREE_FN(), None))
        return
    fa = RPQ_ALLOC_FN(lambda n, s, _ctx: alloc(int(n), s or 0) or None)
    ff = RPQ_FREE_FN(lambda p, s, _ctx: free(p, s or 0))
    _allocator_refs.append((fa, ff))      # keep the thunks alive for good
    _check(_c["rpq_set_allocator"](fa, ff, None))


def rpq_trim_memory(device: int = 0) -> None:
    """Return the library's cached (pooled, unused) device memory to the driver."""
    _check(_c["rpq_trim_memory"](device))


def rpq_shard_plan(productive_idx, num_candidates: int, batch_sources: int, shard_count: int) -> np.ndarray:
    """Owner shard of every candidate source (host-only, see include/rpq.h)."""
    p = _arr(productive_idx if len(productive_idx) else [0], np.uint32)
    owner = np.zeros(max(1, num_candidates), np.uint32)
    _check(_c["rpq_shard_plan"](_ptr(p, ctypes.c_uint32), len(productive_idx), num_candidates, batch_sources,
                                shard_count, _ptr(owner, ctypes.c_uint32)))
    return owner[:num_candidates]


def rpq_last_error() -> str:
    return _c["rpq_last_error"]().decode(errors="replace")


def rpq_graph_load(graph=None, *, num_vertices=None, src=None, dst=None, label=None, label_names=None,
                   vertex_label=None, vertex_label_names=None, device: int = 0, stream=None,
                   in_edges: bool = False) -> Graph:
    """Load a graph (anything with num_vertices/src/dst/label/label_names, or
    the arrays as keywords) into a per-label device CSR (plus the in-edge CSR
    with in_edges=True: RPQ_GRAPH_IN_EDGES)."""
    if graph is not None:
        num_vertices, src, dst, label = graph.num_vertices, graph.src, graph.dst, graph.label
        label_names = graph.label_names
        vertex_label = getattr(graph, "vertex_label", None)
        vertex_label_names = getattr(graph, "vertex_label_names", None)
    src = _arr(src, np.uint32)
    dst = _arr(dst, np.uint32)
    label = _arr(label, np.uint16)
    d = rpq_graph_desc()
    d.num_vertices = int(num_vertices)
    d.num_edges = int(src.size)
    d.src = _ptr(src, ctypes.c_uint32)
    d.dst = _ptr(dst, ctypes.c_uint32)
    d.label = _ptr(label, ctypes.c_uint16)
    names = _names(label_names)
    d.num_labels = len(label_names)
    d.label_names = names
    vnames = None
    if vertex_label is not None:
        vl = _arr(vertex_label, np.uint16)
        d.vertex_label = _ptr(vl, ctypes.c_uint16)
        vnames = _names(vertex_label_names or [])
        d.num_vertex_labels = len(vertex_label_names or [])
        d.vertex_label_names = vnames
    d.device = device
    d.cuda_stream = stream
    d.flags = RPQ_GRAPH_IN_EDGES if in_edges else 0
    h = ctypes.c_void_p()
    _check(_c["rpq_graph_load"](ctypes.byref(d), ctypes.byref(h)))
    return Graph(h.value, label_names, vertex_label_names or [], int(num_vertices))


def rpq_graph_add_label(g: Graph, name: str, src, dst, stream=None) -> int:
    """Add a derived edge label from host (src, dst) arrays; returns its id."""
    a = _arr(src if len(src) else [0], np.uint32)
    b = _arr(dst if len(dst) else [0], np.uint32)
    lid = ctypes.c_uint32()
    _check(_c["rpq_graph_add_label"](g.h, name.encode(), a.ctypes.data, b.ctypes.data, len(src), 0, stream,
                                     ctypes.byref(lid)))
    g.label_names.append(name)
    return lid.value


def rpq_cache_closure(g: Graph, inner: Nfa, name: str, opts: Optional[rpq_eval_opts] = None, **kw) -> int:
    """Install R(inner) as the derived label `name` (loop-cache plan)."""
    o = opts if opts is not None else make_opts(**kw)
    lid = ctypes.c_uint32()
    _check(_c["rpq_cache_closure"](g.h, inner.h, name.encode(), ctypes.byref(o), ctypes.byref(lid)))
    g.label_names.append(name)
    return lid.value


def rpq_eval_loop_cached(g: Graph, prefix: str, loop: str, suffix: str,
                         opts: Optional[rpq_eval_opts] = None, **kw) -> Result:
    """All-pairs R(prefix (loop)* suffix) with the loop-cache plan (WavePlan
    A2; see include/rpq.h).  Same pairs as the direct plan."""
    o = opts if opts is not None else make_opts(**kw)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_loop_cached"](g.h, (prefix or "").encode(), loop.encode(), (suffix or "").encode(),
                                      ctypes.byref(o), ctypes.byref(h)))
    return Result(h.value)


def rpq_graph_info(g: Graph):
    nv, ne, nl = ctypes.c_uint32(), ctypes.c_uint64(), ctypes.c_uint32()
    _check(_c["rpq_graph_info"](g.h, ctypes.byref(nv), ctypes.byref(ne), ctypes.byref(nl)))
    return {"num_vertices": nv.value, "num_edges": ne.value, "num_labels": nl.value}


def rpq_graph_label_csr(g: Graph, label: int):
    off, nbr, m = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_uint64()
    _check(_c["rpq_graph_label_csr"](g.h, label, ctypes.byref(off), ctypes.byref(nbr), ctypes.byref(m)))
    return off.value, nbr.value, m.value


def rpq_compile(g: Graph, regex: str, flags: int = 0) -> Nfa:
    h = ctypes.c_void_p()
    off = ctypes.c_size_t()
    st = _c["rpq_compile"](g.h, regex.encode(), flags, ctypes.byref(h), ctypes.byref(off))
    _check(st, off.value)
    return Nfa(h.value)


def rpq_nfa_reverse(a: Nfa) -> Nfa:
    """Automaton of the reversed language."""
    h = ctypes.c_void_p()
    _check(_c["rpq_nfa_reverse"](a.h, ctypes.byref(h)))
    return Nfa(h.value)


def rpq_compile_labels(label_names: Sequence[str], regex: str, flags: int = 0) -> Nfa:
    h = ctypes.c_void_p()
    off = ctypes.c_size_t()
    st = _c["rpq_compile_labels"](_names(label_names), len(label_names), regex.encode(), flags,
                                  ctypes.byref(h), ctypes.byref(off))
    _check(st, off.value)
    return Nfa(h.value)


def make_opts(mode: int = RPQ_COUNT, batch_sources: int = 0, hbm_budget_bytes: int = 0, shard_index: int = 0,
              shard_count: int = 1, stream=None, chunk_words: int = 0, max_hops: Optional[int] = None) -> rpq_eval_opts:
    """max_hops=k (not None) sets RPQ_BOUNDED: paths of length <= k only."""
    o = rpq_eval_opts()
    if max_hops is not None:
        mode |= RPQ_BOUNDED
        o.max_hops = int(max_hops)
    o.mode, o.batch_sources, o.hbm_budget_bytes = mode, batch_sources, hbm_budget_bytes
    o.shard_index, o.shard_count, o.cuda_stream, o.chunk_words = shard_index, shard_count, stream, chunk_words
    return o


def rpq_eval_allpairs(g: Graph, a: Nfa, opts: Optional[rpq_eval_opts] = None, **kw) -> Result:
    o = opts if opts is not None else make_opts(**kw)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_allpairs"](g.h, a.h, ctypes.byref(o), ctypes.byref(h)))
    return Result(h.value)


def rpq_plan(g: Graph, a: Nfa, opts: Optional[rpq_eval_opts] = None, **kw) -> dict:
    """Batch plan of rpq_eval_allpairs under these options (nothing evaluated)."""
    o = opts if opts is not None else make_opts(**kw)
    info = rpq_plan_info()
    _check(_c["rpq_plan"](g.h, a.h, ctypes.byref(o), ctypes.byref(info)))
    return {k: getattr(info, k) for k, _ in info._fields_}


def rpq_result_batches(r: Result) -> np.ndarray:
    return r.batches()


def rpq_result_source_pe(r: Result) -> np.ndarray:
    return r.source_pe()


def rpq_eval_single_source(g: Graph, a: Nfa, src: int, opts: Optional[rpq_eval_opts] = None, **kw) -> Result:
    o = opts if opts is not None else make_opts(**kw)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_single_source"](g.h, a.h, int(src), ctypes.byref(o), ctypes.byref(h)))
    return Result(h.value)


def rpq_eval_sources(g: Graph, a: Nfa, sources, opts: Optional[rpq_eval_opts] = None, **kw) -> Result:
    o = opts if opts is not None else make_opts(**kw)
    s = _arr(sources if len(sources) else [0], np.uint32)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_sources"](g.h, a.h, _ptr(s, ctypes.c_uint32), len(sources), ctypes.byref(o),
                                  ctypes.byref(h)))
    return Result(h.value)


def rpq_eval_allpairs_stream(g: Graph, a: Nfa, sink=None, device_budget_bytes: int = 0, piece_pairs: int = 0,
                             opts: Optional[rpq_eval_opts] = None, **kw):
    """All-pairs result streamed to the host in (src, dst) order.  sink(src,
    dst) receives numpy views valid during the call (return True to stop);
    without a sink the pieces are collected and returned as an (n, 2) array.
    Returns (total pairs delivered, collected array or None)."""
    o = opts if opts is not None else make_opts(**kw)
    pieces = []

    def _cb(ps, pd, n, _ctx):
        src = np.ctypeslib.as_array(ps, (n,)) if n else np.zeros(0, np.uint32)
        dst = np.ctypeslib.as_array(pd, (n,)) if n else np.zeros(0, np.uint32)
        if sink is None:
            pieces.append(np.stack([src.copy(), dst.copy()], 1))
            return 0
        return 1 if sink(src, dst) else 0

    cb = RPQ_PAIRS_SINK(_cb)
    tot = ctypes.c_uint64()
    _check(_c["rpq_eval_allpairs_stream"](g.h, a.h, ctypes.byref(o), int(device_budget_bytes), int(piece_pairs), cb,
                                          None, ctypes.byref(tot)))
    if sink is None:
        return tot.value, (np.concatenate(pieces) if pieces else np.zeros((0, 2), np.uint32))
    return tot.value, None


def rpq_eval_targets(g: Graph, a: Nfa, targets, opts: Optional[rpq_eval_opts] = None, **kw) -> Result:
    """(x, t) pairs for the given targets (rows sorted by (t, x)); the graph
    needs in_edges=True."""
    o = opts if opts is not None else make_opts(**kw)
    t = _arr(targets if len(targets) else [0], np.uint32)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_targets"](g.h, a.h, _ptr(t, ctypes.c_uint32), len(targets), ctypes.byref(o),
                                  ctypes.byref(h)))
    return Result(h.value)


def rpq_eval_single_target(g: Graph, a: Nfa, t: int, opts: Optional[rpq_eval_opts] = None, **kw) -> Result:
    o = opts if opts is not None else make_opts(**kw)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_single_target"](g.h, a.h, int(t), ctypes.byref(o), ctypes.byref(h)))
    return Result(h.value)


def rpq_eval_middle(g: Graph, alpha: str, mid: str, beta: str, opts: Optional[rpq_eval_opts] = None,
                    **kw) -> Result:
    """Start-in-the-middle plan for R(alpha mid beta) (see include/rpq.h)."""
    o = opts if opts is not None else make_opts(**kw)
    h = ctypes.c_void_p()
    _check(_c["rpq_eval_middle"](g.h, alpha.encode(), mid.encode(), beta.encode(), ctypes.byref(o),
                                 ctypes.byref(h)))
    return Result(h.value)


def crpq_eval(g: Graph, var_label, var_const, atoms, distinct=(), opts: Optional[rpq_eval_opts] = None,
              out_vars=None, **kw) -> Result:
    """var_label/var_const: per variable (-1 = any / free); atoms: list of
    (x, Nfa, y) with variable indices; distinct: list of (var, var)."""
    o = opts if opts is not None else make_opts(**kw)
    nv = len(var_label)
    vl = _arr(var_label, np.int32)
    vc = _arr(var_const, np.int64)
    ax = _arr([a[0] for a in atoms] or [0], np.uint32)
    ay = _arr([a[2] for a in atoms] or [0], np.uint32)
    an = (ctypes.c_void_p * max(1, len(atoms)))(*[a[1].h for a in atoms])
    dp = _arr([x for p in distinct for x in p] or [0], np.uint32)
    q = crpq_query()
    q.num_vars = nv
    q.var_label = _ptr(vl, ctypes.c_int32)
    q.var_const = _ptr(vc, ctypes.c_int64)
    q.num_atoms = len(atoms)
    q.atom_x = _ptr(ax, ctypes.c_uint32)
    q.atom_y = _ptr(ay, ctypes.c_uint32)
    q.atom_nfa = an
    q.num_distinct = len(distinct)
    q.distinct_pairs = _ptr(dp, ctypes.c_uint32)
    h = ctypes.c_void_p()
    if out_vars is None:
        _check(_c["crpq_eval"](g.h, ctypes.byref(q), ctypes.byref(o), ctypes.byref(h)))
    else:
        ov = _arr(list(out_vars) or [0], np.uint32)
        _check(_c["crpq_eval_project"](g.h, ctypes.byref(q), _ptr(ov, ctypes.c_uint32), len(out_vars),
                                       ctypes.byref(o), ctypes.byref(h)))
    return Result(h.value)


def rpq_result_count(r: Result) -> int:
    return r.count


def rpq_result_stats(r: Result) -> dict:
    return r.stats()


def rpq_result_copy_host(r: Result) -> np.ndarray:
    return r.rows()


def rpq_result_source_counts(r: Result):
    return r.source_counts()


def rpq_result_device_view(r: Result):
    return r.device_view()


def crpq(g: Graph, vars, atoms, var_label=None, var_const=None, distinct=(), project=None, **kw) -> Result:
    """Convenience marshalling for crpq_eval: vars = names; atoms = (x, regex,
    y) with variable names; var_label = {var: vertex-label name};
    var_const = {var: vertex id}; distinct = [(var, var)]."""
    idx = {v: i for i, v in enumerate(vars)}
    vl = [-1] * len(vars)
    for v, name in (var_label or {}).items():
        vl[idx[v]] = g.vertex_label_names.index(name)
    vc = [-1] * len(vars)
    for v, c in (var_const or {}).items():
        vc[idx[v]] = int(c)
    at = [(idx[x], rpq_compile(g, rx), idx[y]) for (x, rx, y) in atoms]
    ov = None if project is None else [idx[v] for v in project]
    return crpq_eval(g, vl, vc, at, [(idx[a], idx[b]) for a, b in distinct], out_vars=ov, **kw)
