"""Multi-GPU evaluation: source batches sharded over ranks, results gathered
with torch.distributed (NCCL over NVLink on a GPU node, gloo for tests).

PAPER.md P:1532-1535: cuRPQ "executes batches of base-TGs concurrently across
multiple GPUs" and scales almost linearly.  Here: the
productive sources are cut into batches of B consecutive sources, batch b is
evaluated by rank b % world on that rank's replica of the graph (built
locally, no broadcast), and a batch's visited set is private, so the
traversal itself has no collective.  The only exchanges are this module's
gathers, after the kernels:

  1. B: every rank plans (rpq_plan) and the ranks agree on the MIN, so that
     "batch b" is the same set of sources everywhere;
  2. COUNT: all-reduce SUM of the per-rank totals (and of the RPQ_STATS
     counters: product edges traversed etc.; MAX for times / levels);
  3. PER_SOURCE: all-gather of the (source, count) lists -> every rank gets
     the global list, ascending source;
  4. PAIRS: each rank's rows are its batches' blocks in order; all ranks'
     batches sorted by first source tile the globally (src, dst)-sorted
     result (rpq_result_batches), so rank 0 receives every rank's rows with
     one point-to-point transfer per rank and copies the blocks to their
     global offsets (gather="rank0"), or each rank keeps its rows and learns
     their global offsets (gather="shard", SURVEY §8(e)'s default for
     outputs beyond one GPU's HBM).

Argument marshalling and collectives only; every step of the evaluation runs
in librpq.so.  Without an initialised process group the call is the plain
single-GPU evaluation.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import (RPQ_COUNT, RPQ_PAIRS, RPQ_PER_SOURCE, RPQ_STATS, Graph, Nfa, Result, rpq_eval_allpairs,
               rpq_plan)

# stats fields reduced with MAX over ranks (the rest are summed)
_STAT_MAX = {"levels", "batch_sources", "chunk_words", "productive_sources", "state_words", "expand_ms",
             "total_ms"}


def _world(group):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def _coll_device(group):
    """Tensors for collectives live on the GPU for NCCL, on the host for gloo."""
    import torch
    import torch.distributed as dist
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")


def agree_batch_sources(local_b: int, group=None) -> int:
    """All-reduce MIN of the per-rank batch widths (a whole number of words)."""
    import torch
    import torch.distributed as dist
    rank, world = _world(group)
    if world == 1:
        return int(local_b)
    t = torch.tensor([int(local_b)], dtype=torch.int64, device=_coll_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


def allgather_var(arr: np.ndarray, group=None) -> List[np.ndarray]:
    """Gather a variable-length 1-D (or (k, c)) numpy array from every rank;
    returns the list of per-rank arrays on every rank."""
    import torch
    import torch.distributed as dist
    rank, world = _world(group)
    if world == 1:
        return [arr]
    dev = _coll_device(group)
    a = np.ascontiguousarray(arr)
    tail = a.shape[1:]
    n = torch.tensor([a.shape[0]], dtype=torch.int64, device=dev)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    ns = [int(x.item()) for x in ns]
    m = max(max(ns), 1)
    raw = a.view(np.uint8).reshape(a.shape[0], -1) if a.size else np.zeros((0, a.dtype.itemsize * int(np.prod(tail) or 1)), np.uint8)
    row = raw.shape[1]
    pad = np.zeros((m, row), np.uint8)
    pad[:raw.shape[0]] = raw
    t = torch.from_numpy(pad).to(dev)
    outs = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    res = []
    for k, o in enumerate(outs):
        b = o.cpu().numpy()[:ns[k]].copy()
        res.append(b.view(a.dtype).reshape((ns[k],) + tail))
    return res


def placement(tables: List[np.ndarray]):
    """Global placement of every rank's batch blocks.

    tables[r]: (k, 4) uint64 rows (cand_lo, cand_hi, offset, count) of rank
    r's batches in its own row order.  Batches of all ranks cover disjoint
    candidate intervals; sorted by cand_lo they tile the global sorted result.
    Returns (total rows, list of (rank, local_offset, global_offset, count))
    in global order."""
    rows = []
    for r, t in enumerate(tables):
        for lo, hi, off, cnt in np.asarray(t, np.uint64).reshape(-1, 4).tolist():
            rows.append((int(lo), int(hi), r, int(off), int(cnt)))
    rows.sort()
    out, g = [], 0
    for k, (lo, hi, r, off, cnt) in enumerate(rows):
        if k and lo < rows[k - 1][1]:
            raise ValueError("overlapping batches across ranks: the ranks did not use the same batch plan")
        out.append((r, off, g, cnt))
        g += cnt
    return g, out


def gather_rows_to_root(local, table: np.ndarray, group=None, root: int = 0):
    """Rank `root` receives every rank's rows (a (c, n) integer tensor, its
    batches' blocks in order) and returns them in global order as a (c,
    total) tensor on its own device; other ranks return None.  One transfer
    per rank (NCCL send/recv over NVLink, or gloo on the host)."""
    import torch
    import torch.distributed as dist
    rank, world = _world(group)
    tables = allgather_var(np.asarray(table, np.uint64).reshape(-1, 4), group)
    total, place = placement(tables)
    if world == 1:
        return local
    dev = _coll_device(group)
    counts = [int(t[:, 3].sum()) if t.size else 0 for t in tables]
    c = local.shape[0]
    if rank != root:
        if counts[rank]:
            dist.send(local.to(dev).contiguous(), dst=root, group=group)
        return None
    out = torch.empty((c, total), dtype=local.dtype, device=local.device)
    bufs = {root: local}
    for r in range(world):
        if r == root or not counts[r]:
            continue
        t = torch.empty((c, counts[r]), dtype=local.dtype, device=dev)
        dist.recv(t, src=r, group=group)
        bufs[r] = t.to(local.device)
    for r, off, goff, cnt in place:
        if cnt:
            out[:, goff:goff + cnt].copy_(bufs[r][:, off:off + cnt])
    return out


class _CudaBuf:
    """Zero-copy __cuda_array_interface__ view of a result column."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (int(ptr or 0), False),
                                         "version": 2, "strides": None}


def result_columns(r: Result):
    """(ncols, n) int32 CUDA tensor (u32 bit patterns) viewing r's rows
    (valid while r lives; no copy)."""
    import torch
    ptrs, n = r.device_view()
    if n == 0:
        return torch.zeros((len(ptrs), 0), dtype=torch.int32, device="cuda")
    return torch.stack([torch.as_tensor(_CudaBuf(p, n), device="cuda") for p in ptrs])


@dataclass
class DistResult:
    count: int                                  # |R| over all ranks
    stats: dict                                 # RPQ_STATS counters summed (MAX for times/levels)
    batch_sources: int                          # the B every rank used
    local: Optional[Result] = None              # this rank's shard (its batches)
    sources: Optional[np.ndarray] = None        # PER_SOURCE: global ascending sources ...
    source_counts: Optional[np.ndarray] = None  # ... and their counts
    pairs: Optional[object] = None              # PAIRS, gather="rank0": (2, n) int32 tensor on rank 0
    offsets: Optional[List[tuple]] = field(default=None)   # gather="shard": (local_off, global_off, count)

    def rows(self) -> np.ndarray:
        """(n, 2) uint32 host copy of the gathered pairs (rank 0)."""
        return self.pairs.cpu().numpy().view(np.uint32).T.copy()


def rpq_eval_allpairs_dist(g: Graph, a: Nfa, *, group=None, mode: int = RPQ_COUNT, stream=None,
                           batch_sources: int = 0, hbm_budget_bytes: int = 0, gather: str = "rank0",
                           chunk_words: int = 0) -> DistResult:
    """All-pairs RPQ over every rank of `group` (one process per GPU): each
    rank evaluates batches b % world == rank of the same batch plan and the
    results are gathered as described in the module docstring."""
    import torch
    import torch.distributed as dist
    if gather not in ("rank0", "shard"):
        raise ValueError("gather must be 'rank0' or 'shard'")
    rank, world = _world(group)
    if batch_sources == 0 and world > 1:
        plan = rpq_plan(g, a, mode=mode, hbm_budget_bytes=hbm_budget_bytes, shard_count=world, stream=stream)
        batch_sources = agree_batch_sources(plan["batch_sources"], group)
    r = rpq_eval_allpairs(g, a, mode=mode, batch_sources=batch_sources, hbm_budget_bytes=hbm_budget_bytes,
                          shard_index=rank, shard_count=world, stream=stream, chunk_words=chunk_words)
    st = r.stats()
    if world == 1:
        out = DistResult(count=r.count, stats=st, batch_sources=batch_sources, local=r)
        if mode & RPQ_PER_SOURCE or mode & RPQ_PAIRS:
            s, c = r.source_counts()
            out.sources, out.source_counts = s, c
        if mode & RPQ_PAIRS:
            if gather == "rank0":
                out.pairs = result_columns(r).clone()
            else:
                out.offsets = [(int(o), int(o), int(n)) for (_, _, o, n) in r.batches().tolist()]
        return out
    dev = _coll_device(group)
    keys = [k for k, v in st.items() if isinstance(v, (int, float))]
    vals = torch.tensor([float(st[k]) for k in keys] + [float(r.count)], dtype=torch.float64, device=dev)
    vmax = vals.clone()
    cnt = torch.tensor([int(r.count)], dtype=torch.int64, device=dev)
    dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(vmax, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
    stats = {k: (vmax[i].item() if k in _STAT_MAX else vals[i].item()) for i, k in enumerate(keys)}
    stats = {k: (int(v) if isinstance(st[k], int) else v) for k, v in stats.items()}
    stats["count"] = int(cnt.item())
    out = DistResult(count=int(cnt.item()), stats=stats, batch_sources=batch_sources, local=r)
    if mode & (RPQ_PER_SOURCE | RPQ_PAIRS):
        s, c = r.source_counts()
        ss = allgather_var(s.astype(np.uint32), group)
        cc = allgather_var(c.astype(np.uint64), group)
        s_all, c_all = np.concatenate(ss), np.concatenate(cc)
        order = np.argsort(s_all, kind="stable")
        out.sources, out.source_counts = s_all[order], c_all[order]
    if mode & RPQ_PAIRS:
        table = r.batches()
        if gather == "rank0":
            out.pairs = gather_rows_to_root(result_columns(r), table, group)
        else:
            tables = allgather_var(np.asarray(table, np.uint64).reshape(-1, 4), group)
            _, place = placement(tables)
            out.offsets = [(off, goff, n) for (rr, off, goff, n) in place if rr == rank]
    return out
