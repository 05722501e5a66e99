"""Multi-rank host logic on CPU (gloo, world size 2).

The multi-GPU path shards source batches round-robin over ranks (batch b ->
rank b % N); the plan is the library's own host function
`rpq_shard_plan` (the same code `rpq_eval_*` uses).  Each rank evaluates its
owned sources -- here with the CPU oracle, since there is no GPU -- and the
ranks combine counts (all_reduce SUM) and pairs (all_gather).  Checked: the
shards are disjoint, their union is the 1-rank result, the summed count is
the total.  The same sharding on the GPU is covered by
tests/test_gpu_parity.py::test_shard_union_equals_whole.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def productive(g, rx):
    """Sources with an out-edge under a label leaving the initial state of
    the automaton (from the product compiler, host-only)."""
    import paper_2602_20748_b200 as R
    a = R.rpq_compile_labels(g.label_names, rx)
    trans, _ = a.transitions()
    labels = {l for (f, l, t) in trans if f == 0}
    has = np.zeros(g.num_vertices, bool)
    for l in labels:
        has[g.src[g.label == l]] = True
    return np.nonzero(has)[0].astype(np.uint32)


def _worker(rank, world, port, rx, B, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_20748_b200 as R
    g = synth.random_graph(600, 2400, 3, seed=31)
    pidx = productive(g, rx)
    owner = R.rpq_shard_plan(pidx, g.num_vertices, B, world)
    mine = np.nonzero(owner == rank)[0].astype(np.uint32)
    og = oracle.OracleGraph(g)
    r = oracle.eval_sources(og, rx, mine, threads=2)
    cnt = torch.tensor([int(r["counts"].sum())], dtype=torch.int64)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    pairs = list(zip(r["src"].tolist(), r["dst"].tolist()))
    gathered = [None] * world
    dist.all_gather_object(gathered, pairs)
    owners = [None] * world
    dist.all_gather_object(owners, mine.tolist())
    if rank == 0:
        out_q.put((int(cnt.item()), gathered, owners))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("rx,B", [("(a|b)*c*", 64), ("a b* c", 100), ("c+", 7)])
def test_two_rank_shards_union_equals_whole(rx, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rx, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, gathered, owners = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = synth.random_graph(600, 2400, 3, seed=31)
    full = oracle.pair_set(oracle.allpairs(g, rx))
    parts = [set(map(tuple, x)) for x in gathered]
    assert parts[0].isdisjoint(parts[1])
    assert parts[0] | parts[1] == full
    assert total == len(full)
    # every source is owned by exactly one rank; both ranks got work
    o0, o1 = set(owners[0]), set(owners[1])
    assert o0.isdisjoint(o1) and len(o0 | o1) == g.num_vertices
    assert o0 and o1


def test_shard_plan_properties():
    import paper_2602_20748_b200 as R
    rng = np.random.default_rng(3)
    for _ in range(50):
        n = int(rng.integers(1, 300))
        pidx = np.sort(rng.choice(n, int(rng.integers(0, n + 1)), replace=False)).astype(np.uint32)
        B = int(rng.integers(1, 40))
        k = int(rng.integers(1, 9))
        own = R.rpq_shard_plan(pidx, n, B, k)
        nb = -(-len(pidx) // B) if len(pidx) else 0
        # batch b of P starts at P[b*B]; ownership is b % k and monotone in b
        for b in range(nb):
            assert own[pidx[b * B]] == b % k
            for j in pidx[b * B:(b + 1) * B]:
                assert own[j] == b % k
        if nb == 0:
            assert (own == 0).all()
        else:
            assert (own[:pidx[0] + 1] == 0).all()          # leading non-productive -> batch 0


def _dist_worker(rank, world, port, rx, B, out_q):
    """The product's multi-GPU gather (paper_2602_20748_b200.dist) on gloo:
    each rank holds the rows of its batches (here from the oracle: no GPU on
    this box) and its batch table; rank 0 gathers them into global order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_20748_b200 import dist as D
    g = synth.random_graph(600, 2400, 3, seed=31)
    pidx = productive(g, rx)
    nb = -(-len(pidx) // B) if len(pidx) else 1
    js = [0] + [int(pidx[k * B]) for k in range(1, nb)] + [g.num_vertices]
    og = oracle.OracleGraph(g)
    rows, table, off = [], [], 0
    for k in range(rank, nb, world):
        srcs = np.arange(js[k], js[k + 1], dtype=np.uint32)
        r = oracle.eval_sources(og, rx, srcs, threads=2)
        p = np.stack([r["src"], r["dst"]], 1).astype(np.uint32)
        p = p[np.lexsort((p[:, 1], p[:, 0]))]
        rows.append(p)
        table.append((js[k], js[k + 1], off, len(p)))
        off += len(p)
    local = np.concatenate(rows) if rows else np.zeros((0, 2), np.uint32)
    t = torch.from_numpy(local.view(np.int32).T.copy())
    agreed = D.agree_batch_sources(64 * (rank + 1))
    got = D.gather_rows_to_root(t, np.array(table, np.uint64).reshape(-1, 4))
    parts = D.allgather_var(local[:, 0].copy())
    if rank == 0:
        out_q.put((agreed, got.numpy().view(np.uint32).T.copy(), [len(x) for x in parts]))
    else:
        assert got is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("rx,B", [("(a|b)*c*", 64), ("a b* c", 100)])
def test_dist_gather_rows_in_global_order(rx, B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, 2, port, rx, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    agreed, got, sizes = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = synth.random_graph(600, 2400, 3, seed=31)
    o = oracle.allpairs(g, rx)
    want = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    want = want[np.lexsort((want[:, 1], want[:, 0]))]
    assert agreed == 64                       # all-reduce MIN of the per-rank widths
    assert np.array_equal(got, want)          # every rank's blocks at their global offsets
    assert sum(sizes) == len(want) and min(sizes) > 0


def test_dist_placement_rejects_overlap():
    from paper_2602_20748_b200 import dist as D
    tot, pl = D.placement([np.array([[0, 10, 0, 5], [20, 30, 5, 2]], np.uint64),
                           np.array([[10, 20, 0, 4]], np.uint64)])
    assert tot == 11 and pl == [(0, 0, 0, 5), (1, 0, 5, 4), (0, 5, 9, 2)]
    with pytest.raises(ValueError):
        D.placement([np.array([[0, 10, 0, 5]], np.uint64), np.array([[5, 20, 0, 4]], np.uint64)])
