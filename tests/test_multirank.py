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
