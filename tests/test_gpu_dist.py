"""The product's multi-GPU path (paper_2602_20748_b200.dist) on one GPU:
two ranks (processes) share cuda:0 over gloo, each evaluates its batches
through the C-ABI and the results are gathered.
Checked against O1: the global count, PE, per-source counts and the pair
set gathered to rank 0 in (src, dst) order; gather="shard" offsets tile the
same result."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

R = pytest.importorskip("paper_2602_20748_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


GRAPH = dict(num_vertices=8000, num_edges=32000, num_labels=3, seed=41)


def _worker(rank, world, port, rx, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2602_20748_b200 import dist as D
    g = synth.random_graph(GRAPH["num_vertices"], GRAPH["num_edges"], GRAPH["num_labels"], seed=GRAPH["seed"])
    G = R.rpq_graph_load(g)
    a = R.rpq_compile(G, rx)
    out = {}
    # auto B agreed by all-reduce MIN; a small budget forces several batches
    c = D.rpq_eval_allpairs_dist(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, hbm_budget_bytes=64 << 20)
    out["count"], out["pe"], out["B"] = c.count, c.stats["product_edges"], c.batch_sources
    p = D.rpq_eval_allpairs_dist(G, a, mode=R.RPQ_PAIRS, batch_sources=1024)
    out["ps"] = (p.sources, p.source_counts)
    out["nbatches_local"] = len(p.local.batches())
    if rank == 0:
        out["pairs"] = p.rows()
    sh = D.rpq_eval_allpairs_dist(G, a, mode=R.RPQ_PAIRS, batch_sources=1024, gather="shard")
    rows = sh.local.rows()
    pieces = [(goff, rows[off:off + n]) for (off, goff, n) in sh.offsets]
    allp = [None] * world
    dist.all_gather_object(allp, pieces)
    if rank == 0:
        out["shard_pieces"] = [x for lst in allp for x in lst]
        out_q.put(out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("rx", ["(a|b)*c*", "a b* c"])
def test_two_ranks_one_gpu(rx):
    import torch.multiprocessing as mp
    if R.rpq_device_count() == 0:
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rx, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = synth.random_graph(GRAPH["num_vertices"], GRAPH["num_edges"], GRAPH["num_labels"], seed=GRAPH["seed"])
    o = oracle.allpairs(g, rx)
    want = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    want = want[np.lexsort((want[:, 1], want[:, 0]))]
    assert out["count"] == len(want)
    assert out["pe"] == int(o["pe"].sum())
    assert out["B"] % 64 == 0 and out["B"] >= 64
    s, c = out["ps"]
    nz = o["counts"] > 0
    assert np.array_equal(s, np.nonzero(nz)[0]) and np.array_equal(c, o["counts"][nz])
    assert np.array_equal(out["pairs"], want)
    pieces = sorted(out["shard_pieces"], key=lambda x: x[0])
    got = np.concatenate([x[1] for x in pieces]) if pieces else np.zeros((0, 2), np.uint32)
    assert np.array_equal(got, want)
    assert [x[0] for x in pieces] == list(np.cumsum([0] + [len(x[1]) for x in pieces[:-1]]))
