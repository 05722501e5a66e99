"""One COUNT evaluation of each query of a bench workload, for ncu captures
(development aid).  python scripts/prof_workload.py cfg2|cfg3|cfg5 [SHARDS]
(shard 0 of SHARDS; cfg5 defaults to 64 to bound the capture time)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
shards = int(sys.argv[2]) if len(sys.argv) > 2 else (64 if wl == "cfg5" else 1)
g = bench.make_graph(wl)
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
for rx in bench.WORKLOADS[wl]["queries"]:
    a = R.rpq_compile(G, rx)
    mode = R.RPQ_COUNT if os.environ.get("PROF_NOSTATS") else R.RPQ_COUNT | R.RPQ_STATS
    if os.environ.get("PROF_PAIRS"):
        mode = R.RPQ_PAIRS
    B = R.rpq_plan(G, a, stream=s, shard_count=shards)["batch_sources"] if shards > 1 else 0
    r = R.rpq_eval_allpairs(G, a, mode=mode, stream=s, shard_index=0, shard_count=shards, batch_sources=B)
    torch.cuda.synchronize()
    st = r.stats()
    print(wl, rx, r.count, st["levels"], st["batches"], st["batch_sources"], flush=True)
