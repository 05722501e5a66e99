"""Whole RMAT-24 (a|b)*c* all-pairs on one GPU, and the sum of its 16 shards
(consistency evidence for the north-star configuration; development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, bench
g = bench.make_graph("cfg5")
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, "(a|b)*c*")
torch.cuda.synchronize(); t = time.perf_counter()
r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=s)
torch.cuda.synchronize(); dt = time.perf_counter() - t
st = r.stats()
print(f"whole: count={r.count} PE={st['product_edges']} batches={st['batches']} B={st['batch_sources']} "
      f"time={dt:.1f}s (STATS on) PE/s={st['product_edges']/dt:.3e}", flush=True)
B = st["batch_sources"]
tot, pe = 0, 0
t = time.perf_counter()
for i in range(16):
    ri = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=s, batch_sources=B, shard_index=i, shard_count=16)
    tot += ri.count
    pe += ri.stats()["product_edges"]
torch.cuda.synchronize()
print(f"16 shards: count={tot} PE={pe} equal={tot == r.count and pe == st['product_edges']} time={time.perf_counter()-t:.1f}s",
      flush=True)
