"""Device-side phase times (RPQ_DEBUG_EVENTS) of one cfg2 query at the per-rank
work of N ranks (shard 0 of N, batch P/N) -- development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rx = sys.argv[2] if len(sys.argv) > 2 else "a*"
g = bench.make_graph("cfg2")
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, rx)
P = R.rpq_eval_allpairs(G, a, mode=R.RPQ_STATS, stream=s).stats()["productive_sources"]
B = (-(-P // n) + 63) // 64 * 64
for i in range(4):
    if i == 3:
        os.environ["RPQ_DEBUG_EVENTS"] = "1"; os.environ["RPQ_DEBUG_HOST"] = "1"
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, stream=s, batch_sources=B, shard_count=n)
    torch.cuda.synchronize()
    st = r.stats()
    print(rx, "B", B, "total_ms %.3f loop_ms %.3f levels %d" % (st["total_ms"], st["expand_ms"], st["levels"]), flush=True)
