"""Phase breakdown of a single-target evaluation on the cfg3 graph (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, synth
g = synth.ldbc_graph(1.0)
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s, in_edges=True)
a = R.rpq_compile(G, "hasTag")
for i in range(3):
    if i == 2:
        os.environ["RPQ_DEBUG_EVENTS"] = "1"; os.environ["RPQ_DEBUG_HOST"] = "1"
    r = R.rpq_eval_single_target(G, a, g.meta["sports"], mode=R.RPQ_PAIRS, stream=s)
    torch.cuda.synchronize()
    print(r.count, r.stats()["total_ms"], r.stats()["batches"], r.stats()["batch_sources"], flush=True)
