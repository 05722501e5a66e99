"""cfg2 evaluations for ncu capture (development aid): one COUNT-mode
all-pairs evaluation per query (default: the three cfg2 queries)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, synth
queries = sys.argv[1].split(",") if len(sys.argv) > 1 else ["a*", "(a|b)*c", "a b* c"]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = synth.uniform_graph()
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
for rx in queries:
    a = R.rpq_compile(G, rx)
    mode = R.RPQ_COUNT if os.environ.get("PROF_NOSTATS") else R.RPQ_COUNT | R.RPQ_STATS
    r = R.rpq_eval_allpairs(G, a, mode=mode, batch_sources=B, stream=s)
    torch.cuda.synchronize()
    st = r.stats()
    print(rx, r.count, st["levels"], st["product_edges"], st["word_items"], st["item_transitions"],
          st["item_edges"], st["word_edge_ops"], st["expand_launches"], flush=True)
