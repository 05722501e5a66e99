"""One cfg2 evaluation for ncu capture (development aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, synth
rx = sys.argv[1] if len(sys.argv) > 1 else "a*"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = synth.uniform_graph()
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, rx)
r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, batch_sources=B, stream=s)
torch.cuda.synchronize()
print(rx, r.count, r.stats()["levels"])
