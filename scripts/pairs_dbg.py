import os, sys
sys.path.insert(0, "/root/repo")
import torch, bench, paper_2602_20748_b200 as R
g = bench.make_graph("cfg2")
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, "a*")
for i in range(3):
    if i == 2:
        os.environ["RPQ_DEBUG_EVENTS"] = "1"; os.environ["RPQ_DEBUG_HOST"] = "1"
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS, stream=s)
    torch.cuda.synchronize()
    del r
