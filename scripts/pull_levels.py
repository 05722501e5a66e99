"""Per-level cost of top-down vs bottom-up levels (development aid): run under
ncu --metrics gpu__time_duration.sum with RPQ_HOST_LOOP=1.
python scripts/pull_levels.py cfg2|knows|rmat20"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, synth
wl = sys.argv[1]
if wl == "cfg2":
    g, qs = synth.uniform_graph(), ["a*", "(a|b)*c"]
elif wl == "knows":
    g, qs = synth.ldbc_graph(1.0), ["knows+"]
else:
    g, qs = synth.rmat_graph(int(wl[4:]), seed=24), ["(a|b)*c*"]
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s, in_edges=True)
for rx in qs:
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, stream=s, shard_count=int(os.environ.get("SHARDS", "1")))
    torch.cuda.synchronize()
    print(rx, r.count, flush=True)
