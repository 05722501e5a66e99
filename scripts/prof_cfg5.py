"""cfg5 (R-MAT) evaluation for ncu capture (development aid): bench.py's
1-GPU workload, shard 0 of S (default 16), COUNT, one evaluation.
python scripts/prof_cfg5.py [SCALE] [SHARDS] [MAXBATCHES]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = synth.rmat_graph(scale, seed=24)
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, "(a|b)*c*")
mode = R.RPQ_COUNT if os.environ.get("PROF_NOSTATS") else R.RPQ_COUNT | R.RPQ_STATS
r = R.rpq_eval_allpairs(G, a, mode=mode, stream=s, shard_index=0, shard_count=shards)
torch.cuda.synchronize()
st = r.stats()
print(r.count, st["levels"], st["batches"], st["batch_sources"], st["product_edges"], st["word_items"],
      st["item_transitions"], st["item_edges"], st["word_edge_ops"], flush=True)
