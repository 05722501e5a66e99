"""Device-side phase times of one COUNT evaluation per cfg2 query (RPQ_DEBUG_EVENTS=1),
at full width and as one shard of N (development aid).
python scripts/phase_times.py [SHARDS]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_20748_b200 as R, synth  # noqa: E402
shards = int(sys.argv[1]) if len(sys.argv) > 1 else 1
g = synth.uniform_graph()
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
for rx in ["a*", "(a|b)*c", "a b* c"]:
    a = R.rpq_compile(G, rx)
    B = R.rpq_plan(G, a, stream=s, shard_count=shards)["batch_sources"] if shards > 1 else 0
    for it in range(3):
        if it == 2:
            os.environ["RPQ_DEBUG_EVENTS"] = "1"
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, stream=s, batch_sources=B, shard_count=shards)
        torch.cuda.synchronize()
        os.environ.pop("RPQ_DEBUG_EVENTS", None)
    print(rx, r.count, flush=True)
