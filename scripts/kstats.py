"""RPQ_STATS counters of the level kernel per query (cfg2; RMAT-24 1/64 of
the batches): where the bytes of a top-down level go."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "cfg2":
    g, qs, kw = synth.uniform_graph(), ["a*", "(a|b)*c", "a b* c"], {}
else:
    g, qs = synth.rmat_graph(24, seed=24), ["(a|b)*c*"]
G = R.rpq_graph_load(g)
for rx in qs:
    a = R.rpq_compile(G, rx)
    kw = {}
    if which != "cfg2":
        B = R.rpq_plan(G, a)["batch_sources"]
        kw = dict(batch_sources=B, shard_index=0, shard_count=64)
    st = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS | R.RPQ_TIME_KERNELS, **kw).stats()
    keep = ["product_edges", "word_items", "word_edge_ops", "items", "item_edges", "item_transitions",
            "activations", "next_reds", "levels", "batches", "batch_sources", "adv_words", "adv_zero_sectors",
            "expand_ms", "total_ms", "state_words"]
    print(json.dumps({"workload": which, "query": rx, **{k: st[k] for k in keep}}))
