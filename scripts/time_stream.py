"""Streamed PAIRS throughput (development aid): cfg2 queries, pairs to host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, synth
g = synth.uniform_graph()
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
for rx in sys.argv[1:] or ["a*"]:
    a = R.rpq_compile(G, rx)
    n = [0]
    def sink(src, dst):
        n[0] += src.size
        return False
    for budget in (0, 8 << 30):
        t = time.perf_counter()
        tot, _ = R.rpq_eval_allpairs_stream(G, a, sink=sink, device_budget_bytes=budget, stream=s)
        dt = time.perf_counter() - t
        print(f"{rx} budget={budget} pairs={tot} {dt:.2f}s -> {tot/dt:.3e} pairs/s, {tot*8/dt/1e9:.1f} GB/s to host", flush=True)
