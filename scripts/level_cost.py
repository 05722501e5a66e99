"""Fixed cost per BFS level (development aid): a chain graph forces one level
per vertex with almost no work."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = synth.chain_graph(n)
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, "a*")
for B in (64, 4096):
    for i in range(3):
        r = R.rpq_eval_sources(G, a, list(range(min(B, 64))), mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS | R.RPQ_STATS,
                               stream=s, batch_sources=B)
        st = r.stats()
    print(f"chain {n}: levels {st['levels']} loop {st['expand_ms']:.2f} ms -> {st['expand_ms'] * 1e3 / max(1, st['levels']):.1f} us/level "
          f"(B={st['batch_sources']}, launches {st['kernel_launches']})", flush=True)
