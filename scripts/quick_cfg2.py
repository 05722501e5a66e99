"""Quick timing of the cfg2 queries (development aid; bench.py is the contract)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_20748_b200 as R, synth
g = synth.uniform_graph()
torch.cuda.init()
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
Bs = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else [0, 8192, 2048]
for B in Bs:
    for rx in ["a*", "(a|b)*c", "a b* c"]:
        a = R.rpq_compile(G, rx)
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, batch_sources=B, stream=s)
        st = r.stats()
        ts = []
        for i in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            r2 = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, batch_sources=B, stream=s)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        st2 = r2.stats()
        t = min(ts)
        print(f"B={B} {rx:10s} count={r.count} PE={st['product_edges']:.3e} wordops={st['word_edge_ops']:.3e} "
              f"keff={st['product_edges']/max(1,st['word_edge_ops']):.2f} levels={st['levels']} batches={st['batches']} "
              f"Bsrc={st['batch_sources']} cw={st['chunk_words']} t={t*1e3:.2f}ms expand={st2['expand_ms']:.2f}ms "
              f"TEPS={st['product_edges']/t:.3e} act={st['activations']:.3e} nred={st['next_reds']:.3e} items={st['items']:.3e}",
              flush=True)
