"""cfg4 CRPQ timing on the LDBC-shaped graph (development aid):
python scripts/quick_cfg4.py [SCALE] -- forward plan, then with the in-edge CSR
(backward plan for the Sports atom)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_20748_b200 as R, synth
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
g = synth.ldbc_graph(scale)
s = torch.cuda.current_stream().cuda_stream
sports = g.meta["sports"]
tagged = np.unique(g.src[(g.label == g.label_names.index("hasTag")) & (g.dst == sports)])
for ie in (False, True):
    G = R.rpq_graph_load(g, stream=s, in_edges=ie)
    for i in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = R.crpq(G, ["m", "t", "u", "p"], [("m", "hasTag", "t"), ("m", "hasCreator", "u"), ("m", "replyOf*", "p")],
                   var_label={"p": "Post"}, var_const={"t": sports}, stream=s, mode=R.RPQ_STATS)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        st = r.stats()
        print(f"cfg4 scale={scale} in_edges={ie}: tuples={r.count} closed_form={tagged.size} ok={r.count == tagged.size} "
              f"t={dt*1e3:.1f}ms PE={st['product_edges']:.3e} batches={st['batches']}", flush=True)
    del G
