"""Where the end-to-end (host arrays -> counts on the host) time of a cfg2
step goes: graph load, and each query's first (cold plan) vs repeated
evaluation (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch  # noqa: E402
import paper_2602_20748_b200 as R, synth  # noqa: E402
g = synth.uniform_graph()
s = torch.cuda.current_stream().cuda_stream
pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
       {"src": g.src, "dst": g.dst, "lab": g.label.astype(np.int16)}.items()}
hs, hd, hl = pin["src"].numpy(), pin["dst"].numpy(), pin["lab"].numpy().view(np.uint16)
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    G = R.rpq_graph_load(num_vertices=g.num_vertices, src=hs, dst=hd, label=hl, label_names=g.label_names, stream=s)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    out = [f"load {1e3*(t1-t0):6.2f}"]
    for rx in ["a*", "(a|b)*c", "a b* c"]:
        for rep in range(2):
            torch.cuda.synchronize(); a0 = time.perf_counter()
            a = R.rpq_compile(G, rx)
            a1 = time.perf_counter()
            c = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, stream=s).count
            torch.cuda.synchronize(); a2 = time.perf_counter()
            out.append(f"{rx}[{rep}] compile {1e3*(a1-a0):5.2f} eval {1e3*(a2-a1):6.2f}")
    print(" | ".join(out), flush=True)
    del G
os.environ["RPQ_DEBUG_TIMING"] = "1"
G = R.rpq_graph_load(num_vertices=g.num_vertices, src=hs, dst=hd, label=hl, label_names=g.label_names, stream=s)
R.rpq_eval_allpairs(G, R.rpq_compile(G, "a*"), mode=R.RPQ_COUNT, stream=s)
