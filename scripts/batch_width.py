"""RMAT-24 (a|b)*c* over one fixed seeded source set at several batch widths
(development aid): does a width that fills whole 8-chunk row groups beat the
HBM-maximal width?  python scripts/batch_width.py [NSRC]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300_000
cache = "/tmp/rpq_graph_rmat24.npz"
if os.path.exists(cache):
    z = np.load(cache, allow_pickle=True)
    g = synth.Graph(int(z["nv"]), z["src"], z["dst"], z["label"], list(z["names"]))
else:
    g = synth.rmat_graph(24, seed=24)
    np.savez(cache, nv=g.num_vertices, src=g.src, dst=g.dst, label=g.label, names=np.array(g.label_names))
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
a = R.rpq_compile(G, "(a|b)*c*")
src = synth.sample_sources(g.num_vertices, n, seed=3)
print("plan", R.rpq_plan(G, a, stream=s)["batch_sources"], flush=True)
for B in [19584, 16384, 19584, 16384, 18432, 20480]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = R.rpq_eval_sources(G, a, src, mode=R.RPQ_COUNT | R.RPQ_PE | R.RPQ_TIME_KERNELS, stream=s, batch_sources=B)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = r.stats()
    print(f"B={B:6d} nw={(B + 63) // 64:4d} batches={st['batches']:3d} total={dt * 1e3:9.1f} ms loop={st['expand_ms']:9.1f} ms "
          f"count={r.count} PE={st['product_edges']:.4e} PE/s={st['product_edges'] / dt:.4e}", flush=True)
