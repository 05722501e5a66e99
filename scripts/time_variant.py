"""Time one library build (RPQ_LIB_PATH) on a workload (development aid).
python scripts/time_variant.py rmat24|cfg2|knows [SHARDS]
The generated graph is cached under /tmp (per box) to keep variant sweeps short."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

wl = sys.argv[1]
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cache = f"/tmp/rpq_graph_{wl}.npz"
if wl.startswith("rmat"):
    mk, qs = (lambda: synth.rmat_graph(int(wl[4:]), seed=24)), ["(a|b)*c*"]
elif wl == "cfg2":
    mk, qs = (lambda: synth.uniform_graph()), ["a*", "(a|b)*c", "a b* c"]
else:
    mk, qs = (lambda: synth.ldbc_graph(1.0, seed=10)), ["knows+"]
if os.path.exists(cache):
    z = np.load(cache, allow_pickle=True)
    g = synth.Graph(int(z["nv"]), z["src"], z["dst"], z["label"], list(z["names"]))
else:
    g = mk()
    np.savez(cache, nv=g.num_vertices, src=g.src, dst=g.dst, label=g.label, names=np.array(g.label_names))
s = torch.cuda.current_stream()
G = R.rpq_graph_load(g, stream=s.cuda_stream, in_edges=os.environ.get("TV_IN_EDGES") == "1")
tag = os.path.basename(os.environ.get("RPQ_LIB_PATH", "librpq.so"))
for rx in qs:
    a = R.rpq_compile(G, rx)
    B = R.rpq_plan(G, a, stream=s.cuda_stream, shard_count=shards)["batch_sources"] if shards > 1 else 0
    R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, stream=s.cuda_stream, shard_count=shards, batch_sources=B)
    best = None
    for _ in range(3 if not wl.startswith("rmat") else 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, stream=s.cuda_stream,
                                shard_count=shards, batch_sources=B)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        st = r.stats()
        if best is None or dt < best[0]:
            best = (dt, st["expand_ms"], r.count)
    sp = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=s.cuda_stream, shard_count=shards,
                             batch_sources=B).stats()
    print(f"{tag:28s} {rx:10s} total_ms={best[0]:9.2f} loop_ms={best[1]:9.2f} count={best[2]} "
          f"PE={sp['product_edges']:.4e} pull_levels={sp['pull_levels']} levels={sp['levels']} "
          f"pull_loads={sp['pull_loads']:.3e} pull_words={sp['pull_words']:.3e} adv_words={sp['adv_words']:.3e} "
          f"adv_zero_sectors={sp['adv_zero_sectors']:.3e} word_items={sp['word_items']:.3e} wordops={sp['word_edge_ops']:.3e}",
          flush=True)
