"""RMAT cfg5-shaped timing (development aid): python scripts/quick_rmat.py SCALE [SHARDS] [REGEX]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_20748_b200 as R, synth
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rx = sys.argv[3] if len(sys.argv) > 3 else "(a|b)*c*"
t0 = time.time()
g = synth.rmat_graph(scale)
print(f"gen {time.time()-t0:.1f}s V={g.num_vertices} E={g.num_edges}", flush=True)
s = torch.cuda.current_stream().cuda_stream
t0 = time.time()
G = R.rpq_graph_load(g, stream=s)
torch.cuda.synchronize()
print(f"load {time.time()-t0:.2f}s distinct E={R.rpq_graph_info(G)['num_edges']}", flush=True)
a = R.rpq_compile(G, rx)
torch.cuda.synchronize()
t = time.perf_counter()
r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS | R.RPQ_TIME_KERNELS, stream=s, shard_index=0,
                        shard_count=shards)
torch.cuda.synchronize()
dt = time.perf_counter() - t
st = r.stats()
print(f"{rx} shard 0/{shards}: count={r.count} PE={st['product_edges']:.3e} wordops={st['word_edge_ops']:.3e} "
      f"keff={st['product_edges']/max(1,st['word_edge_ops']):.1f} P={st['productive_sources']} B={st['batch_sources']} "
      f"batches={st['batches']} levels={st['levels']} t={dt:.2f}s loop={st['expand_ms']/1e3:.2f}s "
      f"TEPS={st['product_edges']/dt:.3e}", flush=True)
