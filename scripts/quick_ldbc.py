"""LDBC-shaped cfg3 timing + closed-form checks (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_20748_b200 as R, synth
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
t0 = time.time()
g = synth.ldbc_graph(scale)
print(f"gen {time.time()-t0:.1f}s V={g.num_vertices} E={g.num_edges}", flush=True)
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
base, cnt = g.meta["base"], g.meta["count"]
# closed forms
parent = g.meta["reply_parent"]
C = cnt["Comment"]
depth = np.zeros(C, np.int64)
pc = parent - base["Comment"]
is_c = (parent >= base["Comment"]) & (parent < base["Comment"] + C)
for i in range(C):
    depth[i] = 1 + (depth[pc[i]] if is_c[i] else 0)
want_reply = g.num_vertices + int(depth.sum())
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components
m = g.label == 0
P = cnt["Person"]
A = sp.csr_matrix((np.ones(int(m.sum())), (g.src[m] - base["Person"], g.dst[m] - base["Person"])), shape=(P, P))
_, comp = connected_components(A, directed=False)
sizes = np.bincount(comp)
want_knows = int((sizes[sizes >= 2] ** 2).sum())
for rx, want in [("replyOf*", want_reply), ("knows+", want_knows)]:
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=s)
    st = r.stats()
    torch.cuda.synchronize()
    t = time.perf_counter()
    r2 = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, stream=s)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{rx:10s} count={r.count} closed_form={want} ok={r.count == want} PE={st['product_edges']:.3e} "
          f"batches={st['batches']} B={st['batch_sources']} levels={st['levels']} t={dt*1e3:.1f}ms "
          f"loop={r2.stats()['expand_ms']:.1f}ms TEPS={st['product_edges']/dt:.3e}", flush=True)
