"""rpq_graph_load timing from pinned host arrays (development aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2602_20748_b200 as R, bench
for wl in sys.argv[1:] or ["cfg2", "cfg3"]:
    g = bench.make_graph(wl)
    pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
           {"src": g.src, "dst": g.dst, "lab": g.label.astype(np.int16)}.items()}
    hs, hd, hl = pin["src"].numpy(), pin["dst"].numpy(), pin["lab"].numpy().view(np.uint16)
    for ie in (False, True):
        ts = []
        for i in range(4):
            torch.cuda.synchronize(); t = time.perf_counter()
            G = R.rpq_graph_load(num_vertices=g.num_vertices, src=hs, dst=hd, label=hl, label_names=g.label_names,
                                 in_edges=ie)
            torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
            info = R.rpq_graph_info(G)
            del G
        print(f"{wl} in_edges={ie} E={info['num_edges']} load ms: {' '.join(f'{x:.1f}' for x in ts)}", flush=True)
