"""cfg2 queries at several batch widths (development aid): is a whole-group
width plus a small remainder batch faster than the single full-width batch?
python scripts/batch_width_cfg2.py"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

g = synth.uniform_graph()
s = torch.cuda.current_stream().cuda_stream
G = R.rpq_graph_load(g, stream=s)
for rx in ["a*", "(a|b)*c", "a b* c"]:
    a = R.rpq_compile(G, rx)
    for B in [0, 98304, 81920, 0, 98304, 81920, 65536, 49152]:
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, stream=s, batch_sources=B)
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) * 1e3
            st = r.stats()
            if best is None or dt < best[0]:
                best = (dt, st["expand_ms"], st["batches"], st["batch_sources"], r.count)
        print(f"{rx:10s} B={B:6d} -> width {best[3]:6d} batches {best[2]} total {best[0]:7.2f} ms loop {best[1]:7.2f} ms count {best[4]}",
              flush=True)
