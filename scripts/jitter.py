"""Step-time jitter probe (development aid): per-query device (event) and host
(wall) times for the cfg2 queries evaluated back to back, as bench.py does."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

g = synth.uniform_graph(100_000, 1_000_000, 4, seed=2)
qs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["a*", "(a|b)*c", "a b* c"]
s = torch.cuda.current_stream()
sp = s.cuda_stream
G = R.rpq_graph_load(g, stream=sp)
A = {rx: R.rpq_compile(G, rx) for rx in qs}
evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(qs) + 1)]
for it in range(int(os.environ.get("ITERS", "15"))):
    torch.cuda.synchronize()
    walls = []
    evs[0].record(s)
    for i, rx in enumerate(qs):
        t0 = time.perf_counter()
        r = R.rpq_eval_allpairs(G, A[rx], mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, stream=sp)
        walls.append((time.perf_counter() - t0) * 1e3)
        st = r.stats()
        walls.append(st["total_ms"])
        walls.append(st["expand_ms"])
        evs[i + 1].record(s)
    torch.cuda.synchronize()
    dev = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(qs))]
    print("dev " + " ".join(f"{x:6.1f}" for x in dev) + " | wall/total/loop " + " ".join(f"{x:6.1f}" for x in walls), flush=True)
