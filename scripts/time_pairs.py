"""PAIRS evaluation time of the cfg2 queries and an order-sensitive checksum of the
result (development aid; RPQ_LIB_PATH selects a library build).
python scripts/time_pairs.py"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

from cuda.bindings import runtime as rt  # noqa: E402

CH = 1 << 27


def checksum(r):
    """Order-sensitive checksum of both columns, copied D2D in 512 MiB chunks."""
    (ps, pd), n = r.device_view()
    buf = torch.empty(CH, dtype=torch.int32, device="cuda")
    acc = 0
    for col, p in ((1, ps), (2, pd)):
        for o in range(0, n, CH):
            k = min(CH, n - o)
            rt.cudaMemcpy(buf.data_ptr(), p + 4 * o, 4 * k, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
            x = buf[:k].to(torch.int64)
            idx = torch.arange(o, o + k, device="cuda", dtype=torch.int64)
            acc += col * int(((x + 1) * ((idx % 1000003) + 1)).sum())
    return acc


g = synth.uniform_graph()
s = torch.cuda.current_stream()
G = R.rpq_graph_load(g, stream=s.cuda_stream)
for rx in ["a*", "(a|b)*c", "a b* c"]:
    a = R.rpq_compile(G, rx)
    ref = None
    for var in ["run1", "run2"]:
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS, stream=s.cuda_stream)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            n = r.count
            h = checksum(r)
            del r
        ok = "" if ref is None else ("same" if (n, h) == ref else "DIFFERENT")
        ref = ref or (n, h)
        print(f"{rx:10s} {var} ms={min(ts):8.2f} (all {['%.1f' % x for x in ts]}) pairs={n} {ok}", flush=True)
