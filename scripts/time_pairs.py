"""PAIRS-mode timing (development aid): python scripts/time_pairs.py cfg2|cfg3"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
g = bench.make_graph(wl)
s = torch.cuda.current_stream()
G = R.rpq_graph_load(g, stream=s.cuda_stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rx in bench.WORKLOADS[wl]["queries"]:
    a = R.rpq_compile(G, rx)
    for mode, name in [(R.RPQ_COUNT, "COUNT"), (R.RPQ_PER_SOURCE, "PER_SOURCE"), (R.RPQ_PAIRS, "PAIRS")]:
        ts = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record(s)
            r = R.rpq_eval_allpairs(G, a, mode=mode | R.RPQ_TIME_KERNELS, stream=s.cuda_stream)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            st = r.stats()
            cnt = r.count
            del r
        print(f"{wl} {rx:10s} {name:10s} count={cnt} B={st['batch_sources']} batches={st['batches']} "
              f"ms={min(ts):8.2f} loop_ms={st['expand_ms']:8.2f} pairs/s={cnt / min(ts) * 1e3:.3e}", flush=True)
