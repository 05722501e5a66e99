"""Queries of a workload evaluated concurrently on separate streams from host
threads vs one after another (development aid)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2602_20748_b200 as R, bench
wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = bench.make_graph(wl)
qs = bench.WORKLOADS[wl]["queries"]
main = torch.cuda.current_stream()
G = R.rpq_graph_load(g, stream=main.cuda_stream)
A = {rx: R.rpq_compile(G, rx) for rx in qs}
streams = [torch.cuda.Stream() for _ in qs]
def run_seq():
    for rx in qs:
        R.rpq_eval_allpairs(G, A[rx], mode=R.RPQ_COUNT, stream=main.cuda_stream, shard_count=shards)
def run_conc():
    ths = [threading.Thread(target=lambda rx=rx, st=st: R.rpq_eval_allpairs(G, A[rx], mode=R.RPQ_COUNT, stream=st.cuda_stream, shard_count=shards))
           for rx, st in zip(qs, streams)]
    for t in ths: t.start()
    for t in ths: t.join()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("seq", run_seq), ("conc", run_conc), ("seq", run_seq), ("conc", run_conc)]:
    fn()
    ts = []
    for _ in range(8):
        torch.cuda.synchronize(); e0.record(main); fn(); e1.record(main); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{wl} shards={shards} {name}: median {ts[len(ts)//2]:.2f} ms  min {ts[0]:.2f}", flush=True)
