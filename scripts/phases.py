"""Per-query time breakdown (development aid; bench.py is the contract).

python scripts/phases.py cfg2|cfg3|rmatNN [shards]
For each query: event-timed COUNT eval (no in-kernel timers), level-loop
time (RPQ_TIME_KERNELS), and one RPQ_DEBUG_TIMING pass (synchronising) that
prints the host-observed phase times.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if wl == "cfg2":
    g, qs = synth.uniform_graph(100_000, 1_000_000, 4, seed=2), ["a*", "(a|b)*c", "a b* c"]
elif wl == "cfg3":
    g, qs = synth.ldbc_graph(1.0, seed=10), ["replyOf*", "knows+"]
else:
    g, qs = synth.rmat_graph(int(wl[4:]), seed=24), ["(a|b)*c*"]
if len(sys.argv) > 3:
    qs = sys.argv[3].split(",")
reps = int(os.environ.get("PH_REPS", "4"))
s = torch.cuda.current_stream()
sp = s.cuda_stream
G = R.rpq_graph_load(g, stream=sp)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rx in qs:
    a = R.rpq_compile(G, rx)
    st = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=sp, shard_count=shards).stats()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        ev0.record(s)
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, stream=sp, shard_count=shards)
        ev1.record(s)
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    r2 = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_TIME_KERNELS, stream=sp, shard_count=shards)
    loop = r2.stats()["expand_ms"]
    print(f"{rx:10s} count={r.count} PE={st['product_edges']:.3e} wordops={st['word_edge_ops']:.3e} "
          f"B={st['batch_sources']} batches={st['batches']} levels={st['levels']} "
          f"event_ms={min(ts):.2f} (all {', '.join(f'{t:.1f}' for t in ts)}) loop_ms={loop:.2f}", flush=True)
    os.environ["RPQ_DEBUG_TIMING"] = "1"
    R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT, stream=sp, shard_count=shards)
    torch.cuda.synchronize()
    del os.environ["RPQ_DEBUG_TIMING"]
    sys.stderr.flush()
