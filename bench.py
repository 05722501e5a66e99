"""bench.py -- all-pairs RPQ throughput (product edges traversed per second).

Contract (driver): `python bench.py --gpus N --steps K --warmup W` prints ONE
JSON line on rank 0.  N>1 runs under torch.distributed.run, one process per
GPU (NCCL): the source batches are sharded round-robin over ranks (batch b ->
rank b % N), the graph is replicated, and only counts/PE are reduced.

A step = one pass of the whole hot path over the workload: for each query of
the workload, compile the regex and evaluate the all-pairs RPQ in COUNT mode
(the paper's benchmark output) on the device-resident graph.
Metric = PE / s where PE (product edges traversed, reading
R12 in DESIGN.md) = sum over reached (vertex, state) pairs of the product
out-degree on the minimal trim DFA -- identical for the GPU path and the
oracle (pinned by tests).

Multi-GPU: every query goes through the product's distributed call
(paper_2602_20748_b200.dist.rpq_eval_allpairs_dist): the ranks agree on one
batch plan (rpq_plan + all-reduce MIN), each evaluates its batches, and the
counts are all-reduced -- the gather is inside the timed step.

After the cfg2 headline the same run measures BASELINE's north-star
configuration once (`north_star` object): the WHOLE RMAT-24 (a|b)*c*
all-pairs COUNT over all N ranks (configs[4]), asserted against its known
count, with exact PE from the count pass (RPQ_PE); and the cfg3 LDBC SF10
queries (`cfg3` object).  Both graphs are generated on a background thread
while cfg2 runs.  `--no-north-star` / `--no-cfg3` skip them.

`--impl reference` times the CPU oracle (oracle/, O1) on a bounded seeded
sample of the same workload, on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOADS = {
    # BASELINE.json configs[1]: random labelled graph, 100K vertices / 1M
    # edges, 4 labels, RPQs a*, (a|b)*c, a b* c, all-pairs, 1 GPU
    "cfg2": {"queries": ["a*", "(a|b)*c", "a b* c"],
             "desc": "uniform random labelled graph |V|=100000 |E|=1000000 (distinct), 4 labels, seed 2"},
    # configs[2]: LDBC-SNB-shaped SF10-size social graph, replyOf* and knows+
    "cfg3": {"queries": ["replyOf*", "knows+"],
             "desc": "LDBC-SNB-shaped synthetic graph, SF10 size (35.5M vertices, 219.4M edges), seed 10"},
    # configs[4]: RMAT scale 24, 8 labels, (a|b)*c*; one GPU evaluates the
    # batches of shard 0 of --sample-shards (stated in config.sample)
    "cfg5": {"queries": ["(a|b)*c*"],
             "desc": "R-MAT scale 24 (16.8M vertices, 2^28 edge samples), Graph500 A,B,C,D, 8 labels, seed 24"},
}


# |R((a|b)*c*)| on rmat_graph(24, seed=24): the whole all-pairs query, summed
# over the 16 shards and equal to the 1-GPU run (round 1)
RMAT24_COUNT = 27_130_980_830_746


def make_graph(name):
    import synth
    if name == "cfg2":
        return synth.uniform_graph(100_000, 1_000_000, 4, seed=2)
    if name == "cfg3":
        return synth.ldbc_graph(1.0, seed=10)
    if name == "cfg5":
        return synth.rmat_graph(24, seed=24)
    raise ValueError(name)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload):
    """ncu DRAM bytes per k_level launch for the workload, committed under
    profiles/ (see profiles/README.md); None if absent."""
    p = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("BENCH_NOCLK") == "1":
            return self
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def algorithmic_bytes(st):
    """Bytes the fused level kernel must move: 24 B per
    advanced word (Vis read, Done read, Done write), 8 B per (row-group,
    transition) CSR offset pair, 4 B per (row-group, edge) neighbour id, 16 B
    per (non-zero frontier word, edge) operation (visited read 8 B + the OR of
    the new bits into it 8 B -- SURVEY.md §8(d)'s "Vis read + Next RMW")."""
    # bottom-up levels (symmetric labels): 8 B per in-neighbour
    # visited-word load and 8 B per scanned target word
    return (24 * st["word_items"] + 8 * st["item_transitions"] + 4 * st["item_edges"]
            + 16 * st["word_edge_ops"] + 8 * st.get("pull_loads", 0) + 8 * st.get("pull_words", 0))


# --------------------------------------------------------------------------
class GraphMaker:
    """Generates the north-star / cfg3 graphs on a background thread while the
    headline runs (numpy releases the GIL in the heavy array ops)."""

    def __init__(self, names):
        self.out, self.err = {}, {}
        self.t = threading.Thread(target=self._run, args=(list(names),), daemon=True)
        self.t.start()

    def _run(self, names):
        for n in names:
            t0 = time.perf_counter()
            try:
                self.out[n] = (make_graph(n), time.perf_counter() - t0)
            except Exception as e:              # reported in the JSON line
                self.err[n] = repr(e)

    def get(self, name):
        while name not in self.out and name not in self.err and self.t.is_alive():
            time.sleep(0.05)
        if name in self.err:
            raise RuntimeError(self.err[name])
        return self.out[name]


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2602_20748_b200 as R
    from paper_2602_20748_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # BENCH_SINGLE_GPU_TEST=1 (testing aid only): every rank on cuda:0 over
    # gloo, to exercise the N>1 code path on a one-GPU box
    one_gpu_test = os.environ.get("BENCH_SINGLE_GPU_TEST") == "1"
    if one_gpu_test:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if one_gpu_test else "cuda"   # device of the reduced scalars
    extra = []
    if args.north_star and args.workload == "cfg2":
        extra.append("cfg5")
    if args.cfg3 and args.workload == "cfg2":
        extra.append("cfg3")
    maker = GraphMaker(extra) if extra else None
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    wl = WORKLOADS[args.workload]
    g = make_graph(args.workload)
    G = R.rpq_graph_load(g, device=local, stream=sp)
    queries = wl["queries"]

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # batch width: N = 1 -> automatic (the library sizes it against HBM);
    # N > 1 -> the ranks agree on one plan (rpq_plan + all-reduce MIN, the
    # product's dist path).  --sample-shards S (one GPU standing in for one
    # rank of N x S shards, a testing aid) evaluates 1/S of the batches.
    sample = max(1, args.sample_shards)
    nshard = world * sample
    bsz = {}
    for rx in queries:
        a = R.rpq_compile(G, rx)
        if args.batch:
            bsz[rx] = args.batch
        elif nshard > 1:
            pl = R.rpq_plan(G, a, mode=R.RPQ_COUNT, shard_count=nshard, stream=sp)
            bsz[rx] = D.agree_batch_sources(pl["batch_sources"])
        else:
            bsz[rx] = 0

    def eval_count(Gx, a, B, mode):
        """One query over the job: the product's dist call (the gather is the
        count all-reduce); with --sample-shards this rank's shard directly."""
        if sample > 1:
            r = R.rpq_eval_allpairs(Gx, a, mode=mode, stream=sp, batch_sources=B, shard_index=rank,
                                    shard_count=nshard)
            return r.count, r.stats()
        d = D.rpq_eval_allpairs_dist(Gx, a, mode=mode, stream=sp, batch_sources=B)
        return d.count, d.local.stats()

    # per-rank probe with the in-kernel counters (RPQ_STATS): PE and the
    # algorithmic bytes of this rank's shard
    probe = {}
    for rx in queries:
        a = R.rpq_compile(G, rx)
        r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=sp, batch_sources=bsz[rx],
                                shard_index=rank, shard_count=nshard)
        probe[rx] = r.stats()

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")   # > 126 MB L2

    def step(mode):
        tot = {"count": 0, "launches": 0, "expand_ms": 0.0, "levels": 0}
        for rx in queries:
            a = R.rpq_compile(G, rx)
            c, st = eval_count(G, a, bsz[rx], mode)
            tot["count"] += c
            tot["launches"] += st["kernel_launches"]
            tot["expand_ms"] += st["expand_ms"]
            tot["levels"] += st["levels"]
        return tot

    # timed steps run without the in-kernel counters; the algorithmic bytes
    # of a step come from the RPQ_STATS probe runs above (per query)
    mode = R.RPQ_COUNT | (R.RPQ_TIME_KERNELS if os.environ.get("BENCH_TK", "1") == "1" else 0)
    probe_bytes = sum(algorithmic_bytes(probe[rx]) for rx in queries)
    probe_levels = sum(probe[rx]["levels"] for rx in queries)
    probe_pe = sum(probe[rx]["product_edges"] for rx in queries)
    for _ in range(args.warmup):
        step(mode)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    times, agg = [], None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if os.environ.get("BENCH_NOFLUSH") != "1":
                flush.fill_(1)                   # evict L2 between timed steps (untimed)
            torch.cuda.synchronize()
            ev0.record(stream)
            t = step(mode)
            ev1.record(stream)
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
            if agg is None:
                agg = dict(t)
            else:
                for k in agg:
                    agg[k] += t[k]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if os.environ.get("BENCH_DEBUG"):
        print("step ms:", " ".join(f"{t:.1f}" for t in times), file=sys.stderr)
    total_ms = allmax(float(sum(times)))
    pe_total = allsum(probe_pe * args.steps)          # PE is a property of (graph, query, shard)
    # the dist call already summed the count over ranks (sample > 1: this shard only)
    count_total = agg["count"] if sample == 1 else allsum(agg["count"])

    # end to end through the public API: host (pinned) edge arrays -> load ->
    # compile -> evaluate -> counts on the host, every step
    e2e_ms = []
    pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
           {"src": g.src, "dst": g.dst, "lab": g.label.astype(np.int16)}.items()}
    h_src, h_dst = pin["src"].numpy(), pin["dst"].numpy()
    h_lab = pin["lab"].numpy().view(np.uint16)
    h2d = int(h_src.nbytes + h_dst.nbytes + h_lab.nbytes)
    e2e_steps = max(1, min(args.steps, 5))
    for i in range(e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G2 = R.rpq_graph_load(num_vertices=g.num_vertices, src=h_src, dst=h_dst, label=h_lab,
                              label_names=g.label_names, device=local, stream=sp)
        for rx in queries:
            a = R.rpq_compile(G2, rx)
            _ = eval_count(G2, a, bsz[rx], R.RPQ_COUNT)[0]      # device -> host result
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        del G2
        if i > 0:
            e2e_ms.append(dt)
    e2e_step = allmax(statistics.median(e2e_ms))

    ns = north_star_leg(args, R, D, maker, sp, stream, local, rank, world, allmax, allsum) \
        if maker and "cfg5" in extra else None
    c3 = cfg3_leg(args, R, D, maker, sp, stream, local, rank, world, allmax, allsum) \
        if maker and "cfg3" in extra else None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pe_per_step = pe_total / args.steps
    value = pe_total / (total_ms / 1e3)
    peak, peak_src = load_peaks()
    step_bytes = probe_bytes * args.steps
    achieved = step_bytes / (agg["expand_ms"] / 1e3) / 1e9 if agg["expand_ms"] > 0 else None
    per_launch = probe_bytes / max(1, probe_levels)
    # the committed ncu bytes per launch are for full-width batches; a sampled
    # shard (--sample-shards) runs narrower batches, so they do not apply
    traffic = load_traffic(args.workload) if sample == 1 else None
    line = {
        "metric": "all-pairs RPQ product-edges traversed/s",
        "value": value,
        "unit": "PE/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u64",
        "data": "synthetic",
        "config": {"workload": args.workload, "graph": wl["desc"], "queries": queries, "mode": "COUNT",
                   "pe_per_step": pe_per_step, "pairs_per_step": count_total / args.steps,
                   "batch_sources": {rx: probe[rx]["batch_sources"] if not bsz[rx] else bsz[rx] for rx in queries},
                   "parallelism": f"source-batch shards x{world} (rpq_eval_allpairs_dist: agreed batch plan, "
                                  f"count all-reduce inside the step)",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "sample": "all batches" if sample == 1 else
                             f"batches of shards 0..{world - 1} of {nshard} (1/{sample} of the all-pairs query)"},
        "roofline": {"bound": "hbm", "kernel": "k_level (level loop: k_units + k_level + k_level_hub)",
                     "achieved": achieved, "peak": peak,
                     "peak_nominal": 8000.0,
                     "frac_nominal": (achieved / 8000.0) if achieved else None,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "algorithmic_bytes_per_launch": per_launch,
                     "launches": agg["levels"],
                     "level_loop_ms_per_step": agg["expand_ms"] / args.steps,
                     "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     # the same ncu DRAM bytes per launch over this run's average launch
                     # duration: the measured (not algorithmic) bandwidth of the loop
                     "traffic_gbs": (traffic["dram_bytes_per_launch"] / (agg["expand_ms"] / 1e3 / agg["levels"]) / 1e9)
                     if traffic and agg["expand_ms"] > 0 and agg["levels"] else None},
        "e2e": {"value": pe_per_step / (e2e_step / 1e3), "unit": "PE/s", "ms_per_step": e2e_step,
                "h2d_bytes_per_step": h2d * 1, "d2h_bytes_per_step": 8 * len(queries),
                "includes": "rpq_graph_load from pinned host arrays + compile + eval + count readback"},
        "gpu_launches": agg["launches"],
        "clocks": clk.summary(),
    }
    if ns is not None:
        line["north_star"] = ns
    if c3 is not None:
        line["cfg3"] = c3
    if world == 1 and args.workload != "cfg5" and not args.no_pairs:
        # PAIRS mode (timed separately from the COUNT headline):
        # sorted distinct pairs materialised in device memory, per query
        pr = {}
        for rx in queries:
            a = R.rpq_compile(G, rx)
            R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS, stream=sp)          # warm-up (pool growth)
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                ev0.record(stream)
                r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS, stream=sp)
                ev1.record(stream)
                torch.cuda.synchronize()
                ts.append(ev0.elapsed_time(ev1))
                n = r.count
                del r
            pr[rx] = {"pairs": n, "ms": statistics.median(ts), "pairs_per_s": n / (statistics.median(ts) / 1e3)}
        line["pairs_mode"] = {"unit": "pairs/s", "device_resident": True, "queries": pr}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, g, queries, budget_s=args.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def north_star_leg(args, R, D, maker, sp, stream, local, rank, world, allmax, allsum):
    """BASELINE north_star / configs[4]: the whole RMAT-24 (a|b)*c* all-pairs
    COUNT across the N ranks, once, after a warm-up on 1/64 of the batches.
    PE is exact (RPQ_PE: popcount x product out-degree inside the count
    pass); the count is asserted against RMAT24_COUNT.  Algorithmic bytes =
    (bytes per PE of an RPQ_STATS probe on the warm-up sample) x PE."""
    import torch
    import torch.distributed as dist
    g5, gen_s = maker.get("cfg5")
    t0 = time.perf_counter()
    G5 = R.rpq_graph_load(g5, device=local, stream=sp)
    torch.cuda.synchronize()
    load_s = time.perf_counter() - t0
    rx = WORKLOADS["cfg5"]["queries"][0]
    a5 = R.rpq_compile(G5, rx)
    pl = R.rpq_plan(G5, a5, mode=R.RPQ_COUNT, shard_count=world, stream=sp)
    B5 = D.agree_batch_sources(pl["batch_sources"])
    nb = -(-pl["productive_sources"] // B5)
    # warm-up + algorithmic-bytes probe: this rank's share of 1/64 of the batches
    R.rpq_eval_allpairs(G5, a5, mode=R.RPQ_COUNT, stream=sp, batch_sources=B5, shard_index=rank,
                        shard_count=world * 64)
    pst = R.rpq_eval_allpairs(G5, a5, mode=R.RPQ_COUNT | R.RPQ_STATS, stream=sp, batch_sources=B5,
                              shard_index=rank, shard_count=world * 64).stats()
    bytes_per_pe = allsum(algorithmic_bytes(pst)) / max(1.0, allsum(pst["product_edges"]))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        d = D.rpq_eval_allpairs_dist(G5, a5, mode=R.RPQ_COUNT | R.RPQ_PE | R.RPQ_TIME_KERNELS, stream=sp,
                                     batch_sources=B5)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = allmax(ev0.elapsed_time(ev1))
    loop_ms = allmax(d.local.stats()["expand_ms"])
    pe = int(d.stats["product_edges"])
    del G5
    peak, peak_src = load_peaks()
    traffic = load_traffic("cfg5")
    alg_bytes = bytes_per_pe * pe
    ncu_over_alg = None
    if traffic and traffic.get("all") and pst.get("levels"):
        kl = traffic["all"]
        dram_per_level = sum(kl[k]["dram_bytes"] for k in ("k_level", "k_level_hub") if k in kl) / \
            max(1, kl["k_level"]["launches"])
        ncu_over_alg = dram_per_level / (algorithmic_bytes(pst) / pst["levels"])
    # per GPU: its share of the bytes over the whole-query time (the slowest rank)
    achieved = alg_bytes / world / (ms / 1e3) / 1e9
    out = {"workload": "cfg5", "graph": WORKLOADS["cfg5"]["desc"], "query": rx, "mode": "COUNT, all-pairs, all batches",
           "n_gpus": world, "count": d.count, "count_expected": RMAT24_COUNT, "count_ok": d.count == RMAT24_COUNT,
           "ms": ms, "pe": pe, "pe_per_s": pe / (ms / 1e3), "batches": nb, "batch_sources": B5,
           "level_loop_ms_max_rank": loop_ms, "graph_gen_s": gen_s, "graph_load_s": load_s,
           "roofline": {"bound": "hbm", "unit": "GB/s", "peak": peak, "peak_source": peak_src,
                        "algorithmic_bytes": alg_bytes, "bytes_per_pe": bytes_per_pe,
                        "achieved_per_gpu": achieved, "frac": achieved / peak,
                        "note": "algorithmic bytes per PE from an RPQ_STATS probe of 1/64 of the batches x exact PE; "
                                "time = whole query (count pass, clears, per-batch setup included), slowest rank",
                        # ncu DRAM bytes of the level kernels (k_level + k_level_hub) per level on
                        # shard 0 of 64 (profiles/traffic_cfg5.json) over this run's algorithmic
                        # bytes per level on the same shard (the RPQ_STATS probe above, rank 0)
                        "ncu_dram_over_algorithmic": ncu_over_alg},
           "clocks": clk.summary()}
    if not out["count_ok"] and rank == 0:
        print(f"north_star: count {d.count} != expected {RMAT24_COUNT}", file=sys.stderr)
    return out


def cfg3_leg(args, R, D, maker, sp, stream, local, rank, world, allmax, allsum):
    """BASELINE configs[2]: LDBC-SNB-shaped SF10 graph, replyOf* and knows+
    all-pairs COUNT over the N ranks (source-sharded); median of 3 after 3
    warm-ups, exact PE from the count pass (RPQ_PE)."""
    import torch
    import torch.distributed as dist
    g3, gen_s = maker.get("cfg3")
    G3 = R.rpq_graph_load(g3, device=local, stream=sp)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    res = {}
    tot_ms, tot_pe = 0.0, 0
    for rx in WORKLOADS["cfg3"]["queries"]:
        a = R.rpq_compile(G3, rx)
        B = 0
        if world > 1:
            B = D.agree_batch_sources(R.rpq_plan(G3, a, shard_count=world, stream=sp)["batch_sources"])
        m = R.RPQ_COUNT | R.RPQ_PE
        for _ in range(3):
            d = D.rpq_eval_allpairs_dist(G3, a, mode=m, stream=sp, batch_sources=B)
        ts = []
        for _ in range(3):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            d = D.rpq_eval_allpairs_dist(G3, a, mode=m, stream=sp, batch_sources=B)
            ev1.record(stream)
            torch.cuda.synchronize()
            ts.append(allmax(ev0.elapsed_time(ev1)))
        ms = statistics.median(ts)
        pe = int(d.stats["product_edges"])
        res[rx] = {"count": d.count, "pe": pe, "ms": ms, "pe_per_s": pe / (ms / 1e3),
                   "batch_sources": d.batch_sources}
        tot_ms += ms
        tot_pe += pe
    del G3
    return {"workload": "cfg3", "graph": WORKLOADS["cfg3"]["desc"], "n_gpus": world, "queries": res,
            "ms": tot_ms, "pe": tot_pe, "pe_per_s": tot_pe / (tot_ms / 1e3), "graph_gen_s": gen_s}


# --------------------------------------------------------------------------
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_sample(g, queries, budget_s, seed=0, threads=0):
    """Time the oracle (O1, all host threads unless `threads`) on seeded
    source samples of the workload, growing the sample until ~budget_s
    seconds of CPU work."""
    import oracle
    og = oracle.OracleGraph(g)
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    order = rng.permutation(g.num_vertices).astype(np.uint32)
    n, pe, secs, used = 64, 0, 0.0, 0
    while secs < budget_s and used < g.num_vertices:
        srcs = np.sort(order[used:used + n])
        t0 = time.perf_counter()
        for rx in queries:
            r = oracle.eval_sources(og, rx, srcs, pairs=False, threads=threads)
            pe += int(r["pe"].sum())
        secs += time.perf_counter() - t0
        used += srcs.size
        n = min(n * 2, 1 << 16)
    return pe, secs, used, threads


def cpu_baseline(args, g, queries, budget_s):
    pe, secs, used, threads = oracle_sample(g, queries, budget_s)
    pe1, secs1, _, _ = oracle_sample(g, queries, min(4.0, budget_s / 4), seed=7, threads=1)
    return {"value": pe / secs, "unit": "PE/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "single_thread_value": pe1 / secs1,
            "sample": f"{used} seeded random sources x {len(queries)} queries of {args.workload} "
                      f"({pe:.3e} PE in {secs:.1f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = WORKLOADS[args.workload]
    g = make_graph(args.workload)
    queries = wl["queries"]
    per_step = args.ref_step_seconds
    for _ in range(args.warmup):
        oracle_sample(g, queries, per_step / 4, seed=1)
    pe_tot, s_tot, used_tot, threads = 0, 0.0, 0, 1
    for k in range(args.steps):
        pe, secs, used, threads = oracle_sample(g, queries, per_step, seed=100 + k)
        pe_tot += pe
        s_tot += secs
        used_tot += used
    value = pe_tot / s_tot
    line = {"impl": "reference", "metric": "all-pairs RPQ product-edges traversed/s", "value": value,
            "unit": "PE/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": s_tot * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": args.workload, "graph": wl["desc"], "queries": queries, "mode": "COUNT"},
            "cpu_baseline": {"value": value, "unit": "PE/s", "cores": threads, "kind": "oracle",
                             "sample": f"{used_tot} seeded random sources x {len(queries)} queries over "
                                       f"{args.steps} steps"},
            "e2e": {"value": value, "unit": "PE/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="source batch width B (0 = auto)")
    ap.add_argument("--sample-shards", type=int, default=0,
                    help="evaluate 1/S of the batches (default: 16 for cfg5 on one GPU, else 1)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-north-star", dest="north_star", action="store_false",
                    help="skip the whole-RMAT-24 (a|b)*c* north-star measurement")
    ap.add_argument("--no-cfg3", dest="cfg3", action="store_false", help="skip the LDBC SF10 cfg3 measurement")
    ap.add_argument("--no-pairs", action="store_true", help="skip the PAIRS-mode measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.sample_shards == 0:
        args.sample_shards = 16 if (args.workload == "cfg5" and args.gpus == 1) else 1
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
