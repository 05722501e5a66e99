"""Small evaluations for compute-sanitizer (memcheck / racecheck / synccheck):
the toy graph and a 5,000-vertex random graph with a hub row, host-driven
level loop (RPQ_HOST_LOOP=1, every kernel a visible launch), both engines,
bottom-up levels, PAIRS / PER_SOURCE / COUNT, a length-bounded query and a
CRPQ.  Results are checked against the oracle so a silent corruption fails.
Usage: compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("RPQ_HOST_LOOP", "1")

import oracle  # noqa: E402
import paper_2602_20748_b200 as R  # noqa: E402
import synth  # noqa: E402


def check(G, g, rx, **kw):
    a = R.rpq_compile(G, rx)
    r = R.rpq_eval_allpairs(G, a, mode=R.RPQ_PAIRS | R.RPQ_STATS, **kw)
    o = oracle.allpairs(g, rx, max_hops=kw.get("max_hops"))
    want = np.stack([o["src"], o["dst"]], 1).astype(np.uint32)
    assert np.array_equal(r.rows(), want), (rx, kw)
    assert r.stats()["product_edges"] == int(o["pe"].sum()), (rx, kw)
    c = R.rpq_eval_allpairs(G, a, mode=R.RPQ_COUNT | R.RPQ_PE, **kw)
    assert c.count == len(want), (rx, kw)


toy = synth.toy_graph()
Gt = R.rpq_graph_load(toy, in_edges=True)
for rx in ["abc*", "(a|b)*c*", "c+"]:
    check(Gt, toy, rx)
q = R.crpq(Gt, ["u2", "u3", "u4"], [("u3", "ab", "u2"), ("u3", "ab", "u4"), ("u2", "c*", "u4")],
           var_label={"u2": "D", "u3": "A", "u4": "D"})
assert q.count == 4

rng = np.random.default_rng(5)
g = synth.random_graph(5000, 20000, 3, seed=5)
hub = rng.choice(5000, 700, replace=False).astype(np.uint32)
g = synth.Graph(5000, np.concatenate([g.src, np.zeros(700, np.uint32)]), np.concatenate([g.dst, hub]),
                np.concatenate([g.label, np.zeros(700, np.uint16)]), g.label_names).check()
G = R.rpq_graph_load(g, in_edges=True)
for eng in ["dense", "sparse"]:
    os.environ["RPQ_ENGINE"] = eng
    for rx in ["(a|b)*c*", "a b* c"]:
        check(G, g, rx, batch_sources=2048)
os.environ.pop("RPQ_ENGINE")
os.environ["RPQ_PULL"] = "always"
check(G, g, "(a|b)*c", batch_sources=2048)
os.environ.pop("RPQ_PULL")
check(G, g, "a b* c", batch_sources=256, max_hops=3)
# TMA bulk-copy ring in k_level and k_level_hub (all 5,000 sources: 3 chunks per row)
os.environ["RPQ_ENGINE"] = "dense"
os.environ["RPQ_TMA"] = "3"
check(G, g, "(a|b)*c*")
os.environ.pop("RPQ_TMA")
os.environ.pop("RPQ_ENGINE")
print("sanitize workload OK")
