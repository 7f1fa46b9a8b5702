"""Time end-to-end GPU searches (outer_search) on the evaluation models."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402

out = []
for name, alpha in [("squeezenet", 1.0), ("squeezenet", 1.05), ("resnet50", 1.0), ("resnet50", 1.05),
                    ("inception_v3", 1.0), ("inception_v3", 1.05), ("nasnet_a", 1.0)]:
    g = zoo.generate(name, 0)
    db = ef.CostDatabase()
    t0 = time.perf_counter()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    t1 = time.perf_counter()
    trace = []
    res = ef.outer_search(g, ef.default_rules(), db, ef.CostFunction.energy(), ef.SearchConfig(alpha=alpha),
                          ef.SyntheticProfiler(0), trace=trace)
    t2 = time.perf_counter()
    st = res.stats
    row = {"model": name, "alpha": alpha, "search_s": t2 - t1, "profile_s": t1 - t0, "explored": st.graphs_explored,
           "generated": st.graphs_generated, "cost": res.cost, "nodes": len(res.graph.nodes),
           "hash": ef.canonical_hash(res.graph)}
    out.append(row)
    print(json.dumps(row), flush=True)
