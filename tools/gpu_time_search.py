"""Time end-to-end GPU searches on the evaluation models (development aid)."""
import sys, time
sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo
for name, alpha in [("squeezenet", 1.0), ("resnet50", 1.0), ("inception_v3", 1.0)]:
    g = zoo.generate(name, 0)
    db = ef.CostDatabase()
    t0 = time.perf_counter()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    t1 = time.perf_counter()
    res = ef.outer_search(g, ef.default_rules(), db, ef.CostFunction.energy(), ef.SearchConfig(alpha=alpha),
                          ef.SyntheticProfiler(0))
    t2 = time.perf_counter()
    st = res.stats
    print(f"{name} alpha={alpha}: search {t2-t1:.2f}s (profile {t1-t0:.2f}s) explored={st.graphs_explored} "
          f"generated={st.graphs_generated} cost {res.cost:.6g} nodes {len(res.graph.nodes)}", flush=True)
