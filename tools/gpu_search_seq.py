"""The bench's end-to-end searches (bench.SEARCHES) in one process, in order, each capped at
CAP expansions (debugging / sanitizer runs).  Usage: python tools/gpu_search_seq.py CAP [skip_frontiers]"""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402
from paper_2005_05837_b200.frontier import Frontier  # noqa: E402

cap = int(sys.argv[1])
if len(sys.argv) < 3:  # the bench's frontier workloads first, as bench.py runs them
    for w, n in (("dag:20000", 4), ("resnet50", 256)):
        g0 = zoo.generate(w, 0)
        db = ef.CostDatabase()
        ef.ensure_profiled(g0, db, ef.SyntheticProfiler(0))
        fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), n)
        fr.step()
        fr.close()
        print("frontier", w, "ok", flush=True)
for model, obj, alpha, max_exp, golden in bench.SEARCHES:
    g = zoo.generate(model, 0)
    db = ef.CostDatabase()
    t0 = time.perf_counter()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    f = bench._objective(ef, obj, g, db)
    res = ef.outer_search(g, ef.default_rules(), db, f,
                          ef.SearchConfig(alpha=alpha, max_expansions=min(cap, max_exp or cap)),
                          ef.SyntheticProfiler(0))
    print(model, res.stats.graphs_explored, f"{time.perf_counter() - t0:.2f}s", flush=True)
