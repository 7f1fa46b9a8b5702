"""cProfile of end-to-end GPU searches (host-side overhead hunt)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402

for name, alpha in [("squeezenet", 1.0), ("resnet50", 1.0)]:
    g = zoo.generate(name, 0)
    db = ef.CostDatabase()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    res = ef.outer_search(g, ef.default_rules(), db, ef.CostFunction.energy(), ef.SearchConfig(alpha=alpha),
                          ef.SyntheticProfiler(0))
    pr.disable()
    print(f"== {name} alpha={alpha}: {time.perf_counter() - t0:.2f}s explored={res.stats.graphs_explored} "
          f"generated={res.stats.graphs_generated}", flush=True)
    pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
    pstats.Stats(pr).sort_stats("tottime").print_stats(15)
