"""cProfile of a warm end-to-end GPU search (the device session already initialised)."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402

name, alpha = (sys.argv[1], float(sys.argv[2])) if len(sys.argv) > 2 else ("squeezenet", 1.0)
g = zoo.generate(name, 0)


def run():
    return ef.outer_search(g, ef.default_rules(), ef.CostDatabase(), ef.CostFunction.energy(),
                           ef.SearchConfig(alpha=alpha), ef.SyntheticProfiler(0))


run()  # warm: session, tables, kernels
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = run()
pr.disable()
print(f"== {name} alpha={alpha}: {time.perf_counter() - t0:.3f}s explored={res.stats.graphs_explored}", flush=True)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
