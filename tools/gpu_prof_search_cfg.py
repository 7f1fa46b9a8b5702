"""cProfile of a warm batched outer_search of one BASELINE config.
Usage: python tools/gpu_prof_search_cfg.py MODEL OBJECTIVE ALPHA MAX_EXPANSIONS BATCH"""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402

model, obj, alpha, max_exp, batch = sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
g = zoo.generate(model, 0)


def run():
    db = ef.CostDatabase()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    f = ef.CostFunction.energy() if obj == "energy" else \
        ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g, db))
    return ef.outer_search(g, ef.default_rules(), db, f, ef.SearchConfig(alpha=alpha, max_expansions=max_exp),
                           ef.SyntheticProfiler(0), batch=batch)


t0 = time.perf_counter()
run()
print(f"cold {time.perf_counter() - t0:.3f}s", flush=True)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = run()
pr.disable()
print(f"== {model} {obj} alpha={alpha}: warm {time.perf_counter() - t0:.3f}s explored={res.stats.graphs_explored}",
      flush=True)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
