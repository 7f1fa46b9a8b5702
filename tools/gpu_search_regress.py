"""Where the end-to-end search time goes: SqueezeNet alpha=1.0 cold / warm, alone and after a
large-graph session holds its scratch (the bench's order), with a cProfile of the warm run;
NasNet-A 1000 expansions."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402


def run(model, alpha, max_exp=None, prof=False):
    g = zoo.generate(model, 0)
    db = ef.CostDatabase()
    t0 = time.perf_counter()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    pr = cProfile.Profile() if prof else None
    if pr:
        pr.enable()
    f = ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g, db)) if model == "inception_v3" else ef.CostFunction.energy()
    res = ef.outer_search(g, ef.default_rules(), db, f,
                          ef.SearchConfig(alpha=alpha, max_expansions=max_exp), ef.SyntheticProfiler(0))
    if pr:
        pr.disable()
    dt = time.perf_counter() - t0
    print(f"{model} a={alpha} x={max_exp}: {dt:.3f}s explored={res.stats.graphs_explored}", flush=True)
    if pr:
        pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


which = sys.argv[1]
if which == "big":
    from paper_2005_05837_b200.frontier import Frontier
    g = zoo.generate("dag:20000", 0)
    db = ef.CostDatabase()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    fr = Frontier(g, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), 9)
    for _ in range(2):
        fr.step(fr.slots, insert_visited=False)
    fr.close()
    print("big session done", flush=True)
for model, alpha, x in [m.split(":") for m in sys.argv[2:]] if len(sys.argv) > 2 else [("squeezenet", "1.0", "0")]:
    run(model, float(alpha), int(x) or None)
    run(model, float(alpha), int(x) or None, prof=os.environ.get("PROF") == "1")
