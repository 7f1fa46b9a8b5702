import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo
g = zoo.generate("resnet50", 0)
db = ef.CostDatabase()
ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
pr = cProfile.Profile()
pr.enable()
res = ef.outer_search(g, ef.default_rules(), db, ef.CostFunction.energy(), ef.SearchConfig(alpha=1.0), ef.SyntheticProfiler(0))
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
