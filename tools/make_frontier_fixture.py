"""Record the frontier batch bench.py expands for a workload, as rewrite paths from the origin.

    python tools/make_frontier_fixture.py WORKLOAD N_PARENTS      (on a GPU box)

Writes bench_frontiers/<workload>_<n>.json: every parent of `Frontier(...)` (the graphs the
best-first search expands first) as its rewrite path (the index of each rewrite in its
parent's (rule, site) enumeration, rules.neighbors order), with its canonical hash and node
count.  `bench.py --impl reference` rebuilds the same parents on the host with the oracle from
these paths (tests/test_bench_frontier.py checks the rebuild against the hashes), so both arms
expand identical graphs.  The first k parents of an N-parent batch are the k-parent batch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402
from paper_2005_05837_b200.frontier import Frontier  # noqa: E402

workload, n = sys.argv[1], int(sys.argv[2])
name, objective, _ = bench.WORKLOADS[workload]
g0 = zoo.generate(workload, 0)
db = ef.CostDatabase()
ef.ensure_profiled(g0, db, ef.SyntheticProfiler(0))
alpha = bench.workload_alpha(workload)
fr = Frontier(g0, db, ef.SyntheticProfiler(0), bench._objective(ef, objective, g0, db), ef.SearchConfig(alpha=alpha), n)
try:
    hashes = fr.s.hash_slots(fr.slots)
    nodes = [int(fr.s.read_record(sl)[:4].view("int32")[0]) for sl in fr.slots]
    out = {"generator": "tools/make_frontier_fixture.py", "workload": workload, "config": name,
           "objective": objective, "alpha": alpha, "seed": 0, "rules": bench.RULES, "n_parents": len(fr.slots),
           "paths": [list(p) for p in fr.paths], "hashes": [str(h) for h in hashes], "nodes": nodes}
finally:
    fr.close()
path = os.path.join(bench.FRONTIER_DIR, bench.fixture_name(workload, n))
os.makedirs(os.path.dirname(path), exist_ok=True)
with open(path, "w") as fh:
    json.dump(out, fh)
print("wrote", path, len(out["paths"]), "parents, max depth", max(len(p) for p in out["paths"]))
