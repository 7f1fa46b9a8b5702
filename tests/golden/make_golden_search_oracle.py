"""Full-search goldens for BASELINE configs[1-3], made by the pinned oracle on several host cores.

    python tests/golden/make_golden_search_oracle.py resnet50 energy 1.05 max_expansions [workers]

The oracle (oracle/enerflow_oracle.py) is pinned to the real reference by
tests/test_oracle_golden.py / test_oracle_models.py; oracle/parallel_search.py
runs its outer search (search.py:211-272) across worker processes with the
identical result (tests/test_oracle_parallel.py).

At alpha = 1.05 these searches do not end in any practical time (nearly every
rewrite of a graph near the optimum stays within 5% of it, so the queue never
drains: the reference itself runs for days), so the run is the reference's
search stopped at its `max_expansions`-th pop (SearchConfig.max_expansions; the
oracle's `max_expansions`): every quantity below is the reference's state at
that point.  Recorded: the explored-hash
sequence, the optimised graph's hash, its rewrite path from the origin, the
assignment (ascending node id), cost / time / energy and every SearchStats
counter, for a zoo model (seed 0) under SyntheticProfiler(0).  Objectives:
`energy`, or `linear0.5` = linear(w=0.5) over the origin's normalization_refs
(cost.py:284-296; BASELINE configs[2]'s energy-delay tradeoff).  Output:
tests/golden/golden_search_<model>_<objective>_a<alpha>[_q<max_queue>].json.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, ROOT)

from oracle import enerflow_oracle as orc  # noqa: E402
from oracle import parallel_search as ps  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402

RULES = ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs", "split-merged-conv", "fold-identity",
         "fuse-conv-batchnorm"]


def to_oracle(g):
    nodes = {nid: {"kind": v.kind.value, "ins": [(r.node, r.port) for r in v.inputs], "p": dict(v.params),
                   "w": dict(v.weights)} for nid, v in g.nodes.items()}
    return {"inputs": [(n, tuple(s.dims)) for n, s in g.inputs], "nodes": nodes,
            "outputs": [(r.node, r.port) for r in g.outputs]}


def graph_nodes(g):
    """The optimised graph without its weights: [id, kind, inputs, params] per node (ascending id),
    and the outputs (the weights are covered by the canonical hash)."""
    def plain(v):
        return list(v) if isinstance(v, tuple) else v

    nodes = [[n, v["kind"], [list(r) for r in v["ins"]], {k: plain(x) for k, x in sorted(v["p"].items())}]
             for n, v in sorted(g["nodes"].items())]
    return {"nodes": nodes, "outputs": [list(r) for r in g["outputs"]]}


def objective(kind, g):
    if kind == "energy":
        return orc.CostFn("energy")
    if kind == "linear0.5":
        db = orc.CostDB()
        orc.ensure_profiled(g, db, 0)
        return orc.CostFn("linear", w=0.5, refs=orc.normalization_refs(g, db))
    raise ValueError(kind)


def main():
    model, kind, alpha = sys.argv[1], sys.argv[2], float(sys.argv[3])
    max_exp = int(sys.argv[4])
    workers = int(sys.argv[5]) if len(sys.argv) > 5 else os.cpu_count()
    g = to_oracle(zoo.generate(model, 0))
    t0 = time.perf_counter()

    def progress(stats, heap):
        print(f"{time.perf_counter() - t0:8.0f}s explored {stats['graphs_explored']} generated "
              f"{stats['graphs_generated']} heap {heap} best_updates {stats['best_updates']}", flush=True)

    trace = []
    res = ps.outer_search(g, RULES, orc.CostDB(), objective(kind, g), alpha=alpha, seed=0, trace=trace,
                          workers=workers, batch=2 * workers, progress=progress, max_expansions=max_exp)
    secs = time.perf_counter() - t0
    out = {"generator": "tests/golden/make_golden_search_oracle.py (pinned oracle, parallel replay)",
           "python": sys.version.split()[0], "model": model, "seed": 0, "objective": kind, "alpha": alpha,
           "max_expansions": max_exp, "trace": [str(h) for h in trace], "hash": str(res["hash"]),
           "path": [[r, list(s)] for r, s in res["path"]],
           "assignment": [[k, res["assignment"][k]] for k in sorted(res["assignment"])],
           "graph_nodes": graph_nodes(res["graph"]),
           "cost": res["cost"], "time_ms": res["time_ms"], "energy": res["energy"], "stats": res["stats"],
           "oracle_seconds": secs, "workers": workers}
    path = os.path.join(HERE, f"golden_search_{model}_{kind}_a{alpha:g}_x{max_exp}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, sort_keys=True)
    print("wrote", path, f"{secs:.0f}s", len(trace), "expansions")


if __name__ == "__main__":
    main()
