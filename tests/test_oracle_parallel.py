"""The multi-process oracle search (oracle/parallel_search.py, used to make the long-search
goldens) returns exactly what the single-process oracle search returns."""

import pytest

from oracle import enerflow_oracle as orc
from oracle import parallel_search as ps
from paper_2005_05837_b200 import zoo

RULES = ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs", "split-merged-conv", "fold-identity",
         "fuse-conv-batchnorm"]


def to_oracle(g):
    nodes = {nid: {"kind": v.kind.value, "ins": [(r.node, r.port) for r in v.inputs], "p": dict(v.params),
                   "w": dict(v.weights)} for nid, v in g.nodes.items()}
    return {"inputs": [(n, tuple(s.dims)) for n, s in g.inputs], "nodes": nodes,
            "outputs": [(r.node, r.port) for r in g.outputs]}


@pytest.mark.parametrize("model,alpha,kind,max_queue,max_exp", [("toy_squeeze", 1.05, "energy", 100_000, None),
                                                                ("squeezenet", 1.0, "energy", 100_000, None),
                                                                ("toy_squeeze", 1.1, "linear", 7, None),
                                                                ("squeezenet", 1.05, "energy", 100_000, 40)])
def test_parallel_oracle_search_equals_oracle(model, alpha, kind, max_queue, max_exp):
    g = to_oracle(zoo.toy_squeeze(0) if model == "toy_squeeze" else zoo.generate(model, 0))
    if kind == "linear":
        db0 = orc.CostDB()
        orc.ensure_profiled(g, db0, 0)
        fn = orc.CostFn("linear", w=0.5, refs=orc.normalization_refs(g, db0))
    else:
        fn = orc.CostFn(kind)
    runs = []
    for impl in (orc.outer_search, ps.outer_search):
        db = orc.CostDB()
        trace = []
        kw = {"workers": 3, "batch": 5} if impl is ps.outer_search else {}
        res = impl(g, RULES, db, fn, alpha=alpha, seed=0, max_queue=max_queue, trace=trace, max_expansions=max_exp,
                   **kw)
        runs.append((trace, res["hash"], res["assignment"], res["cost"], res["time_ms"], res["energy"],
                     res["stats"], sorted(db.rows)))
    assert runs[0] == runs[1]
