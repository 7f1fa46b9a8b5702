"""Full searches of BASELINE configs[0-3] on the GPU against search goldens.

Goldens (tests/golden/golden_search_*.json):
  * golden_search_ref_*.json — the REAL reference's `outer_search` run here
    (tests/golden/make_golden_search_ref.py), e.g. ResNet-50 energy alpha = 1.0;
  * golden_search_<model>_<objective>_a<alpha>_x<N>.json — the pinned oracle
    (tests/golden/make_golden_search_oracle.py) for ResNet-50 energy alpha = 1.05,
    Inception-v3 linear(0.5) over normalization_refs alpha = 1.05 (energy-delay),
    NasNet-A energy alpha = 1.05.  At alpha = 1.05 these searches do not drain
    their queues in practical time, so each is the reference's search stopped at
    its N-th expansion (SearchConfig.max_expansions): every quantity is the
    reference's state at that point.

Compared with ==: the explored-hash sequence, the optimised graph (hash, node
ids, kinds, inputs, params), the per-node assignment, cost / time / energy,
every SearchStats counter; the step's device alpha-prune flags are checked
against the replay (check_prune).  Search batches of 1 and 64 parents.
"""

import glob
import json
import os

import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDENS = sorted(glob.glob(os.path.join(HERE, "golden", "golden_search_*.json")))


def _plain(v):
    if isinstance(v, (tuple, list)):
        return [_plain(x) for x in v]
    return v


def graph_nodes(g):
    nodes = [[nid, v.kind.value, [[r.node, r.port] for r in v.inputs],
              {k: _plain(x) for k, x in sorted(v.params.items())}] for nid, v in sorted(g.nodes.items())]
    return {"nodes": nodes, "outputs": [[r.node, r.port] for r in g.outputs]}


def _objective(kind, g, db):
    if kind == "energy":
        return ef.CostFunction.energy()
    assert kind == "linear0.5", kind
    return ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g, db))


@pytest.mark.parametrize("batch", [1, 64])
@pytest.mark.parametrize("path", GOLDENS, ids=[os.path.basename(p)[14:-5] for p in GOLDENS])
def test_search_matches_golden(path, batch):
    with open(path) as fh:
        gold = json.load(fh)
    if "search" in gold:  # real-reference golden (make_golden_search_ref.py)
        run = gold["search"]
        model, kind, alpha, max_exp = gold["model"], gold["objective"], run["alpha"], None
        want_assign = run["assignment"]
    else:
        run = gold
        model, kind, alpha, max_exp = gold["model"], gold["objective"], gold["alpha"], gold["max_expansions"]
        want_assign = [a for _, a in run["assignment"]]
    g = zoo.generate(model, 0)
    db0 = ef.CostDatabase()
    ef.ensure_profiled(g, db0, ef.SyntheticProfiler(0))
    f = _objective(kind, g, db0)
    trace = []
    res = ef.outer_search(g, ef.default_rules(), ef.CostDatabase(), f,
                          ef.SearchConfig(alpha=alpha, max_expansions=max_exp), ef.SyntheticProfiler(0),
                          trace=trace, batch=batch, check_prune=True)
    assert [str(h) for h in trace] == run["trace"]
    assert str(ef.canonical_hash(res.graph)) == run["hash"]
    assert [res.assignment[k] for k in sorted(res.assignment)] == want_assign
    if "graph_nodes" in run:
        assert graph_nodes(res.graph) == run["graph_nodes"]
        assert [[k, res.assignment[k]] for k in sorted(res.assignment)] == run["assignment"]
    assert (res.cost, res.time_ms, res.energy) == (run["cost"], run["time_ms"], run["energy"])
    assert {k: v for k, v in vars(res.stats).items() if k != "wall_time_ms"} == run["stats"]
