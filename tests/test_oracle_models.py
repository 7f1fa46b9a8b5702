"""The oracle at model scale against golden vectors from the real reference
(tests/golden/golden_models.json, made by tests/golden/make_golden_models.py):
per-rule sites, every rewrite's canonical hash, the neighbour sequence, the
synthetic cost table and the energy inner search of the origin graph, and the
full traced SqueezeNet search (BASELINE configs[0])."""

import hashlib
import json
import os

import pytest

from oracle import enerflow_oracle as orc
from paper_2005_05837_b200 import zoo

HERE = os.path.dirname(os.path.abspath(__file__))
RULES = ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs", "split-merged-conv", "fold-identity",
         "fuse-conv-batchnorm"]


def golden(model):
    with open(os.path.join(HERE, "golden", "golden_models.json")) as fh:
        return {i["model"]: i for i in json.load(fh)["instances"]}[model]


def to_oracle(g):
    nodes = {nid: {"kind": v.kind.value, "ins": [(r.node, r.port) for r in v.inputs], "p": dict(v.params),
                   "w": dict(v.weights)} for nid, v in g.nodes.items()}
    return {"inputs": [(n, tuple(s.dims)) for n, s in g.inputs], "nodes": nodes,
            "outputs": [(r.node, r.port) for r in g.outputs]}


@pytest.mark.parametrize("model", ["squeezenet", "resnet50"])
def test_oracle_matches_reference_at_model_scale(model):
    gold = golden(model)
    g = to_oracle(zoo.generate(model, 0))
    assert str(orc.canonical_hash(g)) == gold["hash"]
    rewrites = []
    for rule in RULES:
        sites = orc.match(rule, g)
        assert [orc.binding(rule, s) for s in sites] == gold["sites"][rule], rule
        rewrites += [str(orc.canonical_hash(orc.apply(rule, g, s))) for s in sites]
    assert rewrites == gold["rewrites"]
    assert [str(orc.canonical_hash(c)) for c in orc.neighbors(g, RULES)] == gold["neighbors"]
    db = orc.CostDB()
    orc.ensure_profiled(g, db, 0)
    h = hashlib.sha256()
    for sig in sorted(db.rows):
        for alg in sorted(db.rows[sig]):
            t, p = db.rows[sig][alg]
            h.update(f"{sig}|{alg}|{t!r}|{p!r}\n".encode())
    assert h.hexdigest() == gold["db_sha256"]
    assign, cost, t, e, evals, sweeps = orc.sweep(g, db, orc.CostFn("energy"), 1)
    inner = gold["inner_energy_d1"]
    assert [assign[k] for k in sorted(assign)] == inner["assignment"]
    assert (cost, t, e, evals, sweeps) == (inner["cost"], inner["time_ms"], inner["energy"], inner["evals"],
                                           inner["sweeps"])


def test_oracle_squeezenet_search_matches_reference():
    gold = golden("squeezenet")["search"]
    g = to_oracle(zoo.generate("squeezenet", 0))
    trace = []
    res = orc.outer_search(g, RULES, orc.CostDB(), orc.CostFn("energy"), alpha=gold["alpha"], seed=0, trace=trace)
    assert [str(h) for h in trace] == gold["trace"]
    assert str(res["hash"]) == gold["hash"]
    assert [res["assignment"][k] for k in sorted(res["assignment"])] == gold["assignment"]
    assert (res["cost"], res["time_ms"], res["energy"]) == (gold["cost"], gold["time_ms"], gold["energy"])
    assert res["stats"] == gold["stats"]
