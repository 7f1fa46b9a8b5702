"""Golden vectors at model scale, made by running the REAL reference (`enerflow`) here.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_models.py

The evaluation graphs (SqueezeNet, ResNet-50, Inception-v3, NasNet-A; seed 0)
come from paper_2005_05837_b200.zoo, which builds them with the reference's
GraphBuilder semantics and random float64 weights.  Each graph is handed to the
reference as a reference `Graph` object sharing the same numpy weight arrays
(no JSON round trip: ResNet-50 alone carries 25M weights).  Recorded per model:
the canonical hash, the per-rule match sites and every rewrite's hash in
(rule, site) order, the deduplicated neighbour sequence, the synthetic cost
rows' digest, the energy inner search (d=1) of the origin, and for SqueezeNet
(BASELINE configs[0]) a full traced outer search at alpha = 1.0.  The graphs
themselves are regenerated from the zoo by the tests.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, ROOT)

import enerflow  # noqa: E402  (the reference, via PYTHONPATH)
import enerflow.search as ref_search  # noqa: E402
from enerflow import (CostDatabase, CostFunction, SearchConfig, SyntheticProfiler, apply,  # noqa: E402
                      canonical_hash, default_rules, ensure_profiled, match_rule, neighbors, outer_search)
from enerflow.graph import EdgeRef, Graph, Node, OpKind, TensorShape  # noqa: E402

assert "reference" in enerflow.__file__, enerflow.__file__

from paper_2005_05837_b200 import zoo  # noqa: E402


def to_reference(g) -> Graph:
    nodes = {nid: Node(nid, OpKind(v.kind.value), tuple(EdgeRef(r.node, r.port) for r in v.inputs), dict(v.params),
                       dict(v.weights)) for nid, v in g.nodes.items()}
    return Graph(nodes, tuple((n, TensorShape(tuple(s.dims))) for n, s in g.inputs),
                 tuple(EdgeRef(r.node, r.port) for r in g.outputs))


def db_digest(db: CostDatabase) -> str:
    h = hashlib.sha256()
    for (sig, alg), rec in sorted(db.records().items()):
        h.update(f"{sig}|{alg}|{rec.time_ms!r}|{rec.power_w!r}\n".encode())
    return h.hexdigest()


def traced_outer(g, db, alpha):
    trace = []
    real = ref_search.neighbors

    def spy(graph, rs):
        trace.append(str(canonical_hash(graph)))
        return real(graph, rs)

    ref_search.neighbors = spy
    try:
        res = outer_search(g, default_rules(), db, CostFunction.energy(), SearchConfig(alpha=alpha),
                           SyntheticProfiler(0))
    finally:
        ref_search.neighbors = real
    return {"alpha": alpha, "trace": trace, "hash": str(canonical_hash(res.graph)),
            "assignment": [res.assignment[k] for k in sorted(res.assignment)],
            "cost": res.cost, "time_ms": res.time_ms, "energy": res.energy,
            "stats": {k: v for k, v in vars(res.stats).items() if k != "wall_time_ms"},
            "seconds": res.stats.wall_time_ms / 1e3}


def main():
    out = []
    for name in ("squeezenet", "resnet50", "inception_v3", "nasnet_a"):
        t0 = time.perf_counter()
        g = to_reference(zoo.generate(name, 0))
        rules = default_rules()
        sites, rewrites = {}, []
        for rule in rules:
            ss = match_rule(rule, g)
            sites[rule.name] = [[v for _, v in s.binding] for s in ss]
            rewrites += [str(canonical_hash(apply(rule, g, s))) for s in ss]
        nb = [str(canonical_hash(c)) for c in neighbors(g, rules)]
        db = CostDatabase()
        ensure_profiled(g, db, SyntheticProfiler(0))
        assign, cost, t, e, evals, sweeps = ref_search._sweep(g, db, CostFunction.energy(), 1)
        inst = {"model": name, "seed": 0, "hash": str(canonical_hash(g)), "n_nodes": len(g.nodes),
                "sites": sites, "rewrites": rewrites, "neighbors": nb, "db_sha256": db_digest(db),
                "inner_energy_d1": {"assignment": [assign[k] for k in sorted(assign)], "cost": cost, "time_ms": t,
                                    "energy": e, "evals": evals, "sweeps": sweeps}}
        if name == "squeezenet":
            inst["search"] = traced_outer(g, CostDatabase(), 1.0)
        inst["reference_seconds"] = time.perf_counter() - t0
        out.append(inst)
        print(name, f"{inst['reference_seconds']:.1f}s", len(rewrites), "rewrites", flush=True)
    path = os.path.join(HERE, "golden_models.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden_models.py", "python": sys.version.split()[0],
                   "instances": out}, fh, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
