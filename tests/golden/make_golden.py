"""Generate golden vectors by running the REAL reference (`enerflow`) here.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden_small.json: for every instance the graph JSON, the
cost database, and what the reference computes — canonical hash, per-rule
match sites, every rewrite's hash in (rule, site) order, the deduplicated
neighbour sequence, inner-search results under several cost functions and
full outer-search runs including the explored-hash sequence (captured by
wrapping reference `search.neighbors`, which is called once per expansion).

The checked-in oracle (oracle/enerflow_oracle.py) and the GPU path are both
tested against this file.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

import enerflow  # noqa: E402  (the reference, via PYTHONPATH)
import enerflow.search as ref_search  # noqa: E402
from enerflow import (  # noqa: E402
    CostDatabase, CostFunction, SearchConfig, SyntheticProfiler, canonical_hash, default_rules,
    ensure_profiled, graph_to_json, inner_search, match_rule, apply, neighbors, outer_search,
    signatures, SpaceTooLarge,
)
from enerflow.cost import normalization_refs  # noqa: E402
from enerflow.models import (  # noqa: E402
    chain_graph, coordinated_witness, microbench_database, microbench_graph, random_graph,
    toy_resnet, toy_squeeze, valley_instance,
)

assert "reference" in enerflow.__file__, enerflow.__file__


def _db_rows(db: CostDatabase):
    return [[sig, alg, rec.time_ms, rec.power_w] for (sig, alg), rec in sorted(db.records().items())]


def _fn_spec(f: CostFunction):
    return {"kind": f.kind, "w": f.w, "mix": list(f.mix_weights), "refs": [f.t_ref, f.e_ref, f.p_ref]}


def _traced_outer(g, rules, db, f, cfg, profiler, use_inner=True):
    trace = []
    real = ref_search.neighbors

    def spy(graph, rs):
        trace.append(canonical_hash(graph))
        return real(graph, rs)

    ref_search.neighbors = spy
    try:
        res = outer_search(g, rules, db, f, cfg, profiler, use_inner=use_inner)
    finally:
        ref_search.neighbors = real
    stats = {k: v for k, v in vars(res.stats).items() if k != "wall_time_ms"}
    return {
        "hash": canonical_hash(res.graph), "graph": graph_to_json(res.graph),
        "assignment": {str(k): v for k, v in sorted(res.assignment.items())},
        "cost": res.cost, "time_ms": res.time_ms, "energy": res.energy, "power_w": res.power_w,
        "stats": stats, "trace": [str(h) for h in trace],
    }


def _instance(name, g, db, seed, searches, inner_fns, rule_names=None):
    rules = [r for r in default_rules() if rule_names is None or r.name in rule_names]
    db_before = _db_rows(db)
    sites = {}
    rewrites = []
    for rule in rules:
        ss = match_rule(rule, g)
        sites[rule.name] = [[v for _, v in s.binding] for s in ss]
        for s in ss:
            rewrites.append([rule.name, str(canonical_hash(apply(rule, g, s)))])
    nb = [str(canonical_hash(c)) for c in neighbors(g, rules)]
    inner = []
    for f, d in inner_fns:
        a = inner_search(g, db, f, d)
        assign, cost, t, e, evals, sweeps = ref_search._sweep(g, db, f, d)
        assert assign == a
        inner.append({"fn": _fn_spec(f), "d": d, "assignment": {str(k): v for k, v in sorted(a.items())},
                      "cost": cost, "time_ms": t, "energy": e, "evals": evals, "sweeps": sweeps})
    runs = []
    for f, cfg_kw, use_inner in searches:
        cfg = SearchConfig(**cfg_kw)
        db_run = CostDatabase()
        for sig, alg, t, p in db_before:
            db_run.add(sig, alg, enerflow.CostRecord(t, p))
        prof = SyntheticProfiler(seed) if seed is not None else None
        try:
            out = _traced_outer(g, rules, db_run, f, cfg, prof, use_inner)
        except enerflow.EnerflowError as exc:
            out = {"error": type(exc).__name__}
        out.update({"fn": _fn_spec(f), "cfg": cfg_kw, "use_inner": use_inner})
        runs.append(out)
    space = None
    if seed is not None:  # search.py:275-329 closure and its exhaustive oracle (<= 2000 graphs)
        db_bf = CostDatabase()
        for sig, alg, t, p in db_before:
            db_bf.add(sig, alg, enerflow.CostRecord(t, p))
        try:
            members = ref_search.closure(g, rules, 2000)
            bf = ref_search.brute_force_space(g, rules, db_bf, CostFunction.energy(), max_graphs=2000,
                                              profiler=SyntheticProfiler(seed))
            space = {"closure": [str(canonical_hash(m)) for m in members], "hash": str(canonical_hash(bf.graph)),
                     "cost": bf.cost, "assignment": {str(k): v for k, v in sorted(bf.assignment.items())}}
        except SpaceTooLarge:
            space = {"error": "SpaceTooLarge"}
    return {
        "space": space,
        "name": name, "rules": [r.name for r in rules], "graph": graph_to_json(g), "db": db_before, "seed": seed,
        "hash": str(canonical_hash(g)),
        "signatures": {str(k): s.text for k, s in signatures(g).items()},
        "sites": sites, "rewrites": rewrites, "neighbors": nb, "inner": inner, "searches": runs,
    }


def main():
    out = []
    lin = lambda g, db, w: CostFunction.linear(w).with_refs(*normalization_refs(g, db))  # noqa: E731

    g, db = microbench_graph(), microbench_database()
    out.append(_instance("microbench", g, db, None,
                         [(CostFunction.energy(), {"alpha": 1.05}, True),
                          (CostFunction.time(), {"alpha": 1.05}, True)],
                         [(CostFunction.energy(), 1), (CostFunction.time(), 1), (CostFunction.power(), 1),
                          (CostFunction.power(), 2), (lin(g, db, 0.5), 1), (CostFunction.product(0.5), 2)]))

    g, db, _ = valley_instance()
    out.append(_instance("valley", g, db, None,
                         [(CostFunction.energy(), {"alpha": 1.0}, True),
                          (CostFunction.energy(), {"alpha": 1.5}, True)],
                         [(CostFunction.energy(), 1)], ["fuse-conv-relu", "merge-parallel-convs"]))
    out.append(_instance("valley-all-rules", g, db, None,
                         [(CostFunction.energy(), {"alpha": 1.5}, True)], [(CostFunction.energy(), 1)]))

    g, db = coordinated_witness()
    out.append(_instance("witness", g, db, None, [],
                         [(CostFunction.product(0.5), 1), (CostFunction.product(0.5), 2),
                          (CostFunction.power(), 1)]))

    for name, builder in (("toy-squeeze", toy_squeeze), ("toy-resnet", toy_resnet),
                          ("chain3", lambda s: chain_graph(3, s))):
        g = builder(0)
        db = CostDatabase()
        ensure_profiled(g, db, SyntheticProfiler(0))
        out.append(_instance(name, g, db, 0,
                             [(CostFunction.energy(), {"alpha": 1.05}, True),
                              (CostFunction.energy(), {"alpha": 1.2}, False),
                              (lin(g, db, 0.5), {"alpha": 1.05, "d": 1}, True),
                              (CostFunction.power(), {"alpha": 1.0, "d": 2}, True)],
                             [(CostFunction.energy(), 1), (lin(g, db, 0.3), 1), (CostFunction.power(), 2)]))

    for seed in range(40):
        g = random_graph(seed, max_ops=8)
        db = CostDatabase()
        ensure_profiled(g, db, SyntheticProfiler(seed))
        searches = [(CostFunction.energy(), {"alpha": 1.3}, True)]
        if seed % 4 == 0:
            searches.append((lin(g, db, 0.7), {"alpha": 1.05}, True))
        if seed % 4 == 1:
            searches.append((CostFunction.time(), {"alpha": 1.0, "max_queue": 2}, True))
        if seed % 4 == 2:
            searches.append((CostFunction.mix(power=0.5, energy=0.5), {"alpha": 1.1, "d": 2}, True))
        if seed % 4 == 3:
            searches.append((CostFunction.energy(), {"alpha": 2.0, "max_graph_nodes": len(g.compute_nodes())}, True))
        out.append(_instance(f"random-{seed}", g, db, seed, searches,
                             [(CostFunction.energy(), 1), (CostFunction.linear(0.3), 1),
                              (CostFunction.power(), 2)]))

    path = os.path.join(HERE, "golden_small.json")
    with open(path, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py", "python": sys.version.split()[0],
                   "instances": out}, fh, sort_keys=True)
    print(f"wrote {path}: {len(out)} instances")


if __name__ == "__main__":
    main()
