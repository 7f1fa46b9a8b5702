"""Pin the oracle to the real reference: every golden vector in
tests/golden/golden_small.json (made by tests/golden/make_golden.py, which
imports the reference) must be reproduced exactly by oracle/enerflow_oracle.py.
"""

import math
import random

import pytest

from oracle import enerflow_oracle as orc


def _db(inst):
    db = orc.CostDB()
    for sig, alg, t, p in inst["db"]:
        db.add(sig, alg, t, p)
    return db


def _fn(spec):
    return orc.CostFn(spec["kind"], spec["w"], spec["mix"], spec["refs"])


def test_neumaier_matches_builtin_sum():
    rng = random.Random(5)
    for _ in range(2000):
        xs = [rng.uniform(-1, 1) * 10 ** rng.randint(-8, 8) for _ in range(rng.randint(1, 40))]
        assert orc.neumaier_sum(xs) == sum(xs)
        pos = [abs(x) for x in xs]
        assert orc.neumaier_sum(pos) == sum(pos)


def test_hash_signatures_sites(golden_small):
    for inst in golden_small:
        g = orc.from_json(inst["graph"])
        assert str(orc.canonical_hash(g)) == inst["hash"], inst["name"]
        texts = orc.sig_texts(g)
        assert {str(k): v for k, v in texts.items()} == inst["signatures"], inst["name"]
        for rule in inst["rules"]:
            assert [orc.binding(rule, s) for s in orc.match(rule, g)] == inst["sites"][rule], (inst["name"], rule)


def test_rewrites_and_neighbors(golden_small):
    for inst in golden_small:
        g = orc.from_json(inst["graph"])
        got = []
        for rule in inst["rules"]:
            for site in orc.match(rule, g):
                got.append([rule, str(orc.canonical_hash(orc.apply(rule, g, site)))])
        assert got == inst["rewrites"], inst["name"]
        nb = [str(orc.canonical_hash(c)) for c in orc.neighbors(g, inst["rules"])]
        assert nb == inst["neighbors"], inst["name"]


def test_inner_search(golden_small):
    for inst in golden_small:
        g = orc.from_json(inst["graph"])
        db = _db(inst)
        for case in inst["inner"]:
            a, cost, t, e, ev, sw = orc.sweep(g, db, _fn(case["fn"]), case["d"])
            assert {str(k): v for k, v in a.items()} == case["assignment"], inst["name"]
            assert (cost, t, e, ev, sw) == (case["cost"], case["time_ms"], case["energy"],
                                            case["evals"], case["sweeps"]), inst["name"]


def test_outer_search_traces(golden_small):
    for inst in golden_small:
        g = orc.from_json(inst["graph"])
        for run in inst["searches"]:
            db = _db(inst)
            cfg = dict(run["cfg"])
            trace = []
            kw = dict(alpha=cfg.get("alpha", 1.05), d=cfg.get("d", 1), max_queue=cfg.get("max_queue", 100_000),
                      max_graph_nodes=cfg.get("max_graph_nodes"), seed=inst["seed"],
                      use_inner=run["use_inner"], trace=trace)
            if "error" in run:
                with pytest.raises(orc.MissingEntry):
                    orc.outer_search(g, inst["rules"], db, _fn(run["fn"]), **kw)
                continue
            res = orc.outer_search(g, inst["rules"], db, _fn(run["fn"]), **kw)
            where = (inst["name"], run["cfg"])
            assert [str(h) for h in trace] == run["trace"], where
            assert res["hash"] == run["hash"], where
            assert {str(k): v for k, v in res["assignment"].items()} == run["assignment"], where
            assert (res["cost"], res["time_ms"], res["energy"]) == (run["cost"], run["time_ms"], run["energy"]), where
            assert res["stats"] == {k: run["stats"][k] for k in orc.STAT_KEYS}, where
