"""GPU path vs the reference's golden vectors (tests/golden/golden_small.json).

Every quantity the north star asks to be bit-exact is compared with ==:
canonical hashes, match sites, rewrite hashes in (rule, site) order, the
deduplicated neighbour sequence, inner-search assignments / costs / evaluation
counts, and full outer-search runs (explored-hash sequence, optimised graph,
assignment, cost, time, energy, statistics).  All calls go through the
package API, which drives libef200.so (the C ABI) on cuda:0.
"""

import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import frontier, rewrite

pytestmark = pytest.mark.gpu


def _db(inst):
    db = ef.CostDatabase()
    for sig, alg, t, p in inst["db"]:
        db.add(sig, alg, ef.CostRecord(t, p))
    return db


def _fn(spec):
    f = ef.CostFunction(spec["kind"], w=spec["w"], mix_weights=tuple(spec["mix"]))
    return f.with_refs(*spec["refs"])


def _rules(inst):
    return [r for r in ef.default_rules() if r.name in inst["rules"]]


def test_canonical_hash(golden_small):
    for inst in golden_small:
        g = ef.graph_from_json(inst["graph"])
        assert str(ef.canonical_hash(g)) == inst["hash"], inst["name"]


def test_match_sites_and_rewrites(golden_small):
    for inst in golden_small:
        g = ef.graph_from_json(inst["graph"])
        got_rw = []
        for rule in _rules(inst):
            sites = ef.match_rule(rule, g)
            assert [[v for _, v in s.binding] for s in sites] == inst["sites"][rule.name], (inst["name"], rule.name)
            for s in sites:
                got_rw.append([rule.name, str(ef.canonical_hash(ef.apply(rule, g, s)))])
        assert got_rw == inst["rewrites"], inst["name"]


def test_neighbors(golden_small):
    for inst in golden_small:
        g = ef.graph_from_json(inst["graph"])
        nb = [str(ef.canonical_hash(c)) for c in ef.neighbors(g, _rules(inst))]
        assert nb == inst["neighbors"], inst["name"]


def test_inner_search(golden_small):
    for inst in golden_small:
        g = ef.graph_from_json(inst["graph"])
        db = _db(inst)
        for case in inst["inner"]:
            r, assign = frontier._price_one(g, db, _fn(case["fn"]), case["d"], True)
            where = (inst["name"], case["fn"]["kind"], case["d"])
            assert {str(k): v for k, v in assign.items()} == case["assignment"], where
            # product too: pow_py is a double-double log/exp, correctly rounded like CPython's **
            assert (r.cost, r.time_ms, r.energy) == (case["cost"], case["time_ms"], case["energy"]), where
            assert (r.evals, r.sweeps) == (case["evals"], case["sweeps"]), where


@pytest.mark.parametrize("batch", [1, 5, 64])
def test_outer_search(golden_small, batch):
    """Full searches against the reference's goldens for every expansion batch size: the batched,
    speculative expansion replayed in the reference's pop order changes nothing observable, and
    the step's device alpha-prune flags equal the replay's decisions (check_prune)."""
    for inst in golden_small:
        g = ef.graph_from_json(inst["graph"])
        for run in inst["searches"]:
            db = _db(inst)
            cfg = ef.SearchConfig(**run["cfg"])
            prof = ef.SyntheticProfiler(inst["seed"]) if inst["seed"] is not None else None
            where = (inst["name"], run["cfg"], run["fn"]["kind"])
            if "error" in run:
                with pytest.raises(ef.MissingEntry):
                    ef.outer_search(g, _rules(inst), db, _fn(run["fn"]), cfg, prof, use_inner=run["use_inner"],
                                    batch=batch)
                continue
            trace = []
            res = ef.outer_search(g, _rules(inst), db, _fn(run["fn"]), cfg, prof, use_inner=run["use_inner"],
                                  trace=trace, batch=batch, check_prune=True)
            assert [str(h) for h in trace] == run["trace"], where
            assert ef.canonical_hash(res.graph) == run["hash"], where
            assert ef.graph_to_json(res.graph) == run["graph"], where
            assert {str(k): v for k, v in res.assignment.items()} == run["assignment"], where
            assert (res.cost, res.time_ms, res.energy) == (run["cost"], run["time_ms"], run["energy"]), where
            stats = {k: v for k, v in vars(res.stats).items() if k != "wall_time_ms"}
            assert stats == run["stats"], where
