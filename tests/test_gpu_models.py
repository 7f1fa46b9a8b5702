"""Model-scale parity of the frontier step (the bench workload) against the oracle.

For real frontier parents of each evaluation model (the graphs the best-first
search enqueues first), every candidate of one batched `ef_expand` is checked:
its (rule, site) sequence per parent and its canonical hash against the oracle's
`match` / `apply` / `canonical_hash` (pinned to the reference by
tests/test_oracle_golden.py), and every priced candidate's cost, time, energy,
evaluation and sweep counts against the oracle's inner search — all with ==.
"""

import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import _native as N
from paper_2005_05837_b200 import zoo
from paper_2005_05837_b200.frontier import Frontier

pytestmark = pytest.mark.gpu

RULES = [r.name for r in ef.default_rules()]


def to_oracle(g):
    nodes = {nid: {"kind": v.kind.value, "ins": [(r.node, r.port) for r in v.inputs], "p": dict(v.params),
                   "w": dict(v.weights)} for nid, v in g.nodes.items()}
    return {"inputs": [(n, tuple(s.dims)) for n, s in g.inputs], "nodes": nodes,
            "outputs": [(r.node, r.port) for r in g.outputs]}


def oracle_db(db):
    from oracle import enerflow_oracle as orc

    odb = orc.CostDB()
    for (sig, alg), rec in db.records().items():
        odb.add(sig, alg, rec.time_ms, rec.power_w)
    return odb


@pytest.mark.parametrize("model,n_parents,price_every", [("squeezenet", 12, 1), ("resnet50", 6, 3),
                                                          ("inception_v3", 3, 7), ("nasnet_a", 2, 13)])
def test_frontier_step_matches_oracle(model, n_parents, price_every):
    from oracle import enerflow_oracle as orc

    g0 = zoo.generate(model, 0)
    db = ef.CostDatabase()
    prof = ef.SyntheticProfiler(0)
    f = ef.CostFunction.energy()
    fr = Frontier(g0, db, prof, f, ef.SearchConfig(alpha=1.05), n_parents)
    try:
        res = fr.step()
        parents = [fr.decode(sl) for sl in fr.slots]
    finally:
        fr.close()
    odb = oracle_db(db)
    rule_names = {i: r.name for i, r in enumerate(ef.default_rules())}
    checked = priced = 0
    for pi, pg in enumerate(parents):
        og = to_oracle(pg)
        ids = sorted(og["nodes"])
        want = [(rule, site) for rule in RULES for site in orc.match(rule, og)]
        mine = res[res["parent"] == pi]
        got = []
        for r in mine:
            name = rule_names[int(r["rule"])]
            width = len(orc.SITE_NAMES[name])
            got.append((name, tuple(ids[int(x)] for x in (r["site_a"], r["site_b"])[:width])))
        assert got == want, (model, pi)
        for k, ((rule, site), r) in enumerate(zip(want, mine)):
            child = orc.apply(rule, og, site)
            assert int(r["hash"]) == orc.canonical_hash(child), (model, pi, rule, site)
            assert int(r["n_nodes"]) == len(child["nodes"])
            checked += 1
            if r["flags"] & N.F_PRICED and k % price_every == 0:
                orc.ensure_profiled(child, odb, 0)
                _, cost, t, e, evals, sweeps = orc.sweep(child, odb, orc.CostFn("energy"), 1)
                assert (float(r["cost"]), float(r["time_ms"]), float(r["energy"])) == (cost, t, e), (model, rule)
                assert (int(r["evals"]), int(r["sweeps"])) == (evals, sweeps)
                priced += 1
    assert checked == len(res) and priced > 0
