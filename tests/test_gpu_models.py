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


def _objectives(kind, g0, db):
    """(package CostFunction, oracle CostFn) of one objective; normalized ones use the origin's
    normalization_refs (cost.py:284-296)."""
    from oracle import enerflow_oracle as orc

    refs = ef.normalization_refs(g0, db)
    if kind == "energy":
        return ef.CostFunction.energy(), orc.CostFn("energy")
    if kind == "power":
        return ef.CostFunction.power(), orc.CostFn("power")
    if kind == "linear0.5":
        return ef.CostFunction.linear(0.5).with_refs(*refs), orc.CostFn("linear", w=0.5, refs=refs)
    if kind == "product0.3":
        return ef.CostFunction.product(0.3).with_refs(*refs), orc.CostFn("product", w=0.3, refs=refs)
    if kind == "mix":
        return (ef.CostFunction.mix(0.2, 0.5, 0.3).with_refs(*refs),
                orc.CostFn("mix", mix=(0.2, 0.5, 0.3), refs=refs))
    raise ValueError(kind)


# every k_price_v instantiation the step launches: <ENERGY|LINEAR|MIX+1 (power, product, mix), row in
# shared memory (rows <= 256) or not (Inception-v3 / NasNet-A parents)>
@pytest.mark.parametrize("model,n_parents,price_every,objective", [
    ("squeezenet", 12, 1, "energy"), ("resnet50", 6, 3, "energy"), ("inception_v3", 3, 7, "energy"),
    ("nasnet_a", 2, 13, "energy"), ("inception_v3", 3, 5, "linear0.5"), ("squeezenet", 8, 1, "power"),
    ("squeezenet", 8, 1, "product0.3"), ("squeezenet", 8, 1, "mix"), ("resnet50", 3, 4, "mix"),
    ("inception_v3", 2, 5, "product0.3"), ("nasnet_a", 1, 9, "power")])
def test_frontier_step_matches_oracle(model, n_parents, price_every, objective):
    from oracle import enerflow_oracle as orc

    g0 = zoo.generate(model, 0)
    db = ef.CostDatabase()
    prof = ef.SyntheticProfiler(0)
    ef.ensure_profiled(g0, db, prof)
    f, of = _objectives(objective, g0, db)
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
                _, cost, t, e, evals, sweeps = orc.sweep(child, odb, of, 1)
                assert (float(r["cost"]), float(r["time_ms"]), float(r["energy"])) == (cost, t, e), (model, rule)
                assert (int(r["evals"]), int(r["sweeps"])) == (evals, sweeps)
                priced += 1
    assert checked == len(res) and priced > 0


def _golden(model):
    import json
    import os

    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_models.json")) as fh:
        return {i["model"]: i for i in json.load(fh)["instances"]}[model]


@pytest.mark.parametrize("model", ["squeezenet", "resnet50", "inception_v3", "nasnet_a"])
def test_gpu_matches_reference_goldens_at_model_scale(model):
    """GPU path vs golden vectors from the real reference (make_golden_models.py)."""
    from paper_2005_05837_b200 import frontier, rewrite

    gold = _golden(model)
    g = zoo.generate(model, 0)
    assert str(ef.canonical_hash(g)) == gold["hash"]
    ids = sorted(g.nodes)
    rules = ef.default_rules()
    for s, res in rewrite._expand_one(g, rules):
        assert [str(h) for h in res["hash"].tolist()] == gold["rewrites"]
        assert [str(h) for h, fl in zip(res["hash"].tolist(), res["flags"].tolist()) if fl & N.F_FIRST] \
            == gold["neighbors"]
        for rule in rules:
            mine = res[res["rule"] == rule.rule_id]
            sites = [sorted(zip(rewrite._SITE_NAMES[rule.name], (ids[int(r["site_a"])], ids[int(r["site_b"])])))
                     for r in mine]
            assert [[v for _, v in st] for st in sites] == gold["sites"][rule.name], rule.name
    db = ef.CostDatabase()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    r, assign = frontier._price_one(g, db, ef.CostFunction.energy(), 1, True)
    inner = gold["inner_energy_d1"]
    assert [assign[k] for k in sorted(assign)] == inner["assignment"]
    assert (r.cost, r.time_ms, r.energy, r.evals, r.sweeps) == (inner["cost"], inner["time_ms"], inner["energy"],
                                                                inner["evals"], inner["sweeps"])
    if "search" in gold:  # BASELINE configs[0]: the full SqueezeNet search at alpha = 1.0
        run = gold["search"]
        trace = []
        res = ef.outer_search(g, rules, ef.CostDatabase(), ef.CostFunction.energy(),
                              ef.SearchConfig(alpha=run["alpha"]), ef.SyntheticProfiler(0), trace=trace,
                              check_prune=True)
        assert [str(h) for h in trace] == run["trace"]
        assert str(ef.canonical_hash(res.graph)) == run["hash"]
        assert [res.assignment[k] for k in sorted(res.assignment)] == run["assignment"]
        assert (res.cost, res.time_ms, res.energy) == (run["cost"], run["time_ms"], run["energy"])
        assert {k: v for k, v in vars(res.stats).items() if k != "wall_time_ms"} == run["stats"]


def test_packed_uploads_sync_async_match_resident():
    """Compact host uploads (synchronous and pipelined on the upload stream) rebuild the
    parents exactly: keys, sorted order and ranks recomputed on the device give the same
    step as the resident frontier."""
    import numpy as np

    g0 = zoo.generate("resnet50", 0)
    db = ef.CostDatabase()
    fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), 24)
    s = fr.s
    try:
        base = fr.step().copy()
        recs = [s.read_record(sl) for sl in fr.slots]
        blob, offs = s.pack(recs)
        pinned = s.L.ef_host_alloc(blob.nbytes)
        import ctypes as C

        staging = np.ctypeslib.as_array((C.c_uint8 * blob.nbytes).from_address(pinned))
        staging[:] = blob.view(np.uint8)
        a = [s.alloc() for _ in fr.slots]
        b = [s.alloc() for _ in fr.slots]
        s.write_packed(a, staging.view(np.uint32), offs)
        got_sync = fr.step(a).copy()
        s.write_packed(b, staging.view(np.uint32), offs, asynchronous=True)
        s.upload_fence()
        got_async = fr.step(b).copy()
        for sl, sa, sb in zip(fr.slots, a, b):  # whole records identical (keys, sperm, skeys, srank)
            G = s.geo
            ra, rb, r0 = s.read_record(sa), s.read_record(sb), s.read_record(sl)
            n = int(r0[:4].view(np.int32)[0])
            for off, width in ((G.off_keys, 16), (G.off_sperm, 4), (G.off_skeys, 16), (G.off_srank, 4)):
                assert bytes(ra[off: off + width * n]) == bytes(r0[off: off + width * n])
                assert bytes(rb[off: off + width * n]) == bytes(r0[off: off + width * n])
        del staging
        s.L.ef_host_free(pinned)
        for sl in a + b:
            s.free(sl)
    finally:
        fr.close()
    for got in (got_sync, got_async):
        for key in ("hash", "flags", "cost", "time_ms", "energy", "evals", "sweeps"):
            assert np.array_equal(got[key], base[key]), key


def test_results_async_matches_sync():
    """ef_results_async: the step's results snapshotted on the device and copied on the copy
    stream while the next step runs equal the synchronous ef_results of the same step."""
    import numpy as np

    g0 = zoo.generate("resnet50", 0)
    fr = Frontier(g0, ef.CostDatabase(), ef.SyntheticProfiler(0), ef.CostFunction.energy(),
                  ef.SearchConfig(alpha=1.05), 16)
    s = fr.s
    try:
        want = fr.step().copy()
        n = s.expand(fr.slots, fr.rule_ids, fr.pp, False, results=False)
        got = s.results_async(n)
        other = fr.step(fr.slots[:4])  # the next step overwrites the device results meanwhile
        s.results_wait()
        assert n == len(want) and len(other) < n
        for key in want.dtype.names:
            assert np.array_equal(got[key], want[key]), key
    finally:
        fr.close()
