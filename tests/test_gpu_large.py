"""Synthetic random DAGs of 1k-20k nodes (BASELINE configs[4]) through the batched
step: scratch chunking, the CTA key sort (k_sortbig) for rows > 1024 keys, and
thousands of outputs in the graph digest.  A sample of every step's candidates is
checked against the oracle (canonical hash, and the inner search of priced ones)."""

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


@pytest.mark.parametrize("n_ops,n_parents,sample,objective", [
    (1000, 4, 24, "energy"), (1000, 2, 12, "linear0.5"),  # rows <= 2048: interleaved sweep rows
    (5000, 2, 8, "energy"), (5000, 1, 4, "linear0.5"),    # rows > 2048: row-major sweep rows
    (20000, 1, 3, "energy")])
def test_random_dag_step_matches_oracle(n_ops, n_parents, sample, objective):
    """k_price_v<ENERGY / LINEAR, false> with the exact skip of nodes with no cheaper row, on
    both sweep-row layouts; the energy-delay objective over the origin's normalization refs."""
    from oracle import enerflow_oracle as orc

    g0 = zoo.random_dag(n_ops, 0)
    db = ef.CostDatabase()
    ef.ensure_profiled(g0, db, ef.SyntheticProfiler(0))
    if objective == "energy":
        f = ef.CostFunction.energy()
    else:
        f = ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g0, db))
    fr = Frontier(g0, db, ef.SyntheticProfiler(0), f, ef.SearchConfig(alpha=1.05), n_parents)
    try:
        res = fr.step()
        parents = [fr.decode(sl) for sl in fr.slots]
    finally:
        fr.close()
    odb = orc.CostDB()
    for (sig, alg), rec in db.records().items():
        odb.add(sig, alg, rec.time_ms, rec.power_w)
    og0 = to_oracle(g0)
    of = orc.CostFn("energy") if objective == "energy" else orc.CostFn("linear", w=0.5,
                                                                       refs=orc.normalization_refs(og0, odb))
    rule_names = {i: r.name for i, r in enumerate(ef.default_rules())}
    checked = 0
    for pi, pg in enumerate(parents):
        og = to_oracle(pg)
        want = [(rule, site) for rule in RULES for site in orc.match(rule, og)]
        mine = res[res["parent"] == pi]
        assert len(mine) == len(want)
        stride = max(1, len(want) // sample)
        for k in range(0, len(want), stride):
            rule, site = want[k]
            r = mine[k]
            assert rule_names[int(r["rule"])] == rule
            child = orc.apply(rule, og, site)
            assert int(r["hash"]) == orc.canonical_hash(child), (n_ops, pi, rule, site)
            if r["flags"] & N.F_PRICED:
                orc.ensure_profiled(child, odb, 0)
                _, cost, t, e, evals, sweeps = orc.sweep(child, odb, of, 1)
                assert (float(r["cost"]), float(r["time_ms"]), float(r["energy"])) == (cost, t, e)
                assert (int(r["evals"]), int(r["sweeps"])) == (evals, sweeps)
            checked += 1
    assert checked >= sample


def _step_with(g0, monkeypatch, env: dict, parents: int = 6):
    """One frontier step in a fresh device session: the tuning knobs (EF_*) are read when a
    library context is created."""
    from paper_2005_05837_b200.device import DeviceSession

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    s = DeviceSession()
    try:
        fr = Frontier(g0, ef.CostDatabase(), ef.SyntheticProfiler(0), ef.CostFunction.energy(),
                      ef.SearchConfig(alpha=1.05), parents, session=s)
        try:
            return fr.step().copy()
        finally:
            fr.close()
    finally:
        s.close()


@pytest.mark.parametrize("model", ["dag:1000", "nasnet_a"])
def test_wide_level_keys_match_thread_keys(model, monkeypatch):
    """k_keys_wide (a warp per candidate, jobs by level) against k_keys (a thread per
    candidate, jobs in order): every candidate's hash, flags and price identical.  EF_WIDE_MIN
    = 1 sends every candidate of a large-graph step to the level kernel, 0 sends none."""
    import numpy as np

    g0 = zoo.random_dag(1000, 0) if model.startswith("dag") else zoo.generate(model, 0)
    out = {}
    for wide in ("0", "1"):
        out[wide] = _step_with(g0, monkeypatch, {"EF_WIDE_MIN": wide})
    assert len(out["0"]) == len(out["1"]) > 0
    for key in ("hash", "flags", "cost", "time_ms", "energy", "evals", "sweeps"):
        assert np.array_equal(out["0"][key], out["1"][key]), key


@pytest.mark.parametrize("model", ["dag:1000", "nasnet_a"])
def test_merge_path_stream_matches_in_thread_merge(model, monkeypatch):
    """Rows > 256: the merge-path key stream (k_merge_big) + streaming digest against the
    in-thread merge of k_digest (EF_BIG_MERGE=0): every candidate's hash, flags and price."""
    import numpy as np

    g0 = zoo.random_dag(1000, 0) if model.startswith("dag") else zoo.generate(model, 0)
    out = {}
    for big in ("0", "1"):
        out[big] = _step_with(g0, monkeypatch, {"EF_BIG_MERGE": big})
    assert len(out["0"]) == len(out["1"]) > 0
    for key in ("hash", "flags", "cost", "time_ms", "energy", "evals", "sweeps"):
        assert np.array_equal(out["0"][key], out["1"][key]), key


@pytest.mark.parametrize("model", ["dag:1000", "dag:5000", "nasnet_a"])
@pytest.mark.parametrize("knob,values", [
    ("EF_DIRTY_BIG", ("0", "1")),            # k_dirty (thread walk) vs k_dirty_big (warp window walk)
    ("EF_WIDE_LPC", ("32", "16", "8", "4")),  # k_keys_wide lane groups
    ("EF_QUAD_MAX", ("0", "100000000")),     # k_keys (thread) vs k_keys_quad for the rest
    ("EF_DIGEST_PF", ("0", "1")),            # k_digest_pm with / without the next block's words ahead
    ("EF_FUSE_MERGE", ("0", "1")),           # k_merge_big + k_digest_pm vs the fused k_digest_mg
])
def test_large_graph_kernel_variants_agree(model, knob, values, monkeypatch):
    """Every kernel variant of the large-graph step produces the same candidates: hash, flags,
    and price of every candidate identical (EF_WIDE_MIN=1 sends all candidates to the level
    kernel where the knob concerns it)."""
    import numpy as np

    g0 = zoo.random_dag(int(model[4:]), 0) if model.startswith("dag") else zoo.generate(model, 0)
    extra = {"EF_WIDE_MIN": "1"} if knob == "EF_WIDE_LPC" else {}
    outs = [_step_with(g0, monkeypatch, {**extra, knob: v}, 2 if model == "dag:5000" else 6) for v in values]
    assert len(outs[0]) > 0
    for o in outs[1:]:
        assert len(o) == len(outs[0])
        for key in ("hash", "flags", "cost", "time_ms", "energy", "evals", "sweeps"):
            assert np.array_equal(outs[0][key], o[key]), (knob, key)
