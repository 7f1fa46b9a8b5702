"""Incremental table commits (ef_tables_commit / ef_commit_bytes).

A commit sends only what changed since the previous one: new signatures (texts,
cost rows, per-id entries, their lookup-table slots), new names and weight sets.
Its cost must not grow with the tables already resident (the reference memoises
once per new signature, profiling.py:211-252).  Correctness of the tables after
many incremental commits is what every search test relies on; here the hashes
and prices of graphs uploaded across commits are checked against the host.
"""

import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo
from paper_2005_05837_b200.device import DeviceSession, price_params

pytestmark = pytest.mark.gpu


def _refs(g):
    return sum(len(v.inputs) for v in g.nodes.values())


def _session(g0, cap_nodes, cap_refs=None):
    s = DeviceSession(0)
    s.bind_costs(ef.CostDatabase(), ef.SyntheticProfiler(0))
    s.set_geometry(g0, cap_nodes, cap_refs or _refs(g0) + cap_nodes)
    return s


def test_empty_commit_sends_almost_nothing():
    g = zoo.generate("resnet50", 0)
    s = _session(g, len(g.nodes) + 8)
    try:
        s.upload(g)
        s.commit()
        assert s.last_commit_bytes() <= 16  # the text padding and the name-pool terminator
    finally:
        s.close()


def test_commit_cost_independent_of_table_size():
    """Interning SqueezeNet after ResNet-50 (large tables) sends no more than after a
    toy graph (small tables), and the hashes / prices stay those of a fresh session."""
    big, small, add = zoo.generate("resnet50", 0), zoo.toy_squeeze(0), zoo.generate("squeezenet", 0)
    cap = max(len(big.nodes), len(add.nodes)) + 8
    refs = max(_refs(big), _refs(add)) + cap
    sent = {}
    got = {}
    for name, first in (("big", big), ("small", small)):
        s = _session(add, cap, refs)
        try:
            s.upload(first)
            base = len(s.sig_list)
            slot = s.upload(add)  # interns SqueezeNet's signatures and weight sets, then commits
            sent[name] = (s.last_commit_bytes(), len(s.sig_list) - base, base)
            pp = price_params(ef.CostFunction.energy(), 1, True, 1 << 30)
            (r,) = s.price_slots([slot], pp)
            got[name] = (s.hash_slots([slot])[0], r.cost, r.time_ms, r.energy)
        finally:
            s.close()
    fresh = _session(add, cap, refs)
    try:
        slot = fresh.upload(add)
        pp = price_params(ef.CostFunction.energy(), 1, True, 1 << 30)
        (r,) = fresh.price_slots([slot], pp)
        want = (fresh.hash_slots([slot])[0], r.cost, r.time_ms, r.energy)
    finally:
        fresh.close()
    assert got["big"] == want and got["small"] == want
    assert want[0] == ef.canonical_hash(add)
    (b_big, n_big, base_big), (b_small, n_small, base_small) = sent["big"], sent["small"]
    assert base_big > 4 * base_small  # the tables really differ in size
    # per new signature the same bytes, plus at most one lookup-table rebuild of the small one
    assert b_big <= b_small * (n_big + 1) / (n_small + 1) + 16 * 1024, sent
