"""The sharded paths' CUDA kernels on one GPU, two ranks emulated by two library
contexts driven from two threads through the product's code: the sharded step
(`sharded_expand`: ef_expand_hashes / ef_route_owners_padded /
ef_owner_mark_padded / ef_expand_finish_padded), the sharded BFS closure and the
sharded outer search (`exchange=`: shard.gather_batch, ef_reprune).  The
collectives are done in-process by ThreadExchange.  Every candidate's hash,
flags and price must equal a single-context `ef_expand` over the concatenated
frontier; the closure and the search must return exactly the single-GPU result
on every rank.
"""

import threading

import numpy as np
import pytest
import torch

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import _native as N
from paper_2005_05837_b200 import zoo
from paper_2005_05837_b200.device import DeviceSession, price_params
from paper_2005_05837_b200.frontier import Frontier, _node_cap
from paper_2005_05837_b200.shard import owner_of, sharded_expand

pytestmark = pytest.mark.gpu


class ThreadExchange:
    """OwnerExchange semantics between threads of one process."""

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared
        self.device = torch.device("cuda", 0)

    def _gather(self, obj):
        self.sh["slot"][self.rank] = obj
        self.sh["barrier"].wait()
        out = list(self.sh["slot"])
        self.sh["barrier"].wait()
        return out

    def order_base(self):
        return self.rank << 40

    def buffer(self, name, numel, dtype):
        return torch.empty(max(numel, 1), dtype=dtype, device=self.device)[:numel]

    def max_int(self, x):
        return max(self._gather(int(x)))

    def min(self, x):
        return min(self._gather(float(x)))

    def sum(self, x):
        return sum(self._gather(float(x)))

    def all_gather_object(self, obj):
        return self._gather(obj)

    def exclusive_min(self, x, init):
        out = init
        for v in self._gather(float(x))[: self.rank]:
            out = v if v < out else out
        return out

    def to_owners(self, send, counts, cap, session=None):
        torch.cuda.synchronize()  # the library wrote them on its own stream
        data = self._gather((send, counts))
        recv = torch.cat([snd[2 * self.rank * cap: 2 * (self.rank + 1) * cap] for snd, _ in data]).contiguous()
        rc = torch.stack([cnt[self.rank] for _, cnt in data]).to(torch.int32).contiguous()
        torch.cuda.synchronize()
        self._gather(None)  # every rank has copied before the buffers are reused
        return recv, rc

    def back(self, verdict, cap, session=None):
        torch.cuda.synchronize()
        data = self._gather(verdict)
        out = torch.cat([v[self.rank * cap: (self.rank + 1) * cap] for v in data]).contiguous()
        torch.cuda.synchronize()
        self._gather(None)
        return out


def _threads(world, fn):
    """Run fn(rank, exchange) on `world` threads; -> the per-rank results."""
    shared = {"barrier": threading.Barrier(world), "slot": [None] * world}
    out, errs = [None] * world, []

    def run(rank):
        try:
            out[rank] = fn(rank, ThreadExchange(rank, world, shared))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


def _session(g0, db, prof, cap, graphs, visited):
    s = DeviceSession(0)
    s.bind_costs(db, prof)
    n_inputs = len(g0.nodes) - len(g0.compute_nodes())
    n_refs = sum(len(v.inputs) for v in g0.nodes.values())
    cap_nodes = cap + n_inputs + 2
    s.set_geometry(g0, cap_nodes, n_refs + max(0, cap_nodes - len(g0.nodes)) + 4)
    s.visited_reset(1 << 16)
    if visited:
        s.visited_insert(visited)
    return s, [s.upload(g) for g in graphs]


@pytest.mark.parametrize("model,n_parents,spec", [("squeezenet", 24, False), ("resnet50", 16, False),
                                                  ("resnet50", 16, True), ("nasnet_a", 4, True)])
def test_sharded_step_equals_single(model, n_parents, spec, monkeypatch):
    """spec: the ranks' contexts price every candidate speculatively beside the hashing
    (EF_SPEC_PRICE=2: ef_expand_hashes_spec) and keep the survivors' prices after the owners'
    verdicts; the reference is a plain single-context ef_expand."""
    g0 = zoo.generate(model, 0)
    db = ef.CostDatabase()
    prof = ef.SyntheticProfiler(0)
    f = ef.CostFunction.energy()
    cfg = ef.SearchConfig(alpha=1.05)
    fr = Frontier(g0, db, prof, f, cfg, n_parents)
    try:
        graphs = [fr.decode(sl) for sl in fr.slots]
        probe = fr.step()
    finally:
        fr.close()
    # a visited set that hits some candidates: every third distinct hash of the probe step
    visited = sorted({int(h) for h in probe["hash"].tolist()})[::3]
    cap = _node_cap(cfg, g0)
    pp = price_params(f, 1, True, cap)
    rule_ids = [r.rule_id for r in ef.default_rules()]

    s_all, slots_all = _session(g0, db, prof, cap, graphs, visited)
    single = s_all.expand(slots_all, rule_ids, pp, insert_visited=False).copy()
    s_all.close()

    world, split = 2, len(graphs) // 3
    parts = [graphs[:split], graphs[split:]]
    if spec:
        monkeypatch.setenv("EF_SPEC_PRICE", "2")  # read when the ranks' contexts are created

    def run(rank, ex):
        mine = [h for h in visited if owner_of(h, world) == rank]
        s, slots = _session(g0, db, prof, cap, parts[rank], mine)
        try:
            return sharded_expand(s, slots, rule_ids, pp, ex).copy()
        finally:
            s.close()

    out = _threads(world, run)
    sharded = np.concatenate(out)
    assert len(sharded) == len(single)
    for key in ("hash", "flags", "rule", "site_a", "site_b", "n_compute", "n_nodes"):
        assert np.array_equal(sharded[key], single[key]), key
    priced = (single["flags"] & N.F_PRICED) != 0
    assert priced.any() and (~priced).any()
    for key in ("cost", "time_ms", "energy", "evals", "sweeps"):
        assert np.array_equal(sharded[key][priced], single[key][priced]), key


@pytest.mark.parametrize("model,max_graphs,max_nodes", [("squeezenet", 400, None), ("resnet50", 300, 54)])
def test_sharded_closure_equals_single(model, max_graphs, max_nodes):
    """BFS levels split over two ranks, hash-owner dedup: the same graphs in the same order."""
    g0 = zoo.generate(model, 0)
    rules = ef.default_rules()

    def names(gs):
        return [ef.canonical_hash(g) for g in gs]

    try:
        single = names(ef.closure(g0, rules, max_graphs, max_nodes))
        raised = None
    except ef.SpaceTooLarge as e:
        single, raised = None, type(e)

    def run(rank, ex):
        s = DeviceSession(0)
        try:
            try:
                return ef.closure(g0, rules, max_graphs, max_nodes, session=s, exchange=ex)
            except ef.SpaceTooLarge as e:
                return type(e)
        finally:
            s.close()

    # hashed after the threads join: canonical_hash uses the process's default session, which
    # two threads must not drive at once
    got = [r if isinstance(r, type) else names(r) for r in _threads(2, run)]
    want = raised if raised is not None else single
    assert got[0] == want and got[1] == want


@pytest.mark.parametrize("model,alpha,max_exp,batch", [("squeezenet", 1.0, None, 8), ("resnet50", 1.05, 300, 16)])
def test_sharded_search_equals_single(model, alpha, max_exp, batch):
    """The outer search with each batch split over two ranks (prune flags carried across ranks
    by the exclusive minimum, results all-gathered) returns the single-GPU search on every rank:
    explored-hash trace, optimised graph, assignment, cost, every statistic."""
    g0 = zoo.generate(model, 0)
    cfg = ef.SearchConfig(alpha=alpha, max_expansions=max_exp)

    def search(session=None, exchange=None):
        trace = []
        res = ef.outer_search(g0, ef.default_rules(), ef.CostDatabase(), ef.CostFunction.energy(), cfg,
                              ef.SyntheticProfiler(0), trace=trace, batch=batch, check_prune=True,
                              session=session, exchange=exchange)
        st = {k: v for k, v in vars(res.stats).items() if k != "wall_time_ms"}
        return trace, res.graph, res.assignment, (res.cost, res.time_ms, res.energy), st

    def hashed(r):  # after the threads join (canonical_hash drives the default session)
        return (r[0], ef.canonical_hash(r[1]), *r[2:])

    want = hashed(search())

    def run(rank, ex):
        s = DeviceSession(0)
        try:
            return search(s, ex)
        finally:
            s.close()

    got = [hashed(r) for r in _threads(2, run)]
    assert got[0] == want
    assert got[1] == want


@pytest.mark.parametrize("mode", ["1", "2", "3", "4"])
def test_speculative_pricing_equals_plain(mode, monkeypatch):
    """ef_expand with every candidate priced speculatively beside the hashing (from the first
    digest, the plans, the node keys, the key sort) and the survivors' prices committed after
    the dedup equals the plain step -- flags, costs, evaluation counts -- on NasNet-A parents
    (rows > 256), against a visited set that rejects some candidates."""
    g0 = zoo.generate("nasnet_a", 0)
    db = ef.CostDatabase()
    prof = ef.SyntheticProfiler(0)
    f = ef.CostFunction.energy()
    cfg = ef.SearchConfig(alpha=1.05)
    fr = Frontier(g0, db, prof, f, cfg, 6)
    try:
        graphs = [fr.decode(sl) for sl in fr.slots]
        probe = fr.step()
    finally:
        fr.close()
    visited = sorted({int(h) for h in probe["hash"].tolist()})[::4]
    cap = _node_cap(cfg, g0)
    pp = price_params(f, 1, True, cap)
    rule_ids = [r.rule_id for r in ef.default_rules()]

    def step():
        s, slots = _session(g0, db, prof, cap, graphs, visited)
        try:
            return s.expand(slots, rule_ids, pp, insert_visited=False).copy()
        finally:
            s.close()

    plain = step()
    monkeypatch.setenv("EF_SPEC_PRICE", mode)
    spec = step()
    assert len(spec) == len(plain)
    for key in ("hash", "flags", "cost", "time_ms", "energy", "evals", "sweeps"):
        assert np.array_equal(spec[key], plain[key]), key
    assert ((plain["flags"] & N.F_PRICED) != 0).any() and (plain["flags"] & N.F_VISITED).any()
