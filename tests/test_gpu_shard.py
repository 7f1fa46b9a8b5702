"""The sharded step's CUDA kernels (ef_expand_hashes / ef_route_owners /
ef_owner_mark / ef_expand_finish) on one GPU, two ranks emulated by two library
contexts driven from two threads through the product's `sharded_expand`; the
all-to-all is done in-process.  Every candidate's hash, flags and price must
equal a single-context `ef_expand` over the concatenated frontier.
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

    def to_owners(self, send, counts):
        data = self._gather((send, counts))
        parts, rc = [], []
        for snd, cnt in data:
            off = sum(cnt[: self.rank])
            parts.append(snd[2 * off: 2 * (off + cnt[self.rank])])
            rc.append(cnt[self.rank])
        torch.cuda.synchronize()
        return torch.cat(parts).contiguous(), rc

    def back(self, verdict, recv_counts, counts):
        data = self._gather((verdict, recv_counts))
        parts = []
        for v, rco in data:
            off = sum(rco[: self.rank])
            parts.append(v[off: off + rco[self.rank]])
        torch.cuda.synchronize()
        out = torch.cat(parts).contiguous() if sum(counts) else torch.zeros(1, dtype=torch.int32, device="cuda")
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


@pytest.mark.parametrize("model,n_parents", [("squeezenet", 24), ("resnet50", 16)])
def test_sharded_step_equals_single(model, n_parents):
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
    shared = {"barrier": threading.Barrier(world), "slot": [None] * world}
    out, errs = [None] * world, []

    def run(rank):
        try:
            mine = [h for h in visited if owner_of(h, world) == rank]
            s, slots = _session(g0, db, prof, cap, parts[rank], mine)
            out[rank] = sharded_expand(s, slots, rule_ids, pp, ThreadExchange(rank, world, shared)).copy()
            s.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)
            shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    sharded = np.concatenate(out)
    assert len(sharded) == len(single)
    for key in ("hash", "flags", "rule", "site_a", "site_b", "n_compute", "n_nodes"):
        assert np.array_equal(sharded[key], single[key]), key
    priced = (single["flags"] & N.F_PRICED) != 0
    assert priced.any() and (~priced).any()
    for key in ("cost", "time_ms", "energy", "evals", "sweeps"):
        assert np.array_equal(sharded[key][priced], single[key][priced]), key
