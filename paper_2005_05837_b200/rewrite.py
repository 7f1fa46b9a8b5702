"""Substitution rules at the operator API (reference: pkg/src/enerflow/rules.py).

The six rules of reference rules.py:338-353 are implemented as device code
(csrc/ef_kernels.cuh: `k_match` finds every site, `k_materialise` builds the
rewritten graph).  This module keeps the reference's Python surface —
`default_rules`, `select_rules`, `match_rule`, `apply`, `neighbors` — and
routes each call through one GPU frontier step on a scratch record.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass

from . import _native as N
from .costmodel import CostFunction
from .device import RULE_IDS, DeviceSession, price_params
from .errors import InvalidSite
from .ir import Graph

# pattern-node names per rule in the order the device reports (a, b)
_SITE_NAMES = {"fuse-conv-relu": ("conv", "relu"), "split-conv-activation": ("conv",),
               "merge-parallel-convs": ("left", "right"), "split-merged-conv": ("conv", "split"),
               "fold-identity": ("identity",), "fuse-conv-batchnorm": ("conv", "bn")}


@dataclass(frozen=True)
class MatchSite:
    """Injective binding pattern-node name -> graph node id, sorted by name."""

    binding: tuple[tuple[str, int], ...]

    @classmethod
    def of(cls, **names: int) -> "MatchSite":
        return cls(tuple(sorted(names.items())))

    def __getitem__(self, name: str) -> int:
        for k, v in self.binding:
            if k == name:
                return v
        raise KeyError(name)


@dataclass(frozen=True)
class SubstitutionRule:
    name: str
    shrinking: bool

    @property
    def rule_id(self) -> int:
        return RULE_IDS[self.name]

    def __repr__(self):
        return f"SubstitutionRule({self.name!r})"


def default_rules() -> list[SubstitutionRule]:
    return [SubstitutionRule("fuse-conv-relu", True), SubstitutionRule("split-conv-activation", False),
            SubstitutionRule("merge-parallel-convs", True), SubstitutionRule("split-merged-conv", False),
            SubstitutionRule("fold-identity", True), SubstitutionRule("fuse-conv-batchnorm", True)]


def select_rules(spec: str) -> list[SubstitutionRule]:
    """`all`, `none`, `fusion-only` or a comma-separated list (rules.py:356-374)."""
    catalog = default_rules()
    if spec == "all":
        return catalog
    if spec == "none":
        return []
    if spec == "fusion-only":
        return [r for r in catalog if r.shrinking]
    by_name = {r.name: r for r in catalog}
    out = []
    for name in (s.strip() for s in spec.split(",")):
        if name not in by_name:
            raise ValueError(f"unknown rule {name!r} (known: {', '.join(sorted(by_name))})")
        out.append(by_name[name])
    return out


@contextmanager
def scratch_graph(g: Graph, session: DeviceSession | None = None, extra_nodes: int = 4):
    """Upload `g` into a fresh geometry; yields (session, slot); frees everything after."""
    s = session or DeviceSession.default()
    with s.lock:  # the geometry and the scratch record belong to this caller until it is done
        n = len(g.nodes)
        n_refs = sum(len(v.inputs) for v in g.nodes.values())
        s.set_geometry(g, n + extra_nodes, n_refs + extra_nodes)
        s.visited_reset(1 << 12)
        slot = s.upload(g)
        try:
            yield s, slot
        finally:
            s.free(slot)


def _site_of(rule_name: str, g_ids: list[int], r) -> MatchSite:
    names = _SITE_NAMES[rule_name]
    vals = (g_ids[int(r["site_a"])], g_ids[int(r["site_b"])])[: len(names)]
    return MatchSite(tuple(sorted(zip(names, vals))))


def _expand_one(g: Graph, rules: list[SubstitutionRule], session=None):
    with scratch_graph(g, session) as (s, slot):
        pp = price_params(CostFunction.time(), 1, False, 1 << 30)
        res = s.expand([slot], [r.rule_id for r in rules], pp, insert_visited=False)
        yield s, res


def match_rule(rule: SubstitutionRule, g: Graph, session=None) -> list[MatchSite]:
    ids = sorted(g.nodes)
    for _, res in _expand_one(g, [rule], session):
        return [_site_of(rule.name, ids, r) for r in res]
    return []


def apply(rule: SubstitutionRule, g: Graph, site: MatchSite, session=None) -> Graph:
    ids = sorted(g.nodes)
    for s, res in _expand_one(g, [rule], session):
        for i, r in enumerate(res):
            if _site_of(rule.name, ids, r) == site:
                (slot,) = s.keep([i])
                try:
                    return s.decode(s.read_record(slot), g)[0]
                finally:
                    s.free(slot)
    raise InvalidSite(f"{rule.name}: site {site.binding} does not match this graph")


def neighbors(g: Graph, rules: list[SubstitutionRule], session=None) -> list[Graph]:
    """Every one-step rewrite, first graph per canonical hash (rules.py:73-89)."""
    out = []
    for s, res in _expand_one(g, rules, session):
        keep = [i for i, fl in enumerate(res["flags"].tolist()) if fl & N.F_FIRST]
        slots = s.keep(keep)
        try:
            out = [s.decode(s.read_record(sl), g)[0] for sl in slots]
        finally:
            for sl in slots:
                s.free(sl)
    return out
