"""The two-level search with its hot path on the B200 (reference: pkg/src/enerflow/search.py).

`outer_search` keeps the reference's semantics exactly (search.py:211-272):
a best-first heap keyed by (cost, canonical hash), a visited set, the alpha
enqueue rule against the best cost *before* each candidate, stale entries
pruned at pop, and the same statistics.  What moved to the GPU is the
expansion of a popped graph — every rule at every site, materialisation,
canonical hashing, in-step and visited deduplication, and the inner search on
every survivor — one `ef_expand` call per expansion.  The host loop below only
replays the reference's per-candidate bookkeeping on the returned results
(flags, costs, hashes), in the reference's order, so the explored-hash
sequence, the optimised graph, the assignment and every statistic match the
reference bit for bit (tests/test_gpu_parity.py).

Graphs never come back to the host during the search: the frontier lives in
HBM as records; only the final best graph is decoded.
"""

from __future__ import annotations

import heapq
import itertools
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .costmodel import Assignment, CostDatabase, CostFunction, node_cost_table, normalization_refs
from .device import DeviceSession, price_params
from .errors import InfeasibleConstraint, MissingEntry, SpaceTooLarge
from .ir import Graph
from .profiler import ProfilerSpec, ensure_profiled, profile_signature, record_line
from .rewrite import SubstitutionRule, scratch_graph
from .shard import gather_batch, sharded_expand


@dataclass
class SearchConfig:
    alpha: float = 1.05
    d: int = 1
    max_queue: int = 100_000
    max_graph_nodes: int | None = None
    seed: int = 0
    # Extension (not in the reference): stop at the pop that would start expansion number
    # max_expansions + 1 (after that pop's stale-entry check).  None = the reference's search.
    # Every result is then the reference's state at that point; used to bound alpha > 1 searches
    # of large graphs, whose queues never drain (tests/golden/make_golden_search_oracle.py).
    max_expansions: int | None = None

    def __post_init__(self):
        if self.alpha < 1.0:
            raise ValueError(f"alpha must be >= 1, got {self.alpha}")
        if self.d < 1:
            raise ValueError(f"d must be >= 1, got {self.d}")
        if self.max_queue < 1:
            raise ValueError("max_queue must be >= 1")
        if self.max_graph_nodes is not None and self.max_graph_nodes < 1:
            raise ValueError("max_graph_nodes must be >= 1")
        if self.max_expansions is not None and self.max_expansions < 0:
            raise ValueError("max_expansions must be >= 0")


@dataclass
class SearchStats:
    graphs_explored: int = 0
    graphs_generated: int = 0
    graphs_deduped: int = 0
    expanded_at_best: int = 0
    assignments_evaluated: int = 0
    inner_sweeps: int = 0
    best_updates: int = 0
    queue_pruned: int = 0
    queue_cap_hits: int = 0
    node_cap_hits: int = 0
    new_cost_records: int = 0
    wall_time_ms: float = field(default=0.0, compare=False)


@dataclass
class OptimizationResult:
    graph: Graph
    assignment: Assignment
    cost: float
    time_ms: float
    energy: float
    power_w: float
    stats: SearchStats


def _node_cap(cfg: SearchConfig, g0: Graph) -> int:
    return cfg.max_graph_nodes if cfg.max_graph_nodes is not None else 4 * max(1, len(g0.compute_nodes()))


class _Visible:
    """Replays ensure_profiled in the reference's order on the caller's database.

    The device priced candidates against rows profiled eagerly (session shadow);
    the reference profiles a candidate's new signatures only when it evaluates
    that candidate.  This copies those rows into `db` at exactly that point and
    counts them, so `db` contents, `new_cost_records` and the append file match.
    """

    def __init__(self, session: DeviceSession, db: CostDatabase, profiler, append_path):
        self.s, self.db, self.profiler, self.path = session, db, profiler, append_path
        self.known: set[int] = set()  # signature ids whose rows `db` already holds (it only grows)

    def touch(self, sig_ids) -> int:
        made = 0
        fh = None
        try:
            for sid in sig_ids:
                if sid == 0xFFFFFFFF or sid in self.known:
                    continue
                sig = self.s.sig_list[sid]
                if self.db.has_signature(sig.text):
                    self.known.add(sid)
                    continue
                if fh is None and self.path:
                    fh = open(self.path, "a")
                src = self.s.shadow
                if not src.has_signature(sig.text):
                    profile_signature(sig, src, self.profiler)
                for alg, _, _ in src.rows_for(sig.text):
                    rec = src.lookup(sig.text, alg)
                    self.db.add(sig.text, alg, rec)
                    made += 1
                    if fh is not None:
                        fh.write(record_line(sig.text, alg, rec) + "\n")
                        fh.flush()
                self.known.add(sid)
        finally:
            if fh is not None:
                fh.close()
        return made


class _Run:
    """Device state of one search: geometry, records, visited set, slot ownership (refcounts)."""

    def __init__(self, session: DeviceSession, g0: Graph, node_cap: int, db, profiler):
        self.s = session
        n_inputs = len(g0.nodes) - len(g0.compute_nodes())
        n_refs = sum(len(v.inputs) for v in g0.nodes.values())
        # a record holds any graph the search can expand (at most the larger of the cap and the
        # origin) plus one rewrite's growth; the cap itself only flags candidates (CAPPED)
        cap_nodes = max(node_cap, len(g0.compute_nodes())) + n_inputs + 2
        cap_refs = n_refs + max(0, cap_nodes - len(g0.nodes)) + 4
        session.bind_costs(db, profiler)
        session.set_geometry(g0, cap_nodes, cap_refs)
        session.visited_reset(1 << 16)  # grows on the device as the search inserts (ef_visited_*)
        self.root = session.upload(g0)
        self.refs: dict[int, int] = {self.root: 1}

    def hold(self, slot):
        self.refs[slot] = self.refs.get(slot, 0) + 1

    def drop(self, slot):
        self.refs[slot] -= 1
        if self.refs[slot] == 0:
            del self.refs[slot]
            self.s.free(slot)

    def close(self):
        self.s.free_n(list(self.refs))
        self.refs.clear()


def _missing_text(session: DeviceSession, touched, db: CostDatabase) -> str:
    for sid in touched:
        if sid != 0xFFFFFFFF and not db.has_signature(session.sig_list[sid].text):
            return session.sig_list[sid].text
    return "?"


class _Batch:
    """Host copy of one batched expansion: per-candidate columns as Python lists and each parent's
    segment (candidates in (rule, site) order, the device's rewrite numbering)."""

    __slots__ = ("hs", "flags", "cost", "t", "e", "evals", "sweeps", "ncomp", "touched", "seg")

    def __init__(self, res: np.ndarray, n_parents: int):
        self.hs = res["hash"].tolist()
        self.flags = res["flags"].tolist()
        self.cost = res["cost"].tolist()
        self.t = res["time_ms"].tolist()
        self.e = res["energy"].tolist()
        self.evals = res["evals"].tolist()
        self.sweeps = res["sweeps"].tolist()
        self.ncomp = res["n_compute"].tolist()
        self.touched = res["touched_sig"].tolist()
        self.seg = np.searchsorted(res["parent"], np.arange(n_parents + 1)).tolist()


class _Virtual:
    """An enqueued graph not materialised yet: rewrite `local` (the device's numbering, rule then
    site order) of the parent record `slot`, which it keeps alive."""

    __slots__ = ("slot", "local")

    def __init__(self, slot: int, local: int):
        self.slot, self.local = slot, local


def outer_search(g0: Graph, rules: list[SubstitutionRule], db: CostDatabase, f: CostFunction,
                 cfg: SearchConfig, profiler: ProfilerSpec | None, use_inner: bool = True,
                 db_append_path: str | None = None, session: DeviceSession | None = None,
                 trace: list | None = None, batch: int | None = None,
                 check_prune: bool = False, exchange=None) -> OptimizationResult:
    """Best-first search over the rewrite space of g0 (search.py:211-272), expanded on the GPU.

    The reference's loop is kept exactly: heap of (cost, hash), the visited set, the alpha rule
    against the best cost before each candidate, stale entries pruned at pop, the same stats.
    What changes is how expansions are produced.  Expanding a graph (every rule at every site,
    hashing, pricing) does not depend on the search state, only on the graph; so when the search
    pops a graph whose expansion is not cached, one `ef_expand` expands it together with the next
    `batch - 1` graphs of the heap (speculatively: the ones the search is likely to pop next),
    and caches every expansion by parent hash.  The search then replays the reference's
    per-candidate bookkeeping on cached expansions in the reference's pop order: the visited
    check and insertion, the node cap, the evaluation counters and the alpha rule.

    Steps price per parent (EF_F_PFIRST): the first occurrence of each hash within each parent,
    i.e. exactly the graphs `neighbors(parent)` yields, with that parent's node ids, whatever
    order the parents are replayed in.  The device skips candidates already in its visited set
    (every hash the replay has visited, uploaded before each step: a subset of the visited set
    at replay time).  Enqueued graphs stay virtual (parent record + rewrite index) until a step
    expands them or the search returns them (ef_materialise), so records are made only for the
    graphs the search expands.

    While a batch is replayed in its own order from the state it was expanded in, the step's
    alpha-prune flags (EF_F_BEST / EF_F_ENQUEUE: a prefix-min over the step's first occurrences,
    seeded with the best at step time) are exactly the reference's decisions and are used;
    `check_prune=True` also recomputes them on the host and asserts equality (tests).

    `exchange` (shard.OwnerExchange, one process per GPU): every rank runs this same replay;
    each batch is expanded split over the ranks (shard.gather_batch: a contiguous slice per rank,
    the prune flags carried across ranks by an exclusive minimum, the results all-gathered), so
    every rank returns the single-GPU result.
    """
    started = time.perf_counter()
    stats = SearchStats()
    s = session or DeviceSession.default()
    cap = _node_cap(cfg, g0)
    alpha = cfg.alpha
    K = max(1, int(batch if batch is not None else os.environ.get("EF_SEARCH_BATCH", 64)))
    if profiler is not None:
        stats.new_cost_records += ensure_profiled(g0, db, profiler, db_append_path)
    run = _Run(s, g0, cap, db, profiler)
    try:
        pp = price_params(f, cfg.d, use_inner, cap, alpha=alpha, per_parent=True)
        (r0,) = s.price_slots([run.root], pp)  # ctypes CandResult
        if r0.flags & N.F_MISSING:
            node_cost_table(g0, db)  # raises the reference's MissingEntry
        stats.assignments_evaluated += r0.evals
        stats.inner_sweeps += r0.sweeps
        best_ref, best_cost, best_t, best_e = run.root, r0.cost, r0.time_ms, r0.energy
        run.hold(run.root)
        (h0,) = s.hash_slots([run.root])
        visited = {h0}
        new_vis = [h0]  # visited on the host, not yet on the device
        heap: list[tuple[float, int]] = [(r0.cost, h0)]
        pending: dict[int, object] = {h0: run.root}  # hash -> slot | _Virtual
        cache: dict[int, tuple[_Batch, int]] = {}
        visible = _Visible(s, db, profiler, db_append_path)
        rule_ids = [r.rule_id for r in rules]
        inorder: tuple[_Batch, int] | None = None  # the batch whose own prune flags hold, next index
        max_queue = cfg.max_queue

        def release(ref):
            run.drop(ref.slot if isinstance(ref, _Virtual) else ref)

        def materialise(refs: list) -> list[int]:
            """Slots for a list of refs (virtual ones materialised in one call, parents released)."""
            virt = [i for i, r in enumerate(refs) if isinstance(r, _Virtual)]
            out = list(refs)
            if virt:
                parents: dict[int, int] = {}
                cp, cl = [], []
                for i in virt:
                    cp.append(parents.setdefault(refs[i].slot, len(parents)))
                    cl.append(refs[i].local)
                slots = s.materialise(list(parents), rule_ids, cp, cl)
                for i, sl in zip(virt, slots):
                    run.refs[sl] = 1
                    run.drop(refs[i].slot)
                    out[i] = sl
            return out

        def expand_batch(first_h: int) -> None:
            chosen = [first_h]
            bound = alpha * best_cost
            popped = []
            while heap and len(chosen) < K and len(popped) < 4 * K:
                e = heapq.heappop(heap)
                popped.append(e)
                if e[0] > bound or e[1] in cache:
                    continue
                chosen.append(e[1])
            for e in popped:
                heapq.heappush(heap, e)
            slots = materialise([pending[h] for h in chosen])
            for h, sl in zip(chosen, slots):
                pending[h] = sl
            if new_vis:
                s.visited_insert(new_vis)
                new_vis.clear()
            pp.best = best_cost
            if rule_ids and exchange is not None and exchange.world > 1:
                res = gather_batch(s, slots, rule_ids, pp, exchange)
            elif rule_ids:
                res = s.expand(slots, rule_ids, pp, insert_visited=False)
            else:
                res = np.empty(0, dtype=N.CAND_DTYPE)
            B = _Batch(res, len(chosen))
            for j, h in enumerate(chosen):
                cache[h] = (B, j)

        while heap:
            cost, h = heapq.heappop(heap)
            if cost > alpha * best_cost:
                stats.queue_pruned += 1
                ref = pending.pop(h, None)
                if ref is not None:
                    release(ref)
                ent = cache.pop(h, None)
                if ent is not None and inorder is not None and ent[0] is inorder[0]:
                    inorder = None  # the step counted this parent's candidates; the replay will not
                continue
            if cfg.max_expansions is not None and stats.graphs_explored >= cfg.max_expansions:
                break
            stats.graphs_explored += 1
            if trace is not None:
                trace.append(h)
            if cost == best_cost:
                stats.expanded_at_best += 1
            ent = cache.pop(h, None)
            if ent is None:
                expand_batch(h)
                ent = cache.pop(h)
                inorder = (ent[0], 0)
            slot = pending.pop(h)  # materialised: it was expanded
            B, j = ent
            use_dev = inorder is not None and inorder[0] is B and inorder[1] == j
            inorder = (B, j + 1) if use_dev else None
            hs, flags, ncomp = B.hs, B.flags, B.ncomp
            a = B.seg[j]
            local: set[int] = set()
            for i in range(a, B.seg[j + 1]):
                hc = hs[i]
                if hc in local:  # rules.neighbors: first occurrence within the parent
                    continue
                local.add(hc)
                stats.graphs_generated += 1
                if hc in visited:
                    stats.graphs_deduped += 1
                    continue
                visited.add(hc)
                new_vis.append(hc)
                if ncomp[i] > cap:
                    stats.node_cap_hits += 1
                    continue
                fl = flags[i]
                if profiler is not None:
                    stats.new_cost_records += visible.touch(B.touched[i])
                elif fl & N.F_MISSING:
                    raise MissingEntry(_missing_text(s, B.touched[i], db))
                if not fl & N.F_PRICED:
                    raise N.NativeError(f"candidate {hc} was not priced by its step")
                stats.assignments_evaluated += B.evals[i]
                stats.inner_sweeps += B.sweeps[i]
                c = B.cost[i]
                prev = best_cost
                if use_dev:
                    new_best = bool(fl & N.F_BEST)
                    enq = bool(fl & N.F_ENQUEUE)
                    if check_prune and (new_best != (c < prev) or enq != (c < alpha * prev)):
                        raise AssertionError(f"device alpha-prune differs from the replay at {hc}")
                else:
                    new_best = c < prev
                    enq = c < alpha * prev
                if new_best:
                    best_cost, best_t, best_e = c, B.t[i], B.e[i]
                    stats.best_updates += 1
                    run.hold(slot)
                    release(best_ref)
                    best_ref = _Virtual(slot, i - a)
                if enq:
                    if len(heap) >= max_queue:
                        stats.queue_cap_hits += 1
                    else:
                        heapq.heappush(heap, (c, hc))
                        run.hold(slot)
                        pending[hc] = _Virtual(slot, i - a)
            run.drop(slot)
        (best_slot,) = materialise([best_ref])
        # the record's algorithm bytes: the inner search again on the kept graph (deterministic)
        (rb,) = s.price_slots([best_slot], pp)
        if (rb.cost, rb.time_ms, rb.energy) != (best_cost, best_t, best_e):
            raise N.NativeError("re-pricing the optimised graph changed its cost")
        graph, assign = s.decode(s.read_record(best_slot), g0)
    finally:
        run.close()
    stats.wall_time_ms = (time.perf_counter() - started) * 1000.0
    power = best_e / best_t if best_t > 0 else 0.0
    return OptimizationResult(graph, assign, best_cost, best_t, best_e, power, stats)


# ---------------------------------------------------------------------------
# single-graph entry points
# ---------------------------------------------------------------------------

def _price_one(g: Graph, db: CostDatabase, f: CostFunction, d: int, use_inner: bool, session=None):
    s = session or DeviceSession.default()
    s.bind_costs(db, None)
    with scratch_graph(g, s) as (s, slot):
        s.commit()
        (r,) = s.price_slots([slot], price_params(f, d, use_inner, 1 << 30))
        if r.flags & N.F_MISSING:
            node_cost_table(g, db)
        _, assign = s.decode(s.read_record(slot), g)
    return r, assign


def inner_search(g: Graph, db: CostDatabase, f: CostFunction, d: int = 1, session=None) -> Assignment:
    """d-locally optimal assignment of one graph (search.py:106-159), on the GPU."""
    return _price_one(g, db, f, d, True, session)[1]


def default_assignment(g: Graph, db: CostDatabase) -> Assignment:
    table = node_cost_table(g, db)
    return {nid: rows[0][0] for nid, (_, rows) in table.items()}


def canonical_hash(g: Graph, session=None) -> int:
    """Relabel-invariant 64-bit digest (graph.py:520-549), computed on the GPU."""
    with scratch_graph(g, session) as (s, slot):
        return s.hash_slots([slot])[0]


def brute_force_assignment(g: Graph, db: CostDatabase, f: CostFunction, max_points: int = 10**6) -> Assignment:
    """Exhaustive assignment oracle of the reference API (search.py:162-182)."""
    table = node_cost_table(g, db)
    nids = sorted(table)
    if not nids:
        return {}
    rows = [table[n][1] for n in nids]
    total = math.prod(len(r) for r in rows)
    if total > max_points:
        raise SpaceTooLarge(f"{total} assignments exceed the bound {max_points}")
    t = np.array([x[1] for x in rows[0]])
    e = np.array([x[2] for x in rows[0]])
    for r in rows[1:]:
        t = np.add.outer(t, np.array([x[1] for x in r]))
        e = np.add.outer(e, np.array([x[2] for x in r]))
    idx = np.unravel_index(int(np.argmin(f.from_totals(t, e))), t.shape)
    return {n: rows[i][int(k)][0] for i, (n, k) in enumerate(zip(nids, idx))}


def closure(g0: Graph, rules: list[SubstitutionRule], max_graphs: int, max_graph_nodes: int | None = None,
            session: DeviceSession | None = None, exchange=None) -> list[Graph]:
    """BFS closure of g0 under the rules, deduplicated by canonical hash (search.py:275-300).

    Each BFS level is ONE batched ef_expand over all graphs of the level: candidates come back
    in (parent, rule, site) order, FIRST marks the first occurrence inside the level and
    VISITED membership in the hashes seen before it, which is exactly the reference's
    sequential `seen` check; the device inserts the level's new hashes into the visited set.
    Raises SpaceTooLarge past `max_graphs`; graphs above the node cap are seen, not kept.

    `exchange` (shard.OwnerExchange): the levels are expanded split over the ranks with
    hash-owner deduplication (_closure_sharded); every rank returns the same list.
    """
    if exchange is not None and exchange.world > 1:
        return _closure_sharded(g0, rules, max_graphs, max_graph_nodes, session, exchange)
    s = session or DeviceSession.default()
    rule_ids = [r.rule_id for r in rules]
    cap = max_graph_nodes if max_graph_nodes is not None else 1 << 30
    geo_cap = max_graph_nodes if max_graph_nodes is not None else 4 * max(1, len(g0.compute_nodes()))
    db = CostDatabase()  # pricing is not needed: use_inner = 0 and no rows requested
    run = _Run(s, g0, max(geo_cap, len(g0.compute_nodes())), db, None)
    out_slots = [run.root]
    try:
        (h0,) = s.hash_slots([run.root])
        s.visited_insert([h0])
        pp = price_params(CostFunction.time(), 1, False, cap)
        level = [run.root]
        while level and rule_ids:
            res = s.expand(level, rule_ids, pp, insert_visited=True)
            fl = res["flags"].tolist()
            keep = [i for i, f in enumerate(fl) if (f & (N.F_FIRST | N.F_VISITED | N.F_CAPPED)) == N.F_FIRST]
            if len(out_slots) + len(keep) > max_graphs:
                raise SpaceTooLarge(f"rewrite closure exceeds {max_graphs} graphs")
            level = s.keep(keep) if keep else []
            out_slots += level
        return [s.decode(s.read_record(sl), g0)[0] for sl in out_slots]
    finally:
        for sl in out_slots:
            if sl != run.root:
                s.free(sl)
        run.close()


def _closure_sharded(g0: Graph, rules: list[SubstitutionRule], max_graphs: int, max_graph_nodes: int | None,
                     session: DeviceSession | None, ex) -> list[Graph]:
    """The BFS closure over ranks (search.py:275-300).  Every rank holds every graph's record;
    rank r expands the contiguous slice shard.batch_slice(len(level), r, world) of each level
    through shard.sharded_expand, whose hash-owner all-to-all gives global first occurrences
    (rank-major = the single-GPU (parent, rule, site) order) and membership in the owner's
    shard of the visited set (inserted there).  The kept (parent, rewrite) pairs are
    all-gathered in rank order and every rank materialises the next level from them."""
    from .shard import batch_slice, owner_of

    s = session or DeviceSession.default()
    rule_ids = [r.rule_id for r in rules]
    cap = max_graph_nodes if max_graph_nodes is not None else 1 << 30
    geo_cap = max_graph_nodes if max_graph_nodes is not None else 4 * max(1, len(g0.compute_nodes()))
    run = _Run(s, g0, max(geo_cap, len(g0.compute_nodes())), CostDatabase(), None)
    out_slots = [run.root]
    try:
        (h0,) = s.hash_slots([run.root])
        if owner_of(h0, ex.world) == ex.rank:
            s.visited_insert([h0])
        pp = price_params(CostFunction.time(), 1, False, cap)
        level = [run.root]
        while level and rule_ids:
            lo, hi = batch_slice(len(level), ex.rank, ex.world)
            res = sharded_expand(s, level[lo:hi], rule_ids, pp, ex, insert_visited=True)
            fl = res["flags"].tolist()
            par = res["parent"].tolist()
            seg = np.searchsorted(res["parent"], np.arange(hi - lo + 1)).tolist() if len(res) else [0] * (hi - lo + 1)
            keep = [(lo + par[i], i - seg[par[i]]) for i, f in enumerate(fl)
                    if (f & (N.F_FIRST | N.F_VISITED | N.F_CAPPED)) == N.F_FIRST]
            kept = [k for part in ex.all_gather_object(keep) for k in part]
            if len(out_slots) + len(kept) > max_graphs:
                raise SpaceTooLarge(f"rewrite closure exceeds {max_graphs} graphs")
            level = s.materialise(level, rule_ids, [p for p, _ in kept], [q for _, q in kept]) if kept else []
            out_slots += level
        return [s.decode(s.read_record(sl), g0)[0] for sl in out_slots]
    finally:
        for sl in out_slots:
            if sl != run.root:
                s.free(sl)
        run.close()


def brute_force_space(g0: Graph, rules: list[SubstitutionRule], db: CostDatabase, f: CostFunction,
                      max_graphs: int = 10**4, max_points: int = 10**6, profiler: ProfilerSpec | None = None,
                      max_graph_nodes: int | None = None, session=None) -> OptimizationResult:
    """Exhaustive oracle of the reference API (search.py:303-329): the closure (batched BFS on
    the GPU) and the exhaustive assignment of every member; first-found minimum wins."""
    started = time.perf_counter()
    stats = SearchStats()
    best = None
    for g in closure(g0, rules, max_graphs, max_graph_nodes, session):
        stats.graphs_explored += 1
        if profiler is not None:
            stats.new_cost_records += ensure_profiled(g, db, profiler)
        assign = brute_force_assignment(g, db, f, max_points)
        table = node_cost_table(g, db)
        per = {nid: {a: (tt, ee) for a, tt, ee in rows} for nid, (_, rows) in table.items()}
        t = sum(per[nid][assign[nid]][0] for nid in per)
        e = sum(per[nid][assign[nid]][1] for nid in per)
        cost = f.from_totals(t, e)
        stats.assignments_evaluated += math.prod(len(rows) for _, rows in table.values()) if table else 1
        if best is None or cost < best[2]:
            best = (g, assign, cost, t, e)
    stats.wall_time_ms = (time.perf_counter() - started) * 1000.0
    g_best, a_best, c_best, t_best, e_best = best
    power = e_best / t_best if t_best > 0 else 0.0
    return OptimizationResult(g_best, a_best, c_best, t_best, e_best, power, stats)


def constrained_optimize(g0: Graph, rules, db: CostDatabase, cfg: SearchConfig, time_bound_ms: float,
                         profiler: ProfilerSpec | None, iterations: int = 20,
                         db_append_path: str | None = None, session=None) -> OptimizationResult:
    """Least energy under a time bound by binary search on w (search.py:336-381)."""
    if profiler is not None:
        ensure_profiled(g0, db, profiler, db_append_path)
    if not g0.compute_nodes():
        return outer_search(g0, rules, db, CostFunction("time"), cfg, profiler,
                            db_append_path=db_append_path, session=session)
    t_ref, e_ref, p_ref = normalization_refs(g0, db)

    def run(w: float) -> OptimizationResult:
        f = CostFunction.linear(w).with_refs(t_ref, e_ref, p_ref)
        return outer_search(g0, rules, db, f, cfg, profiler, db_append_path=db_append_path, session=session)

    energy_opt = run(1.0)
    if energy_opt.time_ms <= time_bound_ms:
        return energy_opt
    time_opt = run(0.0)
    if time_opt.time_ms > time_bound_ms:
        raise InfeasibleConstraint(time_opt.time_ms)
    best = time_opt
    lo, hi = 0.0, 1.0
    for _ in range(iterations):
        mid = (lo + hi) / 2.0
        res = run(mid)
        if res.time_ms <= time_bound_ms:
            lo = mid
            if res.energy < best.energy:
                best = res
        else:
            hi = mid
    return best


# ---------------------------------------------------------------------------
# frontier batches (bench + scaling): the real frontier of a search, resident in HBM
# ---------------------------------------------------------------------------

class Frontier:
    """A batch of frontier graphs of g0's search, kept as device records.

    Built by expanding the origin and then the cheapest level-1 graphs in the
    reference's best-first order, keeping every candidate the search would
    enqueue (cost < alpha * best).  `step()` expands the whole batch at once:
    one ef_expand over all parents, i.e. every rule at every site of every
    frontier graph, dedup, and the inner search on every survivor.
    """

    def __init__(self, g0: Graph, db: CostDatabase, profiler, f: CostFunction, cfg: SearchConfig,
                 n_parents: int, rules=None, session: DeviceSession | None = None):
        from .rewrite import default_rules

        self.s = session or DeviceSession.default()
        self.g0 = g0
        self.rules = rules if rules is not None else default_rules()
        self.rule_ids = [r.rule_id for r in self.rules]
        cap = _node_cap(cfg, g0)
        if profiler is not None:
            ensure_profiled(g0, db, profiler)
        self.run = _Run(self.s, g0, cap, db, profiler)
        self.pp = price_params(f, cfg.d, True, cap, alpha=cfg.alpha)
        (r0,) = self.s.price_slots([self.run.root], self.pp)
        (h0,) = self.s.hash_slots([self.run.root])
        self.s.visited_insert([h0])
        best = r0.cost
        heap = [(r0.cost, h0, self.run.root)]
        slots: list[int] = []
        seen = {h0}
        # every graph as its rewrite path from g0: the index of each rewrite in its parent's
        # (rule, site) enumeration (rules.neighbors order), so a CPU run can rebuild the batch
        paths: dict[int, tuple[int, ...]] = {self.run.root: ()}
        while heap and len(slots) < n_parents:
            cost, h, slot = heapq.heappop(heap)
            slots.append(slot)
            res = self.s.expand([slot], self.rule_ids, self.pp, insert_visited=True)
            keep = []
            fl, hs, cs = res["flags"].tolist(), res["hash"].tolist(), res["cost"].tolist()
            for i in range(len(res)):
                if (fl[i] & (N.F_FIRST | N.F_VISITED | N.F_CAPPED)) != N.F_FIRST or hs[i] in seen:
                    continue
                if cs[i] < cfg.alpha * best:
                    keep.append(i)
                    seen.add(hs[i])
                best = min(best, cs[i])
            # only the cheapest `room` of them can be popped into the batch before it is full:
            # materialise those (keeps large graphs' frontiers within memory)
            room = n_parents - len(slots)
            if len(keep) > room:
                keep = sorted(sorted(keep, key=lambda i: (cs[i], hs[i]))[:room])
            for i, sl in zip(keep, self.s.keep(keep)):
                heapq.heappush(heap, (cs[i], hs[i], sl))
                paths[sl] = paths[slot] + (i,)
        # fill the batch with the remaining enqueued graphs in heap order
        while heap and len(slots) < n_parents:
            slots.append(heapq.heappop(heap)[2])
        self.leftover = [sl for _, _, sl in heap]
        self.slots = slots
        self.paths = [paths[sl] for sl in slots]
        # The timed steps start from an empty visited set: every parent of the batch was already
        # expanded (or enqueued) while the batch was built, so keeping that set would mark most
        # candidates visited; each step is the first expansion of these graphs.  The step's
        # alpha-prune runs against the best cost found while building the batch.
        self.s.visited_reset(1 << 22)
        self.pp.best = best
        self.best = best

    def step(self, slots=None, insert_visited: bool = False):
        """One batched expansion; the results view is valid until the session's next step."""
        return self.s.expand(slots if slots is not None else self.slots, self.rule_ids, self.pp, insert_visited)

    def decode(self, slot: int) -> Graph:
        return self.s.decode(self.s.read_record(slot), self.g0)[0]

    def close(self):
        for sl in self.slots + self.leftover:
            if sl != self.run.root:
                self.s.free(sl)
        self.slots, self.leftover = [], []
        self.run.close()
