"""ORACLE — TEST INFRASTRUCTURE ONLY.  Never imported by the product package.

The oracle's outer search (enerflow_oracle.outer_search, restating the
reference's search.py:211-272) run on several host cores, for golden vectors of
searches too long for one core (BASELINE configs[1-3]).

Expanding a graph — `neighbors` (rules.py:73-89), each candidate's canonical
hash, node count, `ensure_profiled` and inner search — is a pure function of
the graph.  So a pool of worker processes expands graphs speculatively (the
next few heap entries) and the parent process replays the reference's loop in
its exact order on the cached expansions: pop, stale-entry prune, visited check
and insertion, node cap, the database's new records, evaluation counters, the
alpha rule with the best cost before each candidate, the queue cap.  The result
(trace, optimised graph, assignment, costs, every statistic) is the one
`enerflow_oracle.outer_search` returns; tests/test_oracle_parallel.py checks
that on small searches.

Graphs never cross processes (ResNet-50 carries 25 M weights): a graph is named
by its rewrite path from the origin, ((rule, site), ...), and a worker rebuilds
it by applying the path (keeping recently built graphs).
"""

from __future__ import annotations

import heapq
import multiprocessing as mp
import os
from collections import OrderedDict

from . import enerflow_oracle as orc

_W: dict = {}


def _init(g0, rules, seed, fn, d, cap, use_inner, db):
    _W.update(g0=g0, rules=rules, seed=seed, fn=fn, d=d, cap=cap, use_inner=use_inner, db=db,
              built=OrderedDict())
    orc.canonical_hash(g0)  # digests of the origin's weight sets, kept for the worker's lifetime
    _W["base_digests"] = dict(orc._WDIGEST)


def _trim():
    """The oracle memoises weight digests by array identity and keeps the arrays alive; rewrites
    derive new arrays (merged / sliced / folded weights) for every candidate, so a long-lived
    worker drops all but the origin's entries now and then (recomputing them is cheap)."""
    if len(orc._WDIGEST) > 512:
        orc._WDIGEST.clear()
        orc._WDIGEST.update(_W["base_digests"])


def _build(path):
    built = _W["built"]
    k = len(path)
    while k > 0 and path[:k] not in built:
        k -= 1
    g = built[path[:k]] if k else _W["g0"]
    for i in range(k, len(path)):
        rule, site = path[i]
        g = orc.apply(rule, g, site)
        built[path[: i + 1]] = g
        built.move_to_end(path[: i + 1])
    if k:
        built.move_to_end(path[:k])
    while len(built) > 16:
        built.popitem(last=False)
    return g


def _expand(path):
    """Every first-per-hash rewrite of the graph at `path`, in (rule, site) order, with what the
    replay needs: hash, node count, the candidate's signature rows the parent lacks (its
    ensure_profiled records), and its evaluation."""
    _trim()
    g = _build(path)
    db, seed, fn, d, cap = _W["db"], _W["seed"], _W["fn"], _W["d"], _W["cap"]
    parent_sigs = set(orc.sig_texts(g).values())
    out = []
    seen = set()
    for rule in _W["rules"]:
        for site in orc.match(rule, g):
            cand = orc.apply(rule, g, site)
            h = orc.canonical_hash(cand)
            if h in seen:
                continue
            seen.add(h)
            nc = orc.n_compute(cand)
            rec = {"step": (rule, site), "hash": h, "nc": nc}
            if nc <= cap:
                new = []
                if seed is not None:
                    texts = orc.sig_texts(cand)
                    shapes = None
                    done = set()
                    for n in sorted(cand["nodes"]):
                        t = texts[n]
                        if cand["nodes"][n]["kind"] == "input" or t in done or t in parent_sigs:
                            continue
                        done.add(t)
                        shapes = shapes or orc.out_shapes(cand)
                        new.append((t, orc.synthetic_rows(orc.sig_fields(cand, n, shapes), t, seed)))
                    orc.ensure_profiled(cand, db, seed)
                rec["new_rows"] = new
                try:
                    if _W["use_inner"]:
                        a, c, t, e, ev, sw = orc.sweep(cand, db, fn, d)
                    else:
                        a, c, t, e, ev, sw = orc.default_eval(cand, db, fn)
                    rec.update(assign=a, cost=c, t=t, e=e, ev=ev, sw=sw)
                except orc.MissingEntry as exc:
                    rec["missing"] = str(exc)
            out.append(rec)
    return out


def outer_search(g0, rules, db: orc.CostDB, f: orc.CostFn, alpha=1.05, d=1, max_queue=100_000,
                 max_graph_nodes=None, seed=None, use_inner=True, trace=None, workers=None, batch=None,
                 progress=None, max_expansions=None):
    """enerflow_oracle.outer_search on `workers` processes (same arguments, same result)."""
    stats = dict.fromkeys(orc.STAT_KEYS, 0)
    cap = max_graph_nodes if max_graph_nodes is not None else 4 * max(1, orc.n_compute(g0))
    workers = workers or os.cpu_count() or 1
    batch = batch or 4 * workers
    if seed is not None:
        stats["new_cost_records"] += orc.ensure_profiled(g0, db, seed)
    evaluate = orc.sweep if use_inner else (lambda g, db, f, d: orc.default_eval(g, db, f))
    a0, c0, t0, e0, ev, sw = evaluate(g0, db, f, d)
    stats["assignments_evaluated"] += ev
    stats["inner_sweeps"] += sw
    best = ((), a0, c0, t0, e0)
    h0 = orc.canonical_hash(g0)
    visited = {h0}
    heap = [(c0, h0)]
    pending = {h0: ()}  # hash -> rewrite path from g0
    cache: dict[int, list] = {}
    inflight: dict = {}  # hash -> AsyncResult of a speculative expansion
    ctx = mp.get_context("fork")
    with ctx.Pool(workers, initializer=_init, initargs=(g0, rules, seed, f, d, cap, use_inner, db)) as pool:
        while heap:
            cost, h = heapq.heappop(heap)
            if cost > alpha * best[2]:
                stats["queue_pruned"] += 1
                pending.pop(h, None)
                cache.pop(h, None)
                inflight.pop(h, None)
                continue
            if max_expansions is not None and stats["graphs_explored"] >= max_expansions:
                break
            path = pending.pop(h)
            stats["graphs_explored"] += 1
            if trace is not None:
                trace.append(h)
            if cost == best[2]:
                stats["expanded_at_best"] += 1
            exp = cache.pop(h, None)
            if exp is None:
                job = inflight.pop(h, None) or pool.apply_async(_expand, (path,))
                # keep the workers busy with the next heap entries while this one is computed;
                # the replay never waits for a speculative expansion it does not need yet
                for k in [k for k, r in inflight.items() if r.ready()]:
                    cache[k] = inflight.pop(k).get()
                room = batch - len(inflight)
                if room > 0:
                    for c2, h2 in heapq.nsmallest(room + len(cache) + 8, heap):
                        if room <= 0:
                            break
                        if c2 <= alpha * best[2] and h2 not in cache and h2 not in inflight:
                            inflight[h2] = pool.apply_async(_expand, (pending[h2],))
                            room -= 1
                exp = job.get()
                if progress and stats["graphs_explored"] % 25 == 0:
                    progress(stats, len(heap))
            for rec in exp:
                stats["graphs_generated"] += 1
                hc = rec["hash"]
                if hc in visited:
                    stats["graphs_deduped"] += 1
                    continue
                visited.add(hc)
                if rec["nc"] > cap:
                    stats["node_cap_hits"] += 1
                    continue
                for text, rows in rec["new_rows"]:
                    if text not in db.rows:
                        for a, t, p in rows:
                            db.add(text, a, t, p)
                            stats["new_cost_records"] += 1
                if "missing" in rec:
                    raise orc.MissingEntry(rec["missing"])
                stats["assignments_evaluated"] += rec["ev"]
                stats["inner_sweeps"] += rec["sw"]
                cc = rec["cost"]
                prev = best[2]
                cpath = path + (rec["step"],)
                if cc < prev:
                    best = (cpath, rec["assign"], cc, rec["t"], rec["e"])
                    stats["best_updates"] += 1
                if cc < alpha * prev:
                    if len(heap) >= max_queue:
                        stats["queue_cap_hits"] += 1
                    else:
                        heapq.heappush(heap, (cc, hc))
                        pending[hc] = cpath
    bpath, a, c, t, e = best
    g = g0
    for rule, site in bpath:
        g = orc.apply(rule, g, site)
    return {"graph": g, "hash": orc.canonical_hash(g), "assignment": a, "cost": c, "time_ms": t,
            "energy": e, "power_w": e / t if t > 0 else 0.0, "stats": stats, "path": bpath}
