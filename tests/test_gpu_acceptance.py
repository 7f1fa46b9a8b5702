"""The reference's acceptance criteria that run through the search hot path
(reference pkg/tests/test_acceptance.py criteria 6, 7 and 9), on the GPU path,
plus the rewrite closure / exhaustive-space oracle against the reference's
golden vectors."""

import math

import numpy as np
import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo

pytestmark = pytest.mark.gpu


def test_closure_and_brute_force_space_match_reference(golden_small):
    """search.py:275-329: closure membership in BFS order and the exhaustive optimum."""
    checked = 0
    for inst in golden_small:
        space = inst.get("space")
        if not space or "error" in space:
            continue
        g = ef.graph_from_json(inst["graph"])
        rules = [r for r in ef.default_rules() if r.name in inst["rules"]]
        members = ef.closure(g, rules, 2000)
        assert [str(ef.canonical_hash(m)) for m in members] == space["closure"], inst["name"]
        db = ef.CostDatabase()
        for sig, alg, t, p in inst["db"]:
            db.add(sig, alg, ef.CostRecord(t, p))
        res = ef.brute_force_space(g, rules, db, ef.CostFunction.energy(), max_graphs=2000,
                                   profiler=ef.SyntheticProfiler(inst["seed"]))
        assert str(ef.canonical_hash(res.graph)) == space["hash"], inst["name"]
        assert res.cost == space["cost"]
        assert {str(k): v for k, v in res.assignment.items()} == space["assignment"]
        checked += 1
    assert checked >= 40


def test_criterion_06_outer_search_oracle():
    rules = ef.default_rules()
    f = ef.CostFunction.energy()
    exact = checked = seed = 0
    while checked < 100:
        g = zoo.random_graph(seed, ops=6)
        cap = 4 * len(g.compute_nodes())
        db = ef.CostDatabase()
        try:
            oracle = ef.brute_force_space(g, rules, db, f, max_graphs=10_000, profiler=ef.SyntheticProfiler(seed),
                                          max_graph_nodes=cap)
        except ef.SpaceTooLarge:
            seed += 1
            continue
        cfg = ef.SearchConfig(alpha=10.0, d=len(g.compute_nodes()), max_graph_nodes=cap)
        heuristic = ef.outer_search(g, rules, db, f, cfg, ef.SyntheticProfiler(seed))
        assert oracle.cost <= heuristic.cost * (1 + 1e-12), (seed, oracle.cost, heuristic.cost)
        if abs(oracle.cost - heuristic.cost) <= 1e-9 * max(1.0, oracle.cost):
            exact += 1
        checked += 1
        seed += 1
    assert exact >= 95, f"only {exact}/100 matched the oracle"


def test_criterion_07_alpha_valley():
    g, db, rules = zoo.valley_instance()
    r1 = ef.outer_search(g, rules, db, ef.CostFunction.energy(), ef.SearchConfig(alpha=1.0), None)
    r15 = ef.outer_search(g, rules, db, ef.CostFunction.energy(), ef.SearchConfig(alpha=1.5), None)
    assert r15.cost < r1.cost


def _all_cost_points(g, rules, db, profiler, cap):
    points = []
    for graph in ef.closure(g, rules, 2000, cap):
        ef.ensure_profiled(graph, db, profiler)
        table = ef.node_cost_table(graph, db)
        t_grid, e_grid = np.array([0.0]), np.array([0.0])
        for nid in sorted(table):
            rows = table[nid][1]
            t_grid = np.add.outer(t_grid, np.array([t for _, t, _ in rows])).ravel()
            e_grid = np.add.outer(e_grid, np.array([e for _, _, e in rows])).ravel()
        points.extend(zip(t_grid.tolist(), e_grid.tolist()))
    return points


def _pareto(points):
    best_e, out = math.inf, []
    for t, e in sorted(set(points)):
        if e < best_e - 1e-15:
            out.append((t, e))
            best_e = e
    return out


def _lower_hull(points):
    hull = []
    for p in points:
        while len(hull) >= 2:
            (t1, e1), (t2, e2) = hull[-2], hull[-1]
            if (t2 - t1) * (p[1] - e1) - (p[0] - t1) * (e2 - e1) <= 0:
                hull.pop()
            else:
                break
        hull.append(p)
    return hull


def test_criterion_09_tradeoff_sweep():
    rules = ef.default_rules()
    grid = [0.0, 0.25, 0.5, 0.75, 1.0]
    swept = seed = 0
    while swept < 20 and seed < 200:
        g = zoo.random_graph(seed, ops=4)
        db = ef.CostDatabase()
        profiler = ef.SyntheticProfiler(seed)
        cap = 4 * len(g.compute_nodes())
        try:
            ef.ensure_profiled(g, db, profiler)
            refs = ef.normalization_refs(g, db)
            optima = []
            for w in grid:
                f = ef.CostFunction.linear(w).with_refs(*refs)
                res = ef.brute_force_space(g, rules, db, f, max_graphs=2000, profiler=profiler, max_graph_nodes=cap)
                optima.append((res.time_ms, res.energy))
        except ef.SpaceTooLarge:
            seed += 1
            continue
        for (t_lo, e_lo), (t_hi, e_hi) in zip(optima, optima[1:]):
            assert e_hi <= e_lo + 1e-12 and t_hi >= t_lo - 1e-12, (seed, optima)
        swept += 1
        seed += 1
    assert swept == 20

    matched = seed = 0
    while matched < 20 and seed < 1000:
        g = zoo.random_graph(seed, ops=4)
        db = ef.CostDatabase()
        profiler = ef.SyntheticProfiler(seed)
        cap = 4 * len(g.compute_nodes())
        try:
            points = _all_cost_points(g, rules, db, profiler, cap)
        except ef.SpaceTooLarge:
            seed += 1
            continue
        hull = _lower_hull(_pareto(points))
        if len(hull) < 3:
            seed += 1
            continue
        t_ref, e_ref, _ = ef.normalization_refs(g, db)

        def flip_w(p, q):
            dt = (q[0] - p[0]) / t_ref
            de = (q[1] - p[1]) / e_ref
            return dt / (dt - de)

        target_idx = None
        for i in range(1, len(hull) - 1):
            if flip_w(hull[i], hull[i + 1]) - flip_w(hull[i - 1], hull[i]) >= 5e-3:
                target_idx = i
                break
        if target_idx is None:
            seed += 1
            continue
        target = hull[target_idx]
        bound = (target[0] + hull[target_idx + 1][0]) / 2.0
        result = ef.constrained_optimize(g, rules, db, ef.SearchConfig(alpha=10.0, d=1), bound, profiler)
        assert result.time_ms <= bound + 1e-12, seed
        assert abs(result.energy - target[1]) <= 1e-9 * max(1.0, target[1]), (seed, result.energy, target)
        matched += 1
        seed += 1
    assert matched == 20
