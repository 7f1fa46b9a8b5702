"""The recorded bench frontiers (bench_frontiers/, tools/make_frontier_fixture.py on the GPU):
rebuilt on the host by the oracle from their rewrite paths, the parents have the recorded
canonical hashes, so `bench.py --impl reference` expands exactly the graphs our arm expands."""

import glob
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURES = sorted(glob.glob(os.path.join(ROOT, "bench_frontiers", "*.json")))


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_fixture_rebuilds_recorded_parents(path):
    import bench
    from oracle import enerflow_oracle as orc

    with open(path) as fh:
        fx = json.load(fh)
    assert fx["rules"] == bench.RULES
    assert len(fx["paths"]) == len(fx["hashes"]) == len(fx["nodes"]) == fx["n_parents"]
    # the deepest path and the first parents (a path prefix is rebuilt once)
    pick = sorted({0, 1, max(range(len(fx["paths"])), key=lambda i: len(fx["paths"][i]))})
    pick = [i for i in pick if i < len(fx["paths"])][:3 if fx["nodes"][0] < 5000 else 2]
    parents, _, _, _ = bench.oracle_frontier(fx["workload"], [fx["paths"][i] for i in pick])
    for i, g in zip(pick, parents):
        assert len(g["nodes"]) == fx["nodes"][i]
        assert str(orc.canonical_hash(g)) == fx["hashes"][i], (fx["workload"], i)


def test_load_fixture_prefix_and_config():
    import bench

    if not FIXTURES:
        pytest.skip("no recorded frontier")
    with open(FIXTURES[0]) as fh:
        fx = json.load(fh)
    got = bench.load_fixture(fx["workload"], 1)
    assert got is not None and got["n_parents"] >= 1
    assert bench.load_fixture(fx["workload"], 10**9) is None
    a = bench.bench_config(fx["workload"], 4, 10.0)
    b = bench.bench_config(fx["workload"], 4, 10.0)
    assert a == b and a["model"] == fx["workload"] and a["alpha"] == fx["alpha"]
