"""CPU-only checks: host IR / cost model / profiler against the golden vectors, and the
C-ABI library loading with every symbol include/ef200.h declares."""

import os
import re

import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import _native, zoo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_signatures_match_reference(golden_small):
    for inst in golden_small:
        g = ef.graph_from_json(inst["graph"])
        assert {str(k): s.text for k, s in ef.signatures(g).items()} == inst["signatures"], inst["name"]
        assert ef.validate(g) == []


def test_synthetic_profiler_matches_reference(golden_small):
    for inst in golden_small:
        if inst["seed"] is None:
            continue
        g = ef.graph_from_json(inst["graph"])
        db = ef.CostDatabase()
        ef.ensure_profiled(g, db, ef.SyntheticProfiler(inst["seed"]))
        got = sorted([s, a, r.time_ms, r.power_w] for (s, a), r in db.records().items())
        assert got == sorted(inst["db"]), inst["name"]


def test_reference_instances_identical(golden_small):
    by = {i["name"]: i for i in golden_small}
    for seed in range(40):
        assert ef.graph_to_json(zoo.random_graph(seed, max_ops=8)) == by[f"random-{seed}"]["graph"]
    assert ef.graph_to_json(zoo.toy_squeeze(0)) == by["toy-squeeze"]["graph"]
    assert ef.graph_to_json(zoo.toy_resnet(0)) == by["toy-resnet"]["graph"]
    assert ef.graph_to_json(zoo.microbench_graph()) == by["microbench"]["graph"]
    g, db, _ = zoo.valley_instance()
    assert ef.graph_to_json(g) == by["valley"]["graph"]
    assert sorted([s, a, r.time_ms, r.power_w] for (s, a), r in db.records().items()) == sorted(by["valley"]["db"])


def test_microbench_table():
    g, db = zoo.microbench_graph(), zoo.microbench_database()
    ids = [n.id for n in g.compute_nodes()]
    a = {ids[0]: 1, ids[1]: 0, ids[2]: 2}
    assert ef.model_energy(g, a, db) == pytest.approx(14.195, rel=1e-9)
    assert ef.brute_force_assignment(g, db, ef.CostFunction.energy()) == a


def test_models_validate():
    for name in ("squeezenet", "resnet50", "inception_v3", "nasnet_a"):
        g = zoo.generate(name)
        assert ef.validate(g) == [], name
    g = zoo.random_dag(2000, 1)
    assert ef.validate(g) == [] and len(g.nodes) > 1500


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    header = open(os.path.join(ROOT, "include", "ef200.h")).read()
    declared = set(re.findall(r"^(?:int|void\*?|ef_ctx\*|const char\*)\s+(ef_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name


def test_no_cpu_fallback_without_device():
    if _native.load_library().ef_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(ef.NativeUnavailable):
        ef.canonical_hash(zoo.toy_squeeze(0))
