"""End-to-end GPU searches (outer_search) of BASELINE configs[0-3]: seconds, expansions, per-expansion
time, for several expansion batch sizes.  Usage: python tools/gpu_search_bench.py [out.jsonl]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402

RUNS = [("squeezenet", "energy", 1.0, None, [1, 64]), ("resnet50", "energy", 1.0, None, [1, 64]),
        ("resnet50", "energy", 1.05, 3000, [1, 16, 64, 256]),
        ("inception_v3", "linear0.5", 1.05, 1000, [1, 64, 256]),
        ("nasnet_a", "energy", 1.05, 1000, [1, 64, 256]), ("nasnet_a", "energy", 1.0, None, [1, 64])]
out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None
for model, obj, alpha, max_exp, batches in RUNS:
    g = zoo.generate(model, 0)
    for b in batches:
        db = ef.CostDatabase()
        ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
        f = ef.CostFunction.energy() if obj == "energy" else \
            ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g, db))
        cfg = ef.SearchConfig(alpha=alpha, max_expansions=max_exp)
        for rep in range(2):  # cold (tables, digests) then warm
            trace = []
            t0 = time.perf_counter()
            res = ef.outer_search(g, ef.default_rules(), db, f, cfg, ef.SyntheticProfiler(0), trace=trace, batch=b)
            dt = time.perf_counter() - t0
        st = res.stats
        row = {"model": model, "objective": obj, "alpha": alpha, "max_expansions": max_exp, "batch": b,
               "warm_s": dt, "ms_per_expansion": 1e3 * dt / max(1, st.graphs_explored),
               "explored": st.graphs_explored, "generated": st.graphs_generated, "cost": res.cost,
               "hash": str(ef.canonical_hash(res.graph)), "trace_tail": str(trace[-1]) if trace else None}
        print(json.dumps(row), flush=True)
        if out:
            out.write(json.dumps(row) + "\n")
            out.flush()
