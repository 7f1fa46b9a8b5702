"""Size of the full searches of BASELINE configs[0-3] on the GPU (one config per process, bounded)."""
import json
import subprocess
import sys
import time

CONFIGS = [("squeezenet", "energy", 1.0), ("squeezenet", "energy", 1.05), ("resnet50", "energy", 1.0),
           ("resnet50", "energy", 1.05), ("inception_v3", "linear0.5", 1.05), ("nasnet_a", "energy", 1.05),
           ("nasnet_a", "energy", 1.0), ("inception_v3", "energy", 1.05)]


def one(model, objective, alpha):
    sys.path.insert(0, ".")
    import paper_2005_05837_b200 as ef
    from paper_2005_05837_b200 import zoo

    g = zoo.generate(model, 0)
    db = ef.CostDatabase()
    ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
    f = ef.CostFunction.energy() if objective == "energy" else \
        ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g, db))
    t0 = time.perf_counter()
    trace = []
    res = ef.outer_search(g, ef.default_rules(), db, f, ef.SearchConfig(alpha=alpha), ef.SyntheticProfiler(0),
                          trace=trace)
    st = res.stats
    print(json.dumps({"model": model, "objective": objective, "alpha": alpha, "search_s": time.perf_counter() - t0,
                      **{k: v for k, v in vars(st).items()}, "cost": res.cost}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(sys.argv[1], sys.argv[2], float(sys.argv[3]))
        sys.exit(0)
    limit = float(sys.argv[1]) if len(sys.argv) > 1 else 240
    for m, o, a in CONFIGS:
        t0 = time.time()
        try:
            p = subprocess.run([sys.executable, __file__, m, o, str(a)], timeout=240, capture_output=True, text=True)
            print(p.stdout.strip() or p.stderr[-2000:], flush=True)
        except subprocess.TimeoutExpired:
            print(json.dumps({"model": m, "objective": o, "alpha": a, "timeout_s": time.time() - t0}), flush=True)
