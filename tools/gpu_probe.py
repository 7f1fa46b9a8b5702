"""Quick timing probe of the GPU entry points (development aid)."""
import faulthandler
import json
import sys
import time

faulthandler.dump_traceback_later(120, exit=True)
sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo

gold = json.load(open("tests/golden/golden_small.json"))["instances"]
by = {i["name"]: i for i in gold}
inst = by["toy-squeeze"]
g = ef.graph_from_json(inst["graph"])


def t(label, fn):
    t0 = time.perf_counter()
    out = fn()
    print(f"{label}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    return out


t("hash#1", lambda: ef.canonical_hash(g))
t("hash#2", lambda: ef.canonical_hash(g))
rules = ef.default_rules()
sites = t("match", lambda: ef.match_rule(rules[0], g))
print("sites", [s.binding for s in sites], inst["sites"]["fuse-conv-relu"], flush=True)
t("match2", lambda: ef.match_rule(rules[0], g))
g2 = t("apply", lambda: ef.apply(rules[0], g, sites[0]))
h = t("hash apply", lambda: ef.canonical_hash(g2))
print("rewrite hash", h, inst["rewrites"][0], flush=True)
nb = t("neighbors", lambda: ef.neighbors(g, rules))
print([str(ef.canonical_hash(c)) for c in nb] == inst["neighbors"], flush=True)
db = ef.CostDatabase()
for sig, alg, tt, p in inst["db"]:
    db.add(sig, alg, ef.CostRecord(tt, p))
trace = []
res = t("outer", lambda: ef.outer_search(g, rules, db, ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05),
                                         ef.SyntheticProfiler(0), trace=trace))
run = inst["searches"][0]
print("trace ok", [str(x) for x in trace] == run["trace"], len(trace), len(run["trace"]))
print("cost", res.cost, run["cost"], res.stats, run["stats"], flush=True)
