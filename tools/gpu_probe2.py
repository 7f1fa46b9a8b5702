import faulthandler, json, sys, time
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef
gold = json.load(open("tests/golden/golden_small.json"))["instances"]
for inst in gold:
    t0 = time.perf_counter()
    g = ef.graph_from_json(inst["graph"])
    rules = [r for r in ef.default_rules() if r.name in inst["rules"]]
    bad = []
    for rule in rules:
        print(inst["name"], rule.name, "match", flush=True)
        sites = ef.match_rule(rule, g)
        if [[v for _, v in s.binding] for s in sites] != inst["sites"][rule.name]:
            bad.append(("sites", rule.name))
        for s in sites:
            print(inst["name"], rule.name, "apply", s.binding, flush=True)
            ef.apply(rule, g, s)
    print(inst["name"], f"{1e3*(time.perf_counter()-t0):.1f} ms", bad, flush=True)
