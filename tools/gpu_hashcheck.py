"""Check incremental candidate hashes against a full recomputation (development aid)."""
import sys, collections
sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo, _native as N
from paper_2005_05837_b200.frontier import Frontier

model = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
npar = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g0 = zoo.generate(model, 0)
db = ef.CostDatabase()
fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), npar)
s = fr.s
res = fr.step()
print("candidates", len(res), "first", sum(1 for r in res if r.flags & N.F_FIRST))
idx = list(range(len(res)))
slots = s.keep(idx)
full = s.hash_slots(slots)
bad = [(i, res[i].rule, res[i].site_a, res[i].site_b) for i in idx if full[i] != res[i].hash]
print("mismatches", len(bad), "by rule", collections.Counter(b[1] for b in bad))
print(bad[:10])
# decode a few and compare with host-side recompute via upload+hash
for i in [b[0] for b in bad[:3]]:
    g = s.decode(s.read_record(slots[i]), g0)[0]
    print("cand", i, "incremental", res[i].hash, "full", full[i], "reupload", ef.canonical_hash(g) if model != "resnet50" else "-")
