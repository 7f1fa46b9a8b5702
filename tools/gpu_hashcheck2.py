import sys, collections
import numpy as np
sys.path.insert(0, ".")
import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo, _native as N
from paper_2005_05837_b200.frontier import Frontier

for model, npar in (("squeezenet", 8), ("resnet50", 4)):
    g0 = zoo.generate(model, 0)
    db = ef.CostDatabase()
    fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), npar)
    s = fr.s
    G = s.geo
    res = fr.step()
    idx = list(range(len(res)))
    slots = s.keep(idx)
    inc = [s.read_record(sl) for sl in slots]
    full = s.hash_slots(slots)
    fl = [s.read_record(sl) for sl in slots]
    bad = [i for i in idx if full[i] != res[i].hash]
    print(model, "candidates", len(res), "mismatches", len(bad), collections.Counter(res[i].rule for i in bad))
    for i in bad[:4]:
        n = int(inc[i][:4].view(np.int32)[0])
        ki = inc[i][G.off_keys:G.off_keys + 16 * n].view(np.uint64).reshape(n, 2)
        kf = fl[i][G.off_keys:G.off_keys + 16 * n].view(np.uint64).reshape(n, 2)
        diff = np.nonzero((ki != kf).any(axis=1))[0]
        si = inc[i][G.off_sperm:G.off_sperm + 4 * n].view(np.uint32)
        sf = fl[i][G.off_sperm:G.off_sperm + 4 * n].view(np.uint32)
        print("  cand", i, "rule", res[i].rule, "site", res[i].site_a, res[i].site_b, "n", n,
              "key diffs at", diff[:10].tolist(), "n_diff", len(diff), "sperm equal", bool((si == sf).all()),
              "sorted-key-seq equal", bool((ki[si] == kf[sf]).all()))
    [s.free(x) for x in slots]
    fr.close()
