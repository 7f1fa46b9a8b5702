"""Break down the e2e upload path: H2D of the packed parents, unpack, full-record hashing."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402
from paper_2005_05837_b200.frontier import Frontier  # noqa: E402

g0 = zoo.generate("resnet50", 0)
db = ef.CostDatabase()
fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), 4096)
s = fr.s
mine = fr.slots[:4096]
recs = [s.read_record(sl) for sl in mine]
blob, offs = s.pack(recs)
slots = [s.alloc() for _ in mine]
out = {}


def timed(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    out[name] = 1e3 * min(t)


pinned = torch.empty(blob.nbytes, dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = blob.view(np.uint8)
dev = torch.empty(blob.nbytes, dtype=torch.uint8, device="cuda")
timed("h2d_torch_pinned_ms", lambda: dev.copy_(pinned, non_blocking=True))
timed("write_packed_ms", lambda: s.write_packed(slots, pinned.numpy().view(np.uint32), offs))
timed("hash_slots_4096_ms", lambda: s.hash_slots(slots))
timed("hash_slots_1024_ms", lambda: s.hash_slots(slots[:1024]))
timed("step_ms", lambda: fr.step(slots, insert_visited=False))
timed("results_only_ms", lambda: s.expand(slots, fr.rule_ids, fr.pp, False))
out["blob_mb"] = blob.nbytes / 1e6
print(json.dumps(out))
