"""How well does the pipelined e2e loop overlap the next batch's upload with the current step?

Times (wall clock, synchronised) K iterations of: (a) step only, (b) async upload + fence only,
(c) the bench's pipelined loop (upload i+1 on the upload stream, then step i).
"""
import ctypes as C
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402
from paper_2005_05837_b200.frontier import Frontier  # noqa: E402

K = 8
g0 = zoo.generate("resnet50", 0)
db = ef.CostDatabase()
fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), 4096)
s = fr.s
mine = fr.slots[:4096]
recs = [s.read_record(sl) for sl in mine]
blob, offs = s.pack(recs)
pinned = s.L.ef_host_alloc(blob.nbytes)
staging = np.ctypeslib.as_array((C.c_uint8 * blob.nbytes).from_address(pinned))
staging[:] = blob.view(np.uint8)
sets = [[s.alloc() for _ in mine], [s.alloc() for _ in mine]]
s.write_packed(sets[0], staging.view(np.uint32), offs)
s.write_packed(sets[1], staging.view(np.uint32), offs)
out = {}


def run(name, body):
    body(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        body(i)
    torch.cuda.synchronize()
    out[name] = 1e3 * (time.perf_counter() - t0) / K


def step_only(i):
    fr.step(sets[i % 2], insert_visited=False)


def upload_only(i):
    s.write_packed(sets[i % 2], staging.view(np.uint32), offs, asynchronous=True)
    s.upload_fence()


def pipelined(i):
    s.write_packed(sets[(i + 1) % 2], staging.view(np.uint32), offs, asynchronous=True)
    fr.step(sets[i % 2], insert_visited=False)
    s.upload_fence()


run("step_only_ms", step_only)
run("upload_only_ms", upload_only)
run("pipelined_ms", pipelined)
# host time inside the call that issues the async upload
t = []
for i in range(K):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.write_packed(sets[i % 2], staging.view(np.uint32), offs, asynchronous=True)
    t.append(time.perf_counter() - t0)
    s.upload_fence()
torch.cuda.synchronize()
out["upload_issue_host_ms"] = 1e3 * min(t)
t = []
for i in range(K):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fr.step(sets[i % 2], insert_visited=False)
    t.append(time.perf_counter() - t0)
out["step_wall_ms"] = 1e3 * min(t)
out["step_device_ms"] = s.last_step_ms()
print(json.dumps(out))
