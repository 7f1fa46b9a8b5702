"""ncu launch list of one full-record hash of 4096 ResNet-50 frontier records."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2005_05837_b200 as ef  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402
from paper_2005_05837_b200.frontier import Frontier  # noqa: E402

g0 = zoo.generate("resnet50", 0)
db = ef.CostDatabase()
fr = Frontier(g0, db, ef.SyntheticProfiler(0), ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), 4096)
s = fr.s
s.hash_slots(fr.slots)
torch.cuda.synchronize()
torch.cuda.profiler.start()
s.hash_slots(fr.slots)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
