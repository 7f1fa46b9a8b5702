"""Full outer-search goldens made by running the REAL reference (`enerflow`) here.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_search_ref.py resnet50 1.0

Records the traced outer search (explored-hash sequence, optimised graph hash,
assignment, cost/time/energy, every SearchStats counter) of a zoo model
(seed 0) under the energy objective at the given alpha, using the reference's
own `outer_search` (search.py:211-272) with `SyntheticProfiler(0)`.  Output:
tests/golden/golden_search_ref_<model>_a<alpha>.json.  The real reference
re-digests every weight tensor per canonical hash, so ResNet-50 at alpha = 1.0
takes on the order of an hour of one core.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden_models import to_reference, traced_outer  # noqa: E402  (imports the real enerflow)

from enerflow import CostDatabase, canonical_hash  # noqa: E402
from paper_2005_05837_b200 import zoo  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
    alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    t0 = time.perf_counter()
    g = to_reference(zoo.generate(name, 0))
    res = traced_outer(g, CostDatabase(), alpha)
    out = {"generator": "tests/golden/make_golden_search_ref.py", "python": sys.version.split()[0],
           "model": name, "seed": 0, "objective": "energy", "origin_hash": str(canonical_hash(g)),
           "search": res, "reference_seconds": time.perf_counter() - t0}
    path = os.path.join(HERE, f"golden_search_ref_{name}_a{alpha:g}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, sort_keys=True)
    print("wrote", path, f"{out['reference_seconds']:.0f}s", len(res["trace"]), "expansions")


if __name__ == "__main__":
    main()
