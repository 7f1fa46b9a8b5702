"""Benchmark: candidate graphs priced per second on the frontier of a search.

A step = one frontier expansion of a batch of parent graphs resident in HBM:
every substitution rule at every match site of every parent, materialisation,
canonical hashing, dedup (within the step and against the visited set) and
the inner search on every survivor (libef200 `ef_expand`).  The workload is
BASELINE.json configs[1]: ResNet-50 inference graph, energy objective with
per-node algorithm selection, alpha = 1.05; the parents are the real frontier
of that search (the first graphs its best-first order enqueues).

`value`  = candidates priced / s, device time (CUDA events on the library's
           stream), inputs already in HBM; max over ranks for N > 1.
`e2e`    = the same metric through the C ABI with host buffers: parent
           records copied host->device and results copied back every step.
`--impl reference` times the CPU oracle (oracle/, a restatement of the
reference's Python code path) on a bounded sample of the same workload.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODEL = "resnet50"
CONFIG_NAME = "ResNet-50 inference graph, energy objective with per-node conv-algorithm selection, alpha=1.05"
METRIC = "candidate graphs priced/sec"
UNIT = "candidates/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self):
        self.proc = None
        self.rows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self, device: int) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8 or not parts[0].isdigit() or int(parts[0]) != device:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _setup_workload(n_parents: int, world: int, rank: int):
    import paper_2005_05837_b200 as ef
    from paper_2005_05837_b200 import zoo
    from paper_2005_05837_b200.frontier import Frontier

    g0 = zoo.generate(MODEL, 0)
    db = ef.CostDatabase()
    prof = ef.SyntheticProfiler(0)
    fr = Frontier(g0, db, prof, ef.CostFunction.energy(), ef.SearchConfig(alpha=1.05), n_parents * world)
    # weak scaling: this rank owns its slice of the frontier (graphs are independent objects)
    mine = fr.slots[rank * n_parents:(rank + 1) * n_parents]
    return ef, g0, db, fr, mine


def _to_oracle(g):
    """Package Graph -> oracle graph dict, sharing the weight arrays (no copies)."""
    nodes = {}
    for nid, v in g.nodes.items():
        nodes[nid] = {"kind": v.kind.value, "ins": [(r.node, r.port) for r in v.inputs],
                      "p": dict(v.params), "w": dict(v.weights)}
    return {"inputs": [(n, tuple(s.dims)) for n, s in g.inputs], "nodes": nodes,
            "outputs": [(r.node, r.port) for r in g.outputs]}


def _oracle_db(db):
    from oracle import enerflow_oracle as orc

    odb = orc.CostDB()
    for (sig, alg), rec in db.records().items():
        odb.add(sig, alg, rec.time_ms, rec.power_w)
    return odb


def _oracle_expand(parent, odb, seed: int, visited: set) -> tuple[int, int]:
    """The reference's per-expansion work on one parent: neighbors (rewrite + hash +
    in-expansion dedup), visited dedup, profiling and the inner search of every survivor."""
    from oracle import enerflow_oracle as orc

    f = orc.CostFn("energy")
    rules = ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs", "split-merged-conv",
             "fold-identity", "fuse-conv-batchnorm"]
    generated = priced = 0
    for cand in orc.neighbors(parent, rules):
        generated += 1
        h = orc.canonical_hash(cand)
        if h in visited:
            continue
        visited.add(h)
        orc.ensure_profiled(cand, odb, seed)
        orc.sweep(cand, odb, f, 1)
        priced += 1
    return generated, priced


def _cpu_sample(parents, db, budget_s: float) -> dict:
    odb = _oracle_db(db)
    t0 = time.perf_counter()
    priced = generated = expanded = 0
    visited: set = set()
    for p in parents:
        gen, pr = _oracle_expand(p, odb, 0, visited)
        generated += gen
        priced += pr
        expanded += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": priced / dt, "priced": priced, "generated": generated, "expanded": expanded, "seconds": dt}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    import paper_2005_05837_b200 as ef  # host IR only (graph builder + profiler), no GPU
    from paper_2005_05837_b200 import zoo
    from oracle import enerflow_oracle as orc

    # the same frontier, built on the CPU with the oracle (no GPU on this arm)
    g0 = zoo.generate(MODEL, 0)
    db = ef.CostDatabase()
    ef.ensure_profiled(g0, db, ef.SyntheticProfiler(0))
    og = _to_oracle(g0)
    odb = _oracle_db(db)
    frontier = [og]
    for cand in orc.neighbors(og, ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs",
                                   "split-merged-conv", "fold-identity", "fuse-conv-batchnorm"]):
        frontier.append(cand)
        if len(frontier) >= args.steps + args.warmup + 1:
            break
    times, priced = [], []
    for i in range(args.warmup + args.steps):
        visited: set = set()
        t0 = time.perf_counter()
        _, pr = _oracle_expand(frontier[i % len(frontier)], odb, 0, visited)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            priced.append(pr)
    value = sum(priced) / sum(times)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64",
            "data": "synthetic (random-init weights, synthetic profiler seed 0)",
            "config": {"workload": CONFIG_NAME, "model": MODEL, "parents_per_step": 1,
                       "sample": "one frontier expansion per step (oracle restatement of reference search.py)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": f"{args.steps} expansions of ResNet-50 frontier graphs, "
                                       f"{sum(priced)} candidates priced"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args, world, rank, local):
    import ctypes as C

    import numpy as np

    ef, g0, db, fr, mine = _setup_workload(args.parents, world, rank)
    from paper_2005_05837_b200 import _native as N

    s = fr.s
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    # L2 flush buffer (written between timed steps; the step's own arena already exceeds L2)
    flush_bytes = 256 << 20
    flush = None
    try:
        import torch

        flush = torch.empty(flush_bytes, dtype=torch.uint8, device=f"cuda:{local}")
    except Exception:
        flush = None

    def flush_l2():
        if flush is not None:
            flush.fill_(1)
            torch.cuda.synchronize()

    def step():
        res = fr.step(mine, insert_visited=False)
        return res, s.last_timing()

    for _ in range(args.warmup):
        step()
    prof = os.environ.get("EF_NCU") == "1"  # ncu --profile-from-start off: capture the timed steps only
    if prof:
        import torch

        torch.cuda.profiler.start()
    clocks = Clocks()
    clocks.start()
    dev_ms, stage_ms, priced_n, gen_n = [], [0.0] * 5, 0, 0
    for _ in range(args.steps):
        flush_l2()
        barrier()
        res, ms = step()
        dev_ms.append(sum(ms))
        stage_ms = [a + b for a, b in zip(stage_ms, ms)]
        priced_n += int(np.count_nonzero(res["flags"] & N.F_PRICED))
        gen_n += len(res)
    clk = clocks.stop(local)
    if prof:
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"ncu_capture": True, "stages_ms": stage_ms}))
        return 0
    total_ms = sum(dev_ms)
    if dist is not None:
        import torch

        t = torch.tensor([total_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        pr = torch.tensor([float(priced_n)], device=f"cuda:{local}")
        dist.all_reduce(pr)
        priced_all = float(pr.item())
    else:
        priced_all = float(priced_n)
    value = priced_all / (total_ms / 1e3)

    # e2e through the C ABI with host buffers: parent records H2D, results D2H, every step
    host_recs = [s.read_record(sl) for sl in mine]
    rec_bytes = host_recs[0].nbytes
    e2e_slots = [s.alloc() for _ in mine]
    pinned = s.L.ef_host_alloc(rec_bytes * len(mine))
    staging = np.ctypeslib.as_array((C.c_uint8 * (rec_bytes * len(mine))).from_address(pinned))
    for i, buf in enumerate(host_recs):
        staging[i * rec_bytes:(i + 1) * rec_bytes] = buf
    slot_arr = N.u32_array(e2e_slots)
    e2e_times, e2e_priced = [], 0
    for i in range(args.warmup + args.steps):
        flush_l2()
        barrier()
        t0 = time.perf_counter()
        s._check(s.L.ef_records_write(s.ctx, slot_arr, len(e2e_slots), pinned, rec_bytes, rec_bytes),
                 "ef_records_write")
        res = fr.step(e2e_slots, insert_visited=False)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            e2e_times.append(dt)
            e2e_priced += int(np.count_nonzero(res["flags"] & N.F_PRICED))
    n_cand = len(res)
    s.L.ef_host_free(pinned)
    e2e_total = sum(e2e_times)
    if dist is not None:
        import torch

        t = torch.tensor([e2e_total, float(e2e_priced)], device=f"cuda:{local}", dtype=torch.float64)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t)
        e2e_total, e2e_priced = float(mx[0].item()), float(t[1].item())
    e2e_value = e2e_priced / e2e_total

    # roofline of the dominant stage, from the live per-stage CUDA-event times
    stage_names = ["match", "materialise", "hash", "dedup", "price"]
    dom = max(range(5), key=lambda k: stage_ms[k])
    peak, peak_kind = _peaks()
    geo = s.geo
    # algorithmic bytes of one step: every candidate's record is read from
    # the parent and written once (used bytes only), its keys written, results written
    n_nodes = np.mean([int(np.frombuffer(b[:16].tobytes(), dtype=np.int32)[0]) for b in host_recs])
    n_refs = np.mean([int(np.frombuffer(b[:16].tobytes(), dtype=np.int32)[1]) for b in host_recs])
    per_cand_record = 4 * (6 * n_nodes + n_refs) + 16 * n_nodes + n_nodes
    per_step_cands = gen_n / args.steps
    algo = {
        "materialise": 2 * per_cand_record * per_step_cands,
        "hash": (per_cand_record + 16 * n_nodes) * per_step_cands,
        "price": (4 * n_nodes + n_nodes + 40 * n_nodes) * priced_n / args.steps,
        "match": (per_cand_record + 16 * n_nodes) * len(mine),
        "dedup": 80 * 2 * per_step_cands,
    }
    dom_name = stage_names[dom]
    dom_ms = stage_ms[dom] / args.steps
    achieved = algo[dom_name] / (dom_ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64",
        "data": "synthetic (random-init float64 weights, synthetic profiler seed 0)",
        "config": {"workload": CONFIG_NAME, "model": MODEL, "parents_per_gpu": len(mine),
                   "candidates_per_step": per_step_cands, "priced_per_step": priced_n / args.steps,
                   "rules": "all 6", "inner_search_d": 1,
                   "l2": "flushed (256 MiB write) before every timed step; per-step arena > L2",
                   "parallelism": f"frontier sharded over {world} GPU(s)"},
        "stages_ms_per_step": {n: stage_ms[k] / args.steps for k, n in enumerate(stage_names)},
        "roofline": {"bound": "hbm", "kernel": f"k_{dom_name}", "achieved": achieved, "peak": peak,
                     "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": None},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": rec_bytes * len(mine),
                "d2h_bytes_per_step": n_cand * N.CAND_DTYPE.itemsize},
        "gpu_launches": 7 * args.steps,
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        parents = [_to_oracle(fr.decode(sl)) for sl in mine[:8]]
        cpu = _cpu_sample(parents, db, args.cpu_budget)
        line["cpu_baseline"] = {"value": cpu["value"], "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{cpu['expanded']} frontier expansions ({cpu['priced']} candidates "
                                          f"priced) by the oracle restatement, {cpu['seconds']:.1f}s"}
    if rank == 0:
        print(json.dumps(line))
    fr.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--parents", type=int, default=256, help="frontier graphs per GPU per step")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    world, rank, local = _dist()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
