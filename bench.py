"""Benchmark: candidate graphs priced per second on the frontier of a search.

A step = one frontier expansion of a batch of parent graphs resident in HBM:
every substitution rule at every match site of every parent, the rewrite plans,
canonical hashing, deduplication (within the step and against the visited set)
and the inner search on every survivor (libef200 `ef_expand`).  The default
workload is BASELINE.json configs[4], the configuration its candidates/s sweep
over 1/2/4/8 GPUs is quoted on: the largest synthetic random DAG (20k ops, the
full rule set, energy objective, alpha = 1.05).  The parents are the real
frontier of that search (the graphs its best-first order expands first),
--parents per GPU; they are recorded as rewrite paths in bench_frontiers/ so the
reference arm expands the very same graphs.  ResNet-50 (configs[1]) is measured
beside it (`workloads`), and the searches of configs[0-3] end to end (`search`).

`value`  candidates priced / s over all ranks: device time of the step (CUDA
         events), inputs already in HBM, L2 flushed before every step; max over
         ranks.  With N > 1 GPUs the frontier is split by parent and
         deduplication is owned by hash (NCCL all-to-all, shard.py).
`e2e`    the same metric through the C ABI from host memory: compact parent
         records (used bytes only, pinned) copied host->device, unpacked and
         hashed on the device, the step, and every candidate's result copied
         back, all inside the timed region.
`roofline`  the dominant kernel (k_keys / k_keys_wide: node-key BLAKE2b) is
         integer-ALU bound; its compression rate against the live register-only
         BLAKE2b rate of the same GPU.  `roofline_hbm` gives its algorithmic
         bytes against HBM.
`cpu_baseline` / `--impl reference`: the oracle restatement of the reference's
         path (oracle/, pinned to the reference's golden vectors) on the host.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W]
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

DEFAULT_WORKLOAD = "dag:20000"
# --workload: the BASELINE.json configs as frontier workloads (name, objective, parents per GPU)
WORKLOADS = {
    "dag:20000": ("synthetic random-DAG conv/matmul graph, 20k ops, full rule set, energy objective, alpha=1.05 "
                  "(BASELINE configs[4], largest synthetic graph)", "energy", 9),
    "resnet50": ("ResNet-50 inference graph, energy objective with per-node conv-algorithm selection, alpha=1.05 "
                 "(BASELINE configs[1])", "energy", 4096),
    "squeezenet": ("SqueezeNet inference graph, energy objective, alpha=1.0 search frontier (BASELINE configs[0])",
                   "energy", 4096),
    "inception_v3": ("Inception-v3 graph, energy-delay tradeoff objective (normalized linear w=0.5), alpha=1.05 "
                     "(BASELINE configs[2])", "linear0.5", 2048),
    "nasnet_a": ("NasNet-A style cell-stacked graph, energy objective, alpha=1.05 (BASELINE configs[3])", "energy",
                 1024),
    "dag:1000": ("synthetic random-DAG conv/matmul graph, 1k ops, full rule set (BASELINE configs[4])", "energy", 256),
    "dag:5000": ("synthetic random-DAG conv/matmul graph, 5k ops, full rule set (BASELINE configs[4])", "energy", 32),
}
FRONTIER_DIR = os.path.join(ROOT, "bench_frontiers")


def workload_alpha(workload: str) -> float:
    return 1.0 if workload == "squeezenet" else 1.05


def fixture_name(workload: str, n: int) -> str:
    return f"{workload.replace(':', '_')}_{n}.json"


def load_fixture(workload: str, n: int):
    """The recorded frontier of `workload` with at least n parents (tools/make_frontier_fixture.py),
    or None.  The first n parents of a larger batch are the n-parent batch."""
    best = None
    if os.path.isdir(FRONTIER_DIR):
        stem = workload.replace(":", "_") + "_"
        for f in os.listdir(FRONTIER_DIR):
            if f.startswith(stem) and f.endswith(".json"):
                k = int(f[len(stem):-5])
                if k >= n and (best is None or k < best[0]):
                    best = (k, f)
    if best is None:
        return None
    with open(os.path.join(FRONTIER_DIR, best[1])) as fh:
        fx = json.load(fh)
    fx["file"] = os.path.join("bench_frontiers", best[1])
    return fx


def bench_config(workload: str, parents_per_gpu: int, nodes_per_parent: float) -> dict:
    """The workload's `config`, identical in both arms."""
    name, objective, _ = WORKLOADS[workload]
    return {"workload": name, "model": workload, "objective": objective, "alpha": workload_alpha(workload),
            "parents_per_gpu": parents_per_gpu, "nodes_per_parent": nodes_per_parent, "rules": "all 6",
            "inner_search_d": 1}


def _objective(ef, kind: str, g0, db):
    if kind == "energy":
        return ef.CostFunction.energy()
    return ef.CostFunction.linear(0.5).with_refs(*ef.normalization_refs(g0, db))


METRIC = "candidate graphs priced/sec"
UNIT = "candidates/s"
RULES = ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs", "split-merged-conv", "fold-identity",
         "fuse-conv-batchnorm"]


# the committed `ncu --set full` captures, newest first (tools/ncu_summary.py): the traffic
# figure of a kernel comes from the newest capture that holds it
PROFILES = [os.path.join("profiles", f) for f in ("ncu_r02d_dag20k_kernels.json", "ncu_r02d_resnet50_kernels.json",
                                                   "ncu_r02c_dag20k_kernels.json", "ncu_r02c_resnet50_kernels.json",
                                                   "ncu_r02aa_dag20k_kernels.json", "ncu_r02aa_resnet50_kernels.json",
                                                   "ncu_r02w_kernels.json", "ncu_r01f_kernels.json")]


def _traffic(kernel: str):
    """(DRAM bytes read + written by one launch of `kernel` in the newest committed ncu capture
    that has it, that capture's path), or (None, None)."""
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for prof in PROFILES:
        try:
            with open(os.path.join(ROOT, prof)) as fh:
                rows = json.load(fh)
        except (OSError, ValueError):
            continue
        for r in rows:
            if kernel in (r.get("Kernel Name") or ""):
                tot = 0.0
                for k, v in r.items():
                    if k.startswith("dram__bytes_read.sum") or k.startswith("dram__bytes_write.sum"):
                        unit = k.split("[")[-1].rstrip("]").strip() if "[" in k else "byte"
                        tot += float(v) * scale.get(unit, 1)
                return tot, prof
    return None, None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self):
        self.proc = None

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
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def _to_oracle(g):
    """Package Graph -> oracle graph dict, sharing the weight arrays (no copies)."""
    nodes = {nid: {"kind": v.kind.value, "ins": [(r.node, r.port) for r in v.inputs], "p": dict(v.params),
                   "w": dict(v.weights)} for nid, v in g.nodes.items()}
    return {"inputs": [(n, tuple(s.dims)) for n, s in g.inputs], "nodes": nodes,
            "outputs": [(r.node, r.port) for r in g.outputs]}


def _oracle_db(db):
    from oracle import enerflow_oracle as orc

    odb = orc.CostDB()
    for (sig, alg), rec in db.records().items():
        odb.add(sig, alg, rec.time_ms, rec.power_w)
    return odb


def _oracle_objective(objective: str, og, odb):
    from oracle import enerflow_oracle as orc

    if objective == "energy":
        return orc.CostFn("energy")
    return orc.CostFn("linear", w=0.5, refs=orc.normalization_refs(og, odb))


def _oracle_expand(parent, odb, f, visited: set, deadline: float | None = None) -> tuple[int, int]:
    """The reference's per-expansion work on one parent (search.py:245-267): neighbors
    (rewrite + canonical hash + in-expansion dedup), visited dedup, profiling of new
    signatures and the inner search of every survivor.  Stops at `deadline` (perf_counter)."""
    from oracle import enerflow_oracle as orc

    generated = priced = 0
    seen: set = set()
    for rule in RULES:  # neighbors() unrolled so the sample can stop inside a large expansion
        for site in orc.match(rule, parent):
            if deadline is not None and time.perf_counter() > deadline:
                return generated, priced
            cand = orc.apply(rule, parent, site)
            h = orc.canonical_hash(cand)
            if h in seen:
                continue
            seen.add(h)
            generated += 1
            if h in visited:
                continue
            visited.add(h)
            orc.ensure_profiled(cand, odb, 0)
            orc.sweep(cand, odb, f, 1)
            priced += 1
    return generated, priced


def oracle_frontier(workload: str, paths: list) -> tuple[list, object, object, object]:
    """The frontier parents rebuilt on the host by the oracle from their rewrite paths (a path
    indexes each rewrite in its parent's (rule, site) enumeration, rules.neighbors order).
    -> (parents, origin, oracle cost db, oracle objective)."""
    import paper_2005_05837_b200 as ef  # host IR only (graph builder + profiler), no GPU
    from oracle import enerflow_oracle as orc
    from paper_2005_05837_b200 import zoo

    g0 = zoo.generate(workload, 0)
    db = ef.CostDatabase()
    ef.ensure_profiled(g0, db, ef.SyntheticProfiler(0))
    og = _to_oracle(g0)
    odb = _oracle_db(db)
    memo = {(): og}

    def build(path):
        path = tuple(path)
        if path not in memo:
            g = build(path[:-1])
            rule, site = [(r, st) for r in RULES for st in orc.match(r, g)][path[-1]]
            memo[path] = orc.apply(rule, g, site)
        return memo[path]

    parents = [build(p) for p in paths]
    return parents, og, odb, _oracle_objective(WORKLOADS[workload][1], og, odb)


# ---------------------------------------------------------------------------------------------
# reference arm: the oracle port of the reference's path on every host core
# ---------------------------------------------------------------------------------------------

_REF_STATE: dict = {}


def _ref_worker(i: int) -> int:
    st = _REF_STATE
    parents = st["parents"]
    return _oracle_expand(parents[i % len(parents)], st["odb"], st["f"], set(),
                          time.perf_counter() + st["sample_s"])[1]


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    import multiprocessing as mp

    from oracle import enerflow_oracle as orc

    workload = args.workload
    ppg = args.parents or WORKLOADS[workload][2]
    n = ppg * max(world, args.gpus)
    fx = load_fixture(workload, n)
    if fx is not None:
        parents, og, odb, f = oracle_frontier(workload, fx["paths"][:n])
        source = f"the {n} frontier parents of our arm, rebuilt from {fx['file']}"
    else:  # no recorded frontier: the origin and its level-1 rewrites
        parents, og, odb, f = oracle_frontier(workload, [[]])
        parents = (parents + orc.neighbors(og, RULES))[:n]
        source = f"the origin and its first rewrites ({len(parents)} graphs; no recorded frontier)"
    nodes = sum(len(p["nodes"]) for p in parents) / len(parents)
    cores = os.cpu_count() or 1
    _REF_STATE.update(parents=parents, odb=odb, f=f, sample_s=args.ref_sample_s)
    ctx = mp.get_context("fork")  # workers inherit the graphs (weights are not pickled)
    times, priced = [], []
    with ctx.Pool(cores) as pool:
        nxt = 0
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            got = pool.map(_ref_worker, range(nxt, nxt + cores), chunksize=1)
            dt = time.perf_counter() - t0
            nxt += cores
            if i >= args.warmup:
                times.append(dt)
                priced.append(sum(got))
    value = sum(priced) / sum(times)
    sample = (f"each step: {cores} processes, each expanding one of {source} for at most {args.ref_sample_s:g} s "
              f"(rules x sites, hash, dedup, inner search d=1); {sum(priced)} candidates priced over {args.steps} "
              f"steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64",
            "data": "synthetic (random-init float64 weights, synthetic profiler seed 0)",
            "config": bench_config(workload, ppg, nodes),
            "frontier": {"source": fx["file"] if fx else None, "parents": len(parents)},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _cpu_sample(parents, odb, f, budget_s: float) -> dict:
    t0 = time.perf_counter()
    priced = expanded = 0
    visited: set = set()
    for p in parents:
        priced += _oracle_expand(p, odb, f, visited, t0 + budget_s)[1]
        expanded += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": priced / dt, "priced": priced, "expanded": expanded, "seconds": dt}


# the searches of BASELINE configs[0-3] end to end, with the golden each must reproduce
SEARCHES = [
    ("squeezenet", "energy", 1.0, None, None),
    ("resnet50", "energy", 1.05, 3000, "golden_search_resnet50_energy_a1.05_x3000.json"),
    ("inception_v3", "linear0.5", 1.05, 1000, "golden_search_inception_v3_linear0.5_a1.05_x1000.json"),
    ("nasnet_a", "energy", 1.05, 1000, "golden_search_nasnet_a_energy_a1.05_x1000.json"),
]


def _search_e2e(ef, zoo, no_cpu: bool) -> dict:
    """End-to-end searches through the public API (outer_search: tables, profiling, every
    expansion on the GPU), cold (first search of the model in this process: signatures, weight
    sets and their digests built) and warm (a fresh cost database, the device tables kept).
    configs[1-3] at alpha = 1.05 do not drain their queues in practical time, so they run to the
    expansion count of their golden (the reference's state at that point; tests/golden): the
    result is compared with it, and the oracle's recorded seconds for the same search are given.
    configs[0] runs to completion; the oracle port is timed live on one core."""
    import json as _json

    from oracle import enerflow_oracle as orc

    out = {}
    for model, obj, alpha, max_exp, golden in SEARCHES:
        g = zoo.generate(model, 0)
        times = []
        for _ in range(2):
            db = ef.CostDatabase()
            t0 = time.perf_counter()
            ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
            f = _objective(ef, obj, g, db)
            res = ef.outer_search(g, ef.default_rules(), db, f, ef.SearchConfig(alpha=alpha, max_expansions=max_exp),
                                  ef.SyntheticProfiler(0))
            times.append(time.perf_counter() - t0)
        row = {"alpha": alpha, "objective": obj, "max_expansions": max_exp, "gpu_s": times[0], "gpu_warm_s": times[1],
               "expansions": res.stats.graphs_explored, "generated": res.stats.graphs_generated,
               "ms_per_expansion_warm": 1e3 * times[1] / max(1, res.stats.graphs_explored),
               "optimised_hash": str(ef.canonical_hash(res.graph)), "cost": res.cost}
        if golden:
            try:
                with open(os.path.join(ROOT, "tests", "golden", golden)) as fh:
                    gd = _json.load(fh)
                row["same_result_as_golden"] = gd["hash"] == row["optimised_hash"] and gd["cost"] == res.cost
                row["oracle_s_recorded"] = gd.get("oracle_seconds")
                row["oracle_workers_recorded"] = gd.get("workers")
            except OSError:
                row["same_result_as_golden"] = None
        elif not no_cpu:
            t0 = time.perf_counter()
            ores = orc.outer_search(_to_oracle(g), RULES, orc.CostDB(), orc.CostFn("energy"), alpha=alpha, seed=0)
            row["oracle_cpu_s"] = time.perf_counter() - t0
            row["same_result"] = str(ores["hash"]) == row["optimised_hash"] and ores["cost"] == res.cost
            row["reference_s_build_container"] = 28.5
        out[model] = row
    return out


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------

def measure(args, workload: str, ppg: int, world: int, rank: int, local: int, ex, dist, cpu_budget: float,
            extras: bool) -> tuple[dict, list]:
    """One workload's bench line (without the job-level keys).  -> (line, this rank's parents
    as oracle graphs when the CPU baseline is wanted)."""
    import ctypes as C

    import numpy as np
    import torch

    import paper_2005_05837_b200 as ef
    from paper_2005_05837_b200 import _native as N
    from paper_2005_05837_b200 import zoo
    from paper_2005_05837_b200.frontier import Frontier
    from paper_2005_05837_b200.shard import sharded_expand

    dev = torch.device("cuda", local)
    config_name, objective, _ = WORKLOADS[workload]
    g0 = zoo.generate(workload, 0)
    db = ef.CostDatabase()
    ef.ensure_profiled(g0, db, ef.SyntheticProfiler(0))
    fr = Frontier(g0, db, ef.SyntheticProfiler(0), _objective(ef, objective, g0, db),
                  ef.SearchConfig(alpha=workload_alpha(workload)), ppg * world)
    # weak scaling: this rank owns its slice of the frontier (graphs are independent objects)
    mine = fr.slots[rank * ppg:(rank + 1) * ppg]
    s = fr.s
    fx = load_fixture(workload, ppg * world)
    frontier = {"source": None, "parents": len(fr.slots)}
    if fx is not None:
        got = [str(h) for h in s.hash_slots(fr.slots)]
        frontier = {"source": fx["file"], "parents": len(fr.slots),
                    "same_as_recorded": got == fx["hashes"][:len(got)] and [list(p) for p in fr.paths] ==
                    fx["paths"][:len(got)]}

    def barrier():
        if dist is not None:
            dist.barrier()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    def flush_l2():
        flush.fill_(1)
        torch.cuda.synchronize()

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases: dict = {}  # host seconds per sharded-step phase

    def step(slots):
        """-> (results, device ms of the step)."""
        if ex is None:
            res = fr.step(slots, insert_visited=False)
        else:
            res = sharded_expand(s, slots, fr.rule_ids, fr.pp, ex, phases=phases)
        # the library's events span match .. price (a sharded step: the exchange and its host
        # round trips included), excluding the results copy
        return res, s.last_step_ms()

    for _ in range(args.warmup):
        step(mine)
    prof = os.environ.get("EF_NCU") == "1"  # ncu --profile-from-start off: capture the timed steps only
    if prof:
        torch.cuda.profiler.start()
    clocks = Clocks()
    clocks.start()
    dev_ms, stage_ms, priced_n, gen_n, kcomp, dcomp, launches = [], [0.0] * 8, 0, 0, 0, 0, 0
    for _ in range(args.steps):
        flush_l2()
        barrier()
        res, ms = step(mine)
        dev_ms.append(ms)
        stage_ms = [a + b for a, b in zip(stage_ms, s.last_timing())]
        st = s.last_stats()
        kcomp += st["key_compressions"]
        dcomp += st["digest_compressions"]
        launches += st["kernels"]
        priced_n += int(np.count_nonzero(res["flags"] & N.F_PRICED))
        gen_n += len(res)
    clk = clocks.stop(local)
    if prof:
        torch.cuda.profiler.stop()
        fr.close()
        return {"ncu_capture": True, "stages_ms": stage_ms}, []
    total_ms = sum(dev_ms)
    priced_all = float(priced_n)
    if ex is not None:
        total_ms = -ex.min(-total_ms)  # max over ranks
        priced_all = ex.sum(float(priced_n))
    value = priced_all / (total_ms / 1e3)

    # e2e through the C ABI from host memory: compact parents H2D + unpack + hash, step, results D2H
    host_recs = [s.read_record(sl) for sl in mine]
    blob, offs = s.pack(host_recs)
    pinned = s.L.ef_host_alloc(blob.nbytes)
    staging = np.ctypeslib.as_array((C.c_uint8 * blob.nbytes).from_address(pinned))
    staging[:] = blob.view(np.uint8)
    # (a) serial: upload + hash, then the step, then the results, one step at a time
    e2e_slots = [s.alloc() for _ in mine]
    ser_ms, up_ms = [], 0.0
    evm = torch.cuda.Event(enable_timing=True)
    for i in range(args.warmup + args.steps):
        flush_l2()
        barrier()
        ev0.record()
        s.write_packed(e2e_slots, staging.view(np.uint32), offs)
        evm.record()
        res, _ = step(e2e_slots)
        ev1.record()
        ev1.synchronize()
        if i >= args.warmup:
            ser_ms.append(ev0.elapsed_time(ev1))
            up_ms += ev0.elapsed_time(evm)
    # (b) pipelined (the headline): the next batch's upload + hash run on the upload stream
    # while this batch's step runs; every batch's H2D and results D2H are inside the region
    sets = [e2e_slots, [s.alloc() for _ in mine]]
    e2e_total = 0.0
    e2e_priced = n_cand = 0

    def priced_in(r):
        return int(np.count_nonzero(r["flags"] & N.F_PRICED))

    for rep in range(2):  # rep 0 warms up
        barrier()
        ev0.record()
        s.write_packed(sets[0], staging.view(np.uint32), offs, asynchronous=True)
        s.upload_fence()
        priced_rep, pending = 0, None
        for i in range(args.steps):
            if i + 1 < args.steps:
                s.write_packed(sets[(i + 1) % 2], staging.view(np.uint32), offs, asynchronous=True)
            if ex is None:  # results of step i copied to the host while step i + 1 runs
                n_cand = s.expand(sets[i % 2], fr.rule_ids, fr.pp, False, results=False)
                if pending is not None:
                    s.results_wait()
                    priced_rep += priced_in(pending)
                pending = s.results_async(n_cand)
            else:
                res, _ = step(sets[i % 2])
                priced_rep += priced_in(res)
                n_cand = len(res)
            s.upload_fence()
        if pending is not None:
            s.results_wait()
            priced_rep += priced_in(pending)
        ev1.record()
        ev1.synchronize()
        if rep == 1:
            e2e_total, e2e_priced = ev0.elapsed_time(ev1), priced_rep
    del staging
    s.L.ef_host_free(pinned)
    for sl in sets[0] + sets[1]:
        s.free(sl)
    e2e_all = float(e2e_priced)
    ser_total, ser_priced = sum(ser_ms), float(priced_n)
    if ex is not None:
        e2e_total = -ex.min(-e2e_total)
        e2e_all = ex.sum(e2e_all)
        ser_total = -ex.min(-ser_total)
        ser_priced = ex.sum(ser_priced)
    e2e_value = e2e_all / (e2e_total / 1e3)

    # rooflines of the dominant kernel (node keys), from the live per-stage CUDA-event times
    names = list(s.STAGES)
    keys_ms = stage_ms[names.index("keys")] / args.steps
    peak_c = s.b2b_peak()
    achieved_c = kcomp / args.steps / (keys_ms / 1e3)
    hbm_peak, hbm_src = _peaks()
    n_nodes = float(np.mean([int(b[:4].view(np.int32)[0]) for b in host_recs]))
    # algorithmic bytes of the node-key kernel per job: the 16-byte job, ~1.1 producer keys
    # (16 B) with their refsrc words (4 B) read; the 16-byte key and its 12-byte sort record written
    jobs = kcomp / args.steps
    keys_bytes = jobs * (16 + 1.1 * (16 + 4) + 16 + 12)
    kname = "k_keys_wide" if n_nodes > 256 else "k_keys<"
    keys_traffic, traffic_src = _traffic(kname)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u64",
        "data": "synthetic (random-init float64 weights, synthetic profiler seed 0)",
        "config": bench_config(workload, len(mine), n_nodes),
        "l2": "flushed (256 MiB write) before every timed step",
        "parallelism": ("frontier split by parent, dedup owned by hash (NCCL all-to-all)" if ex is not None
                        else "single GPU"),
        "frontier": frontier,
        "per_step": {"candidates": gen_n / args.steps, "priced": priced_n / args.steps},
        "stages_ms_per_step": {n: stage_ms[k] / args.steps for k, n in enumerate(names)},
        "roofline": {"bound": "alu", "kernel": "node keys (k_keys / k_keys_wide)", "achieved": achieved_c / 1e9,
                     "peak": peak_c / 1e9, "unit": "Gcompressions/s", "frac": achieved_c / peak_c,
                     "traffic": keys_traffic, "traffic_unit": "bytes per launch (dram read + write)",
                     "traffic_source": traffic_src, "traffic_kernel": kname.rstrip("<"),
                     "peak_source": "measured live: ef_b2b_peak (register-only BLAKE2b loop, same GPU)",
                     "compressions_per_step": kcomp / args.steps,
                     "digest_compressions_per_step": dcomp / args.steps},
        "roofline_hbm": {"bound": "hbm", "kernel": "node keys", "achieved": keys_bytes / (keys_ms / 1e3) / 1e9,
                         "peak": hbm_peak, "unit": "GB/s", "frac": keys_bytes / (keys_ms / 1e3) / 1e9 / hbm_peak,
                         "peak_source": hbm_src, "algorithmic_bytes": keys_bytes},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(blob.nbytes),
                "d2h_bytes_per_step": n_cand * N.CAND_DTYPE.itemsize, "ms_per_step": e2e_total / args.steps,
                "mode": "pipelined: batch i+1 uploaded and hashed on the upload stream during step i, the results "
                        "of step i copied to the host during step i+1",
                "serial_value": ser_priced / (ser_total / 1e3), "serial_ms_per_step": ser_total / args.steps,
                "serial_upload_hash_ms_per_step": up_ms / args.steps},
        "gpu_launches": launches,
        "clocks": clk,
    }
    cpu_parents = []
    if extras and not args.no_cpu:
        cpu_parents = [_to_oracle(fr.decode(sl)) for sl in mine[:8]]
    fr.close()  # frees the frontier's records (the next workload sets its own geometry)
    return line, cpu_parents


def run_ours(args, world, rank, local):
    import torch

    import paper_2005_05837_b200 as ef
    from paper_2005_05837_b200 import zoo

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = ex = None
    if world > 1 or args.sharded:
        import torch.distributed as dist

        from paper_2005_05837_b200.shard import OwnerExchange

        dist.init_process_group("nccl", device_id=dev)
        ex = OwnerExchange(device=dev)
    workload = args.workload
    ppg = args.parents or WORKLOADS[workload][2]
    extras = rank == 0 and world == 1 and not os.environ.get("EF_NCU")
    line, cpu_parents = measure(args, workload, ppg, world, rank, local, ex, dist, args.cpu_budget, extras)
    if line.get("ncu_capture"):
        if rank == 0:
            print(json.dumps(line))
        return 0
    if extras and not args.no_extras:
        others = {}
        for w in ([] if workload == "resnet50" else ["resnet50"]):
            wl, _ = measure(args, w, WORKLOADS[w][2], world, rank, local, ex, dist, 0, False)
            others[w] = {k: wl[k] for k in ("value", "ms_per_step", "config", "per_step", "stages_ms_per_step",
                                            "roofline", "e2e", "gpu_launches", "frontier")}
        line["workloads"] = others
        # the searches run as in a fresh process: the frontier steps' session (hashing scratch
        # sized to most of the HBM for DAG-20k) is released first -- with it resident, the small
        # searches' launches run 4-5x slower (SqueezeNet 0.05 -> 0.23 s warm)
        from paper_2005_05837_b200.device import DeviceSession

        DeviceSession.reset_default()
        line["search"] = _search_e2e(ef, zoo, args.no_cpu)
    if extras and not args.no_cpu and cpu_parents:
        fx = load_fixture(workload, ppg)
        _, _, odb, f = oracle_frontier(workload, [[]])
        cpu = _cpu_sample(cpu_parents, odb, f, args.cpu_budget)
        line["cpu_baseline"] = {"value": cpu["value"], "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{cpu['expanded']} {workload} frontier expansions (the last may be "
                                          f"partial; {cpu['priced']} candidates priced) by the oracle restatement on "
                                          f"one core, {cpu['seconds']:.1f}s" +
                                          (f" (parents recorded in {fx['file']})" if fx else "")}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _self_launch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: one rank per GPU through torch.distributed.run
    (the driver's own launch line), rendezvous on 127.0.0.1."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--parents", type=int, default=0, help="frontier graphs per GPU per step (0: workload default)")
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS),
                    help="BASELINE.json config to run as the frontier workload (default: configs[4], DAG-20k)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="only the headline workload (no ResNet-50 line, no searches)")
    ap.add_argument("--ref-sample-s", type=float, default=3.0,
                    help="reference arm: seconds of oracle work per process per step")
    ap.add_argument("--sharded", action="store_true", help="use the hash-owner sharded step even on one rank")
    args = ap.parse_args()
    if (args.gpus > 1 or args.sharded) and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus)
    world, rank, local = _dist()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
