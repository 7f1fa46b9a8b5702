"""ORACLE — TEST INFRASTRUCTURE ONLY.  Never imported by the product package.

CPU restatement of the reference's frontier-expansion-and-pricing path
(arxiv/paper_2005_05837, reference package `enerflow`, /root/reference/pkg).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker / the timed CPU
baseline — the product path (paper_2005_05837_b200) runs on the GPU and fails
loudly without its CUDA extension.

Pinned against the real reference: tests/golden/make_golden.py imports the
reference package in the build container and records canonical hashes,
neighbour sequences, inner-search results and full outer-search traces
(explored-hash sequence, best graph, assignment, costs, stats) into
tests/golden/*.json; tests/test_oracle_golden.py checks this module against
every one of them.

Representation: a graph is a plain dict
    {"inputs": [(name, dims)], "nodes": {id: N}, "outputs": [(id, port)]}
with N = {"kind", "ins": [(id, port)], "p": params dict, "w": {name: ndarray}}.
Weights are shared (never copied) between a graph and its rewrites, exactly
as the reference shares numpy arrays, so weight digests are memoised per
array-set identity; that changes cost, not results.

Each function cites the reference lines it restates.
"""

from __future__ import annotations

import base64
import hashlib
import heapq
import itertools
import json
import math

import numpy as np

# ---------------------------------------------------------------------------
# graph loading (graph.py:824-860, the on-disk schema)
# ---------------------------------------------------------------------------

TUPLE_PARAMS = {"kernel", "stride", "padding", "sizes", "shape"}


def _ref(obj):
    return (obj, 0) if isinstance(obj, int) else (obj[0], obj[1])


def from_json(doc: dict) -> dict:
    nodes = {}
    for item in doc["nodes"]:
        params = {k: (tuple(int(x) for x in v) if k in TUPLE_PARAMS and isinstance(v, list) else v)
                  for k, v in item.get("params", {}).items()}
        w = {}
        for key, val in item.get("weights", {}).items():
            if isinstance(val, dict):
                w[key] = np.frombuffer(base64.b64decode(val["b64"]), dtype=np.float64).reshape(val["shape"]).copy()
            else:
                w[key] = np.asarray(val, dtype=np.float64)
        nodes[item["id"]] = {"kind": item["kind"], "ins": [_ref(r) for r in item.get("inputs", [])],
                             "p": params, "w": w}
    return {"inputs": [(e["name"], tuple(e["shape"])) for e in doc["inputs"]],
            "nodes": nodes, "outputs": [_ref(r) for r in doc["outputs"]]}


def load_json(path: str) -> dict:
    with open(path) as fh:
        return from_json(json.load(fh))


# ---------------------------------------------------------------------------
# shapes and signatures (graph.py:181-311 shapes, 419-498 signature text)
# ---------------------------------------------------------------------------

def topo(g) -> list[int]:
    """graph.py:147-173 — Kahn with smallest ready id first."""
    indeg = {n: len(v["ins"]) for n, v in g["nodes"].items()}
    succ = {n: [] for n in g["nodes"]}
    for n, v in g["nodes"].items():
        for (p, _) in v["ins"]:
            succ[p].append(n)
    ready = sorted(n for n, d in indeg.items() if d == 0)
    out = []
    while ready:
        n = heapq.heappop(ready)
        out.append(n)
        for s in succ[n]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(ready, s)
    assert len(out) == len(g["nodes"]), "cycle"
    return out


def _win(dims, p):
    kh, kw = p["kernel"]
    sh, sw = p["stride"]
    ph, pw = p["padding"]
    return (dims[2] + 2 * ph - kh) // sh + 1, (dims[3] + 2 * pw - kw) // sw + 1


def out_shapes(g) -> dict[int, list[tuple]]:
    """graph.py:181-292 restated for valid graphs."""
    decl = dict(g["inputs"])
    res = {}
    for n in topo(g):
        v = g["nodes"][n]
        ins = [res[p][port] for (p, port) in v["ins"]]
        k, p = v["kind"], v["p"]
        if k == "input":
            res[n] = [tuple(decl[p["name"]])]
        elif k == "conv2d":
            oh, ow = _win(ins[0], p)
            res[n] = [(ins[0][0], p["out_channels"], oh, ow)]
        elif k == "matmul":
            res[n] = [(ins[0][0], p["out_features"])]
        elif k == "concat":
            d = list(ins[0])
            d[p["axis"]] = sum(s[p["axis"]] for s in ins)
            res[n] = [tuple(d)]
        elif k == "split":
            parts = []
            for sz in p["sizes"]:
                d = list(ins[0])
                d[p["axis"]] = int(sz)
                parts.append(tuple(d))
            res[n] = parts
        elif k in ("maxpool", "avgpool"):
            oh, ow = _win(ins[0], p)
            res[n] = [(ins[0][0], ins[0][1], oh, ow)]
        else:
            res[n] = [ins[0]]
    return res


SIG_KEYS = {"conv2d": ("has_activation", "kernel", "out_channels", "padding", "stride"),
            "matmul": ("out_features",), "concat": ("axis",), "split": ("axis", "sizes"),
            "maxpool": ("kernel", "padding", "stride"), "avgpool": ("kernel", "padding", "stride")}


def _render(v):
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (tuple, list)):
        return "x".join(str(int(x)) for x in v)
    return str(v)


def sig_texts(g) -> dict[int, str]:
    """graph.py:441-448 + 480-498: kind|in=..|key=value..."""
    shapes = out_shapes(g)
    decl = dict(g["inputs"])
    out = {}
    for n in sorted(g["nodes"]):
        v = g["nodes"][n]
        if v["kind"] == "input":
            out[n] = "input|shape=" + "x".join(map(str, decl[v["p"]["name"]]))
            continue
        parts = [v["kind"]]
        if v["ins"]:
            parts.append("in=" + ",".join("x".join(map(str, shapes[p][port])) for (p, port) in v["ins"]))
        parts += [f"{key}={_render(v['p'][key])}" for key in SIG_KEYS.get(v["kind"], ())]
        out[n] = "|".join(parts)
    return out


def sig_fields(g, n, shapes=None) -> dict:
    """Structured signature (kind, input shapes, params) — what the profiler consumes."""
    shapes = shapes or out_shapes(g)
    v = g["nodes"][n]
    return {"kind": v["kind"], "ins": [shapes[p][port] for (p, port) in v["ins"]],
            "p": {k: v["p"][k] for k in SIG_KEYS.get(v["kind"], ())}}


# ---------------------------------------------------------------------------
# canonical hash (graph.py:510-549)
# ---------------------------------------------------------------------------

_WDIGEST: dict = {}


def weight_digest(w: dict) -> bytes:
    """graph.py:510-517: blake2b-128 over (key, str(shape), float64 bytes) per sorted key."""
    ident = tuple((k, id(w[k])) for k in sorted(w))
    hit = _WDIGEST.get(ident)
    if hit is not None and all(a is b for a, b in zip(hit[1], (w[k] for k in sorted(w)))):
        return hit[0]
    h = hashlib.blake2b(digest_size=16)
    for key in sorted(w):
        arr = np.ascontiguousarray(w[key], dtype=np.float64)
        h.update(key.encode())
        h.update(str(arr.shape).encode())
        h.update(arr.tobytes())
    d = h.digest()
    _WDIGEST[ident] = (d, tuple(w[k] for k in sorted(w)))
    return d


def node_keys(g, sigs=None) -> dict[int, bytes]:
    """graph.py:528-540: Merkle key per node from sig text, input name, weights, producer keys."""
    sigs = sigs or sig_texts(g)
    keys = {}
    for n in topo(g):
        v = g["nodes"][n]
        h = hashlib.blake2b(digest_size=16)
        h.update(sigs[n].encode())
        if v["kind"] == "input":
            h.update(v["p"]["name"].encode())
        h.update(weight_digest(v["w"]))
        for (p, port) in v["ins"]:
            h.update(keys[p])
            h.update(port.to_bytes(2, "big"))
        keys[n] = h.digest()
    return keys


def canonical_hash(g) -> int:
    """graph.py:520-549."""
    keys = node_keys(g)
    top = hashlib.blake2b(digest_size=8)
    for name, dims in g["inputs"]:
        top.update(f"{name}={'x'.join(map(str, dims))};".encode())
    for (n, port) in g["outputs"]:
        top.update(keys[n])
        top.update(port.to_bytes(2, "big"))
    for k in sorted(keys.values()):
        top.update(k)
    return int.from_bytes(top.digest(), "big")


# ---------------------------------------------------------------------------
# rules (rules.py:96-353)
# ---------------------------------------------------------------------------

RULE_NAMES = ["fuse-conv-relu", "split-conv-activation", "merge-parallel-convs",
              "split-merged-conv", "fold-identity", "fuse-conv-batchnorm"]


# pattern-node names per rule, in the tuple order `match` returns (rules.py MatchSite.of calls)
SITE_NAMES = {"fuse-conv-relu": ("conv", "relu"), "split-conv-activation": ("conv",),
              "merge-parallel-convs": ("left", "right"), "split-merged-conv": ("conv", "split"),
              "fold-identity": ("identity",), "fuse-conv-batchnorm": ("conv", "bn")}


def binding(rule: str, site: tuple) -> list[int]:
    """Site ids in the reference's MatchSite.binding order (sorted by pattern name)."""
    return [v for _, v in sorted(zip(SITE_NAMES[rule], site))]


def _uses(g) -> dict:
    """rules.py:138-144 consumers(): edge -> [(consumer id, slot)] in id order."""
    u = {}
    for n in sorted(g["nodes"]):
        for i, r in enumerate(g["nodes"][n]["ins"]):
            u.setdefault(r, []).append((n, i))
    return u


def _sole(g, uses, ref):
    """rules.py:134-140."""
    lst = uses.get(ref, [])
    if len(lst) != 1 or ref in g["outputs"]:
        return None
    return lst[0][0]


def match(rule: str, g) -> list[tuple]:
    """All sites in the reference's order (rules.py:147-331 matchers)."""
    N = g["nodes"]
    ids = sorted(N)
    if rule == "fuse-conv-relu":                                   # rules.py:147-161
        u = _uses(g)
        out = []
        for n in ids:
            if N[n]["kind"] != "relu":
                continue
            src = N[n]["ins"][0]
            pv = N[src[0]]
            if pv["kind"] == "conv2d" and not pv["p"]["has_activation"] and _sole(g, u, src) == n:
                out.append((src[0], n))
        return out
    if rule == "split-conv-activation":                            # rules.py:173-178
        return [(n,) for n in ids if N[n]["kind"] == "conv2d" and N[n]["p"]["has_activation"]]
    if rule == "merge-parallel-convs":                             # rules.py:200-215
        groups = {}
        for n in ids:
            if N[n]["kind"] == "conv2d":
                groups.setdefault(N[n]["ins"][0], []).append(n)
        out = []
        for src in sorted(groups):
            grp = groups[src]
            for i, a in enumerate(grp):
                for b in grp[i + 1:]:
                    if all(N[a]["p"][k] == N[b]["p"][k] for k in ("kernel", "stride", "padding", "has_activation")):
                        out.append((a, b))
        return sorted(out)
    if rule == "split-merged-conv":                                # rules.py:245-261
        u = _uses(g)
        out = []
        for n in ids:
            v = N[n]
            if v["kind"] != "split" or v["p"]["axis"] != 1 or len(v["p"]["sizes"]) != 2:
                continue
            src = v["ins"][0]
            if N[src[0]]["kind"] == "conv2d" and _sole(g, u, src) == n:
                out.append((src[0], n))
        return out
    if rule == "fold-identity":                                    # rules.py:288-290
        return [(n,) for n in ids if N[n]["kind"] == "identity"]
    if rule == "fuse-conv-batchnorm":                              # rules.py:303-318
        u = _uses(g)
        out = []
        for n in ids:
            if N[n]["kind"] != "batchnorm":
                continue
            src = N[n]["ins"][0]
            pv = N[src[0]]
            if pv["kind"] == "conv2d" and not pv["p"]["has_activation"] and _sole(g, u, src) == n:
                out.append((src[0], n))
        return out
    raise KeyError(rule)


def _rebuild(g, drop, new, remap):
    """rules.py:100-126: drop, add, remap old nodes' edges and outputs, prune unreachable."""
    nodes = {}
    for n, v in g["nodes"].items():
        if n in drop:
            continue
        nodes[n] = dict(v, ins=[remap.get(r, r) for r in v["ins"]])
    for n, v in new:
        nodes[n] = v
    outputs = [remap.get(r, r) for r in g["outputs"]]
    live = set()
    todo = [r[0] for r in outputs]
    while todo:
        n = todo.pop()
        if n not in live:
            live.add(n)
            todo.extend(r[0] for r in nodes[n]["ins"])
    return {"inputs": g["inputs"], "nodes": {n: v for n, v in nodes.items() if n in live}, "outputs": outputs}


def _bias(v):
    """rules.py:218-222."""
    b = v["w"].get("bias")
    return np.zeros(v["p"]["out_channels"], dtype=np.float64) if b is None else b


def apply(rule: str, g, site: tuple):
    """rules.py:164-331 rewriters."""
    N = g["nodes"]
    fresh = max(N) + 1
    if rule == "fuse-conv-relu":                                   # rules.py:164-170
        c, r = site
        v = N[c]
        return _rebuild(g, {c, r}, [(c, dict(v, p={**v["p"], "has_activation": True}))], {(r, 0): (c, 0)})
    if rule == "split-conv-activation":                            # rules.py:181-190
        (c,) = site
        v = N[c]
        bare = dict(v, p={**v["p"], "has_activation": False})
        relu = {"kind": "relu", "ins": [(c, 0)], "p": {}, "w": {}}
        return _rebuild(g, {c}, [(c, bare), (fresh, relu)], {(c, 0): (fresh, 0)})
    if rule == "merge-parallel-convs":                             # rules.py:225-242
        a, b = site
        va, vb = N[a], N[b]
        oa, ob = va["p"]["out_channels"], vb["p"]["out_channels"]
        merged = {"kind": "conv2d", "ins": list(va["ins"]), "p": {**va["p"], "out_channels": oa + ob},
                  "w": {"weight": np.concatenate([va["w"]["weight"], vb["w"]["weight"]], axis=0),
                        "bias": np.concatenate([_bias(va), _bias(vb)])}}
        split = {"kind": "split", "ins": [(fresh, 0)], "p": {"axis": 1, "sizes": (oa, ob)}, "w": {}}
        return _rebuild(g, {a, b}, [(fresh, merged), (fresh + 1, split)],
                        {(a, 0): (fresh + 1, 0), (b, 0): (fresh + 1, 1)})
    if rule == "split-merged-conv":                                # rules.py:264-281
        c, s = site
        v = N[c]
        s0, s1 = N[s]["p"]["sizes"]
        w, b = v["w"]["weight"], _bias(v)
        left = {"kind": "conv2d", "ins": list(v["ins"]), "p": {**v["p"], "out_channels": int(s0)},
                "w": {"weight": w[:s0].copy(), "bias": b[:s0].copy()}}
        right = {"kind": "conv2d", "ins": list(v["ins"]), "p": {**v["p"], "out_channels": int(s1)},
                 "w": {"weight": w[s0:].copy(), "bias": b[s0:].copy()}}
        return _rebuild(g, {c, s}, [(fresh, left), (fresh + 1, right)],
                        {(s, 0): (fresh, 0), (s, 1): (fresh + 1, 0)})
    if rule == "fold-identity":                                    # rules.py:293-296
        (i,) = site
        return _rebuild(g, {i}, [], {(i, 0): N[i]["ins"][0]})
    if rule == "fuse-conv-batchnorm":                              # rules.py:321-331
        c, n = site
        v = N[c]
        scale, shift = N[n]["w"]["scale"], N[n]["w"]["shift"]
        fused = dict(v, w={"weight": v["w"]["weight"] * scale[:, None, None, None],
                           "bias": _bias(v) * scale + shift})
        return _rebuild(g, {c, n}, [(c, fused)], {(n, 0): (c, 0)})
    raise KeyError(rule)


def neighbors(g, rules: list[str]) -> list[dict]:
    """rules.py:73-89: rule order, site order, first graph per hash wins."""
    seen = set()
    out = []
    for rule in rules:
        for site in match(rule, g):
            cand = apply(rule, g, site)
            h = canonical_hash(cand)
            if h in seen:
                continue
            seen.add(h)
            out.append(cand)
    return out


# ---------------------------------------------------------------------------
# synthetic profiler (profiling.py:30-149)
# ---------------------------------------------------------------------------

ALG_COUNTS = {"conv2d": 4, "matmul": 3, "maxpool": 2, "avgpool": 2, "relu": 2, "add": 2,
              "batchnorm": 2, "concat": 2, "split": 1, "identity": 1}


def _unit(seed, *parts) -> float:
    """profiling.py:103-108."""
    key = (seed % 2**64).to_bytes(8, "little")
    d = hashlib.blake2b("|".join(str(p) for p in parts).encode(), key=key, digest_size=8).digest()
    return int.from_bytes(d, "big") / 2.0**64


def _flops(f) -> float:
    """profiling.py:72-93."""
    k = f["kind"]
    if k == "input":
        return 0.0
    if k == "conv2d":
        s = f["ins"][0]
        oh, ow = _win(s, f["p"])
        kh, kw = f["p"]["kernel"]
        return 2.0 * s[0] * f["p"]["out_channels"] * oh * ow * s[1] * kh * kw
    if k == "matmul":
        b, feat = f["ins"][0]
        return 2.0 * b * feat * f["p"]["out_features"]
    if k in ("maxpool", "avgpool"):
        s = f["ins"][0]
        oh, ow = _win(s, f["p"])
        kh, kw = f["p"]["kernel"]
        return float(s[0] * s[1] * oh * ow * kh * kw)
    return float(sum(math.prod(s) for s in f["ins"]))


def synthetic_rows(f, text: str, seed: int) -> list[tuple[int, float, float]]:
    """profiling.py:123-149 for every applicable alg: [(alg, time_ms, power_w)]."""
    cands = list(range(ALG_COUNTS.get(f["kind"], 1)))
    draws = {a: _unit(seed, text, a, "applicable") for a in cands}
    app = [a for a in cands if draws[a] >= 0.2] or [max(cands, key=lambda a: draws[a])]
    rows = []
    for a in app:
        mult = 0.7 + (1.6 - 0.7) * _unit(seed, f["kind"], a, "mult")
        jit = 0.8 + (1.25 - 0.8) * _unit(seed, text, a, "jitter")
        over = 0.001 + (0.01 - 0.001) * _unit(seed, f["kind"], a, "overhead")
        t = 1e-6 * _flops(f) ** 0.9 * mult * jit + over
        speed = min(1.0, max(0.0, (1.6 * 1.25 - mult * jit) / (1.6 * 1.25 - 0.7 * 0.8)))
        frac = 0.55 * speed + 0.45 * _unit(seed, text, a, "power")
        rows.append((a, t, 40.0 + (200.0 - 40.0) * frac))
    return rows


class CostDB:
    """cost.py:53-96 — sig text -> {alg: (time_ms, power_w)}."""

    def __init__(self):
        self.rows: dict[str, dict[int, tuple[float, float]]] = {}

    def add(self, sig, alg, t, p):
        self.rows.setdefault(sig, {})[int(alg)] = (float(t), float(p))

    def table(self, sig):
        """[(alg, time, energy)] ascending; energy = time*power (cost.py:47-50)."""
        r = self.rows.get(sig, {})
        return [(a, r[a][0], r[a][0] * r[a][1]) for a in sorted(r)]

    @classmethod
    def load_jsonl(cls, path):
        db = cls()
        with open(path) as fh:
            for line in fh:
                if line.strip():
                    o = json.loads(line)
                    db.add(o["sig"], o["alg"], o["time_ms"], o["power_w"])
        return db


def ensure_profiled(g, db: CostDB, seed: int) -> int:
    """profiling.py:211-252 with the synthetic profiler; returns #new records."""
    texts = sig_texts(g)
    shapes = None
    made = 0
    done = set()
    for n in sorted(g["nodes"]):
        if g["nodes"][n]["kind"] == "input" or texts[n] in done:
            continue
        done.add(texts[n])
        if texts[n] in db.rows:
            continue
        shapes = shapes or out_shapes(g)
        for a, t, p in synthetic_rows(sig_fields(g, n, shapes), texts[n], seed):
            db.add(texts[n], a, t, p)
            made += 1
    return made


# ---------------------------------------------------------------------------
# cost function (cost.py:175-254) and inner search (search.py:100-182)
# ---------------------------------------------------------------------------

class CostFn:
    def __init__(self, kind, w=0.5, mix=(0.0, 0.0, 0.0), refs=(1.0, 1.0, 1.0)):
        self.kind, self.w, self.mix = kind, float(w), tuple(float(x) for x in mix)
        self.t_ref, self.e_ref, self.p_ref = (float(x) for x in refs)

    def __call__(self, time_ms, energy):
        """cost.py:234-254, same operation order."""
        t = time_ms / self.t_ref
        e = energy / self.e_ref
        if self.kind == "time":
            return time_ms
        if self.kind == "energy":
            return energy
        if self.kind == "power":
            return energy / time_ms if np.any(time_ms) else time_ms * 0.0
        if self.kind == "linear":
            return self.w * e + (1.0 - self.w) * t
        if self.kind == "product":
            return e ** self.w * t ** (1.0 - self.w)
        ct, ce, cp = self.mix
        p = (energy / time_ms if np.any(time_ms) else time_ms * 0.0) / self.p_ref
        return ct * t + ce * e + cp * p


class MissingEntry(Exception):
    pass


def cost_table(g, db: CostDB):
    """cost.py:120-134: {compute node id: [(alg, t, e)]}."""
    texts = sig_texts(g)
    out = {}
    for n in sorted(g["nodes"]):
        if g["nodes"][n]["kind"] == "input":
            continue
        rows = db.table(texts[n])
        if not rows:
            raise MissingEntry(texts[n])
        out[n] = rows
    return out


def sweep(g, db: CostDB, f: CostFn, d: int):
    """search.py:106-153: returns (assign, cost, t, e, evals, sweeps)."""
    table = cost_table(g, db)
    nids = sorted(table)
    per = {n: {a: (t, e) for a, t, e in rows} for n, rows in table.items()}
    assign = {n: table[n][0][0] for n in nids}
    t_tot = sum(per[n][assign[n]][0] for n in nids)
    e_tot = sum(per[n][assign[n]][1] for n in nids)
    cost = f(t_tot, e_tot)
    evals = sweeps = 0
    if not nids:
        return assign, cost, t_tot, e_tot, evals, sweeps
    radius = min(d, len(nids))
    changed = True
    while changed:
        changed = False
        sweeps += 1
        for k in range(1, radius + 1):
            for combo in itertools.combinations(nids, k):
                alts = [[a for a in sorted(per[n]) if a != assign[n]] for n in combo]
                if any(not x for x in alts):
                    continue
                for choice in itertools.product(*alts):
                    dt = de = 0.0
                    for n, a in zip(combo, choice):
                        ct, ce = per[n][assign[n]]
                        nt, ne = per[n][a]
                        dt += nt - ct
                        de += ne - ce
                    cand = f(t_tot + dt, e_tot + de)
                    evals += 1
                    if cand < cost:
                        for n, a in zip(combo, choice):
                            assign[n] = a
                        t_tot += dt
                        e_tot += de
                        cost = cand
                        changed = True
    return assign, cost, t_tot, e_tot, evals, sweeps


def normalization_refs(g, db: CostDB):
    """cost.py:284-296: (T_ref, E_ref, P_ref) = per-metric optima = sums of per-node minima."""
    table = cost_table(g, db)
    if not table:
        raise ValueError("normalization references undefined for a graph with no compute nodes")
    t_ref = sum(min(t for _, t, _ in rows) for rows in table.values())
    e_ref = sum(min(e for _, _, e in rows) for rows in table.values())
    return t_ref, e_ref, e_ref / t_ref


def default_eval(g, db: CostDB, f: CostFn):
    """search.py:196-202 (use_inner=False): lowest alg per node."""
    table = cost_table(g, db)
    assign = {n: rows[0][0] for n, rows in table.items()}
    t = sum(rows[0][1] for rows in table.values())
    e = sum(rows[0][2] for rows in table.values())
    return assign, f(t, e), t, e, 1, 0


def neumaier_sum(xs) -> float:
    """CPython 3.12 builtin sum() over floats (Neumaier compensation) — the
    summation the reference's sum() calls perform; the CUDA pricing kernel
    restates this exact sequence (see tests/test_oracle_golden.py)."""
    it = iter(xs)
    try:
        f = 0 + next(it)
    except StopIteration:
        return 0
    c = 0.0
    for x in it:
        t = f + x
        if abs(f) >= abs(x):
            c += (f - t) + x
        else:
            c += (x - t) + f
        f = t
    if c and math.isfinite(c):
        f += c
    return f


# ---------------------------------------------------------------------------
# outer search (search.py:211-272)
# ---------------------------------------------------------------------------

STAT_KEYS = ("graphs_explored", "graphs_generated", "graphs_deduped", "expanded_at_best",
             "assignments_evaluated", "inner_sweeps", "best_updates", "queue_pruned",
             "queue_cap_hits", "node_cap_hits", "new_cost_records")


def n_compute(g) -> int:
    return sum(1 for v in g["nodes"].values() if v["kind"] != "input")


def outer_search(g0, rules, db: CostDB, f: CostFn, alpha=1.05, d=1, max_queue=100_000,
                 max_graph_nodes=None, seed=None, use_inner=True, max_expansions=None, trace=None):
    """search.py:211-272.  `seed` = synthetic profiler seed (None: no profiling).

    `trace`, when a list, receives the canonical hash of every expanded graph
    in order (the explored-hash sequence the GPU search must reproduce).
    `max_expansions` bounds the run for large instances (not in the reference;
    None reproduces it exactly).
    """
    stats = dict.fromkeys(STAT_KEYS, 0)
    cap = max_graph_nodes if max_graph_nodes is not None else 4 * max(1, n_compute(g0))
    evaluate = sweep if use_inner else (lambda g, db, f, d: default_eval(g, db, f))
    if seed is not None:
        stats["new_cost_records"] += ensure_profiled(g0, db, seed)
    a0, c0, t0, e0, ev, sw = evaluate(g0, db, f, d)
    stats["assignments_evaluated"] += ev
    stats["inner_sweeps"] += sw
    best = (g0, a0, c0, t0, e0)
    h0 = canonical_hash(g0)
    visited = {h0}
    heap = [(c0, h0)]
    pending = {h0: g0}
    expansions = 0
    while heap:
        cost, h = heapq.heappop(heap)
        if cost > alpha * best[2]:
            stats["queue_pruned"] += 1
            pending.pop(h, None)
            continue
        if max_expansions is not None and expansions >= max_expansions:
            break
        g = pending.pop(h)
        expansions += 1
        stats["graphs_explored"] += 1
        if trace is not None:
            trace.append(h)
        if cost == best[2]:
            stats["expanded_at_best"] += 1
        for cand in neighbors(g, rules):
            stats["graphs_generated"] += 1
            hc = canonical_hash(cand)
            if hc in visited:
                stats["graphs_deduped"] += 1
                continue
            visited.add(hc)
            if n_compute(cand) > cap:
                stats["node_cap_hits"] += 1
                continue
            if seed is not None:
                stats["new_cost_records"] += ensure_profiled(cand, db, seed)
            ca, cc, ct, ce, ev, sw = evaluate(cand, db, f, d)
            stats["assignments_evaluated"] += ev
            stats["inner_sweeps"] += sw
            prev = best[2]
            if cc < prev:
                best = (cand, ca, cc, ct, ce)
                stats["best_updates"] += 1
            if cc < alpha * prev:
                if len(heap) >= max_queue:
                    stats["queue_cap_hits"] += 1
                else:
                    heapq.heappush(heap, (cc, hc))
                    pending[hc] = cand
    g, a, c, t, e = best
    return {"graph": g, "hash": canonical_hash(g), "assignment": a, "cost": c, "time_ms": t,
            "energy": e, "power_w": e / t if t > 0 else 0.0, "stats": stats}
