"""Host-side graph IR: the operator DAG a user builds and hands to the search.

This is the drop-in surface of the reference's graph module
(reference: pkg/src/enerflow/graph.py).  Names, argument meaning, error types
and the on-disk JSON schema are the reference's; the representation is ours.
A `Graph` here is an immutable snapshot; the B200 search never walks these
Python objects on its hot path — `device.py` flattens a graph once into the
CSR records that live in HBM, and candidate graphs are only ever rebuilt as
Python objects when a caller asks for one (the optimised result, or
`neighbors`/`apply` at the operator API).

Conventions kept bit-for-bit because the canonical hash and the cost database
are keyed on them:
  * signature text: ``kind|in=AxBxC,..|key=value|...`` with the per-kind key
    order of reference graph.py:460-467 (graph.py:441-448 renders it);
  * tensor layout channels-first, weights float64.
"""

from __future__ import annotations

import base64
import functools
import heapq
import json
from dataclasses import dataclass, field
from enum import Enum
from typing import Any, Callable, Mapping

import numpy as np

from .errors import GraphFormatError, MissingInput, ShapeMismatch


class OpKind(str, Enum):
    INPUT = "input"
    CONV2D = "conv2d"
    MATMUL = "matmul"
    RELU = "relu"
    ADD = "add"
    CONCAT = "concat"
    SPLIT = "split"
    MAXPOOL = "maxpool"
    AVGPOOL = "avgpool"
    BATCHNORM = "batchnorm"
    IDENTITY = "identity"


# numeric kind codes shared with the CUDA side (csrc/ef_types.h EF_KIND_*)
KIND_CODE = {k: i for i, k in enumerate(OpKind)}

# fixed input counts; concat is variadic (>= 2) and handled separately
_FIXED_ARITY = {
    OpKind.INPUT: 0, OpKind.CONV2D: 1, OpKind.MATMUL: 1, OpKind.RELU: 1,
    OpKind.ADD: 2, OpKind.SPLIT: 1, OpKind.MAXPOOL: 1, OpKind.AVGPOOL: 1,
    OpKind.BATCHNORM: 1, OpKind.IDENTITY: 1,
}

# signature parameter keys per kind, alphabetical (reference graph.py:460-467)
SIG_KEYS = {
    OpKind.CONV2D: ("has_activation", "kernel", "out_channels", "padding", "stride"),
    OpKind.MATMUL: ("out_features",),
    OpKind.CONCAT: ("axis",),
    OpKind.SPLIT: ("axis", "sizes"),
    OpKind.MAXPOOL: ("kernel", "padding", "stride"),
    OpKind.AVGPOOL: ("kernel", "padding", "stride"),
}

_NEEDED_PARAMS = {
    OpKind.INPUT: ("name",),
    OpKind.CONV2D: ("out_channels", "kernel", "stride", "padding", "has_activation"),
    OpKind.MATMUL: ("out_features",),
    OpKind.CONCAT: ("axis",),
    OpKind.SPLIT: ("axis", "sizes"),
    OpKind.MAXPOOL: ("kernel", "stride", "padding"),
    OpKind.AVGPOOL: ("kernel", "stride", "padding"),
}
_NEEDED_WEIGHTS = {
    OpKind.CONV2D: ("weight",),
    OpKind.MATMUL: ("weight",),
    OpKind.BATCHNORM: ("scale", "shift"),
}


@dataclass(frozen=True)
class TensorShape:
    dims: tuple[int, ...]

    def __post_init__(self):
        dims = tuple(self.dims)
        object.__setattr__(self, "dims", dims)
        if not dims:
            raise ValueError("tensor rank must be >= 1")
        for d in dims:
            if not isinstance(d, int) or d < 1:
                raise ValueError(f"tensor dims must be positive integers, got {dims}")

    @property
    def rank(self) -> int:
        return len(self.dims)

    @property
    def numel(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    def __str__(self) -> str:
        return "x".join(map(str, self.dims))


def shape(*dims: int) -> TensorShape:
    return TensorShape(tuple(dims))


@dataclass(frozen=True)
class EdgeRef:
    node: int
    port: int = 0


@dataclass(frozen=True, eq=False)
class Node:
    id: int
    kind: OpKind
    inputs: tuple[EdgeRef, ...] = ()
    params: Mapping[str, Any] = field(default_factory=dict)
    weights: Mapping[str, np.ndarray] = field(default_factory=dict)

    def n_outputs(self) -> int:
        return len(self.params["sizes"]) if self.kind is OpKind.SPLIT else 1


@dataclass(frozen=True, eq=False)
class Graph:
    nodes: dict[int, Node]
    inputs: tuple[tuple[str, TensorShape], ...]
    outputs: tuple[EdgeRef, ...]

    def node(self, node_id: int) -> Node:
        return self.nodes[node_id]

    def node_ids(self) -> list[int]:
        return sorted(self.nodes)

    def compute_nodes(self) -> list[Node]:
        return [self.nodes[i] for i in sorted(self.nodes) if self.nodes[i].kind is not OpKind.INPUT]

    def input_shape(self, name: str) -> TensorShape | None:
        return dict(self.inputs).get(name)


def consumers(g: Graph) -> dict[EdgeRef, list[tuple[int, int]]]:
    uses: dict[EdgeRef, list[tuple[int, int]]] = {}
    for nid in sorted(g.nodes):
        for slot, ref in enumerate(g.nodes[nid].inputs):
            uses.setdefault(ref, []).append((nid, slot))
    return uses


def topological_order(g: Graph) -> list[int]:
    """Kahn order with the smallest ready id first (reference graph.py:147-173)."""
    pending = {nid: len(n.inputs) for nid, n in g.nodes.items()}
    users: dict[int, list[int]] = {nid: [] for nid in g.nodes}
    for nid, n in g.nodes.items():
        for ref in n.inputs:
            if ref.node not in g.nodes:
                raise ValueError(f"node {nid} references missing node {ref.node}")
            users[ref.node].append(nid)
    ready = sorted(nid for nid, c in pending.items() if c == 0)
    order: list[int] = []
    while ready:
        nid = heapq.heappop(ready)
        order.append(nid)
        for u in users[nid]:
            pending[u] -= 1
            if pending[u] == 0:
                heapq.heappush(ready, u)
    if len(order) != len(g.nodes):
        raise ValueError("cycle detected")
    return order


# ---------------------------------------------------------------------------
# shape rules
# ---------------------------------------------------------------------------

def _two(v) -> tuple[int, int]:
    a, b = v
    return int(a), int(b)


def _window_out(node: Node, s: TensorShape, what: str) -> tuple[int, int]:
    _, _, h, w = s.dims
    kh, kw = _two(node.params["kernel"])
    sh, sw = _two(node.params["stride"])
    ph, pw = _two(node.params["padding"])
    if h + 2 * ph < kh or w + 2 * pw < kw:
        raise ShapeMismatch(node.id, f"{what} kernel {kh}x{kw} larger than padded input {s}")
    return (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1


def _shape_conv(node, ins, g):
    (s,) = ins
    if s.rank != 4:
        raise ShapeMismatch(node.id, f"conv2d expects rank-4 input, got {s}")
    b, c, _, _ = s.dims
    oc = node.params["out_channels"]
    kh, kw = _two(node.params["kernel"])
    w = node.weights.get("weight")
    if w is not None and w.shape != (oc, c, kh, kw):
        raise ShapeMismatch(node.id, f"conv2d weight shape {w.shape} != ({oc}, {c}, {kh}, {kw})")
    bias = node.weights.get("bias")
    if bias is not None and bias.shape != (oc,):
        raise ShapeMismatch(node.id, f"conv2d bias shape {bias.shape} != ({oc},)")
    oh, ow = _window_out(node, s, "conv2d")
    return (shape(b, oc, oh, ow),)


def _shape_matmul(node, ins, g):
    (s,) = ins
    if s.rank != 2:
        raise ShapeMismatch(node.id, f"matmul expects rank-2 input, got {s}")
    b, f = s.dims
    of = node.params["out_features"]
    w = node.weights.get("weight")
    if w is not None and w.shape != (f, of):
        raise ShapeMismatch(node.id, f"matmul weight shape {w.shape} != ({f}, {of})")
    return (shape(b, of),)


def _shape_same(node, ins, g):
    return (ins[0],)


def _shape_bn(node, ins, g):
    (s,) = ins
    if s.rank < 2:
        raise ShapeMismatch(node.id, f"batchnorm expects rank >= 2, got {s}")
    for key in ("scale", "shift"):
        arr = node.weights.get(key)
        if arr is not None and arr.shape != (s.dims[1],):
            raise ShapeMismatch(node.id, f"batchnorm {key} shape {arr.shape} != ({s.dims[1]},)")
    return (s,)


def _shape_add(node, ins, g):
    a, b = ins
    if a != b:
        raise ShapeMismatch(node.id, f"add inputs differ: {a} vs {b}")
    return (a,)


def _shape_concat(node, ins, g):
    axis = node.params["axis"]
    first = ins[0]
    if not 0 <= axis < first.rank:
        raise ShapeMismatch(node.id, f"concat axis {axis} out of range for {first}")
    for s in ins:
        if s.rank != first.rank:
            raise ShapeMismatch(node.id, f"concat rank mismatch: {first} vs {s}")
        if any(d != axis and s.dims[d] != first.dims[d] for d in range(first.rank)):
            raise ShapeMismatch(node.id, f"concat inputs differ off-axis: {first} vs {s}")
    dims = list(first.dims)
    dims[axis] = sum(s.dims[axis] for s in ins)
    return (TensorShape(tuple(dims)),)


def _shape_split(node, ins, g):
    (s,) = ins
    axis = node.params["axis"]
    sizes = [int(x) for x in node.params["sizes"]]
    if not 0 <= axis < s.rank:
        raise ShapeMismatch(node.id, f"split axis {axis} out of range for {s}")
    if sum(sizes) != s.dims[axis]:
        raise ShapeMismatch(node.id, f"split sizes {tuple(sizes)} do not sum to dim {s.dims[axis]}")
    out = []
    for part in sizes:
        dims = list(s.dims)
        dims[axis] = part
        out.append(TensorShape(tuple(dims)))
    return tuple(out)


def _shape_pool(node, ins, g):
    (s,) = ins
    if s.rank != 4:
        raise ShapeMismatch(node.id, f"pool expects rank-4 input, got {s}")
    kh, kw = _two(node.params["kernel"])
    ph, pw = _two(node.params["padding"])
    if ph >= kh or pw >= kw:
        raise ShapeMismatch(node.id, f"pool padding ({ph},{pw}) must be < kernel ({kh},{kw})")
    oh, ow = _window_out(node, s, "pool")
    return (shape(s.dims[0], s.dims[1], oh, ow),)


def _shape_input(node, ins, g):
    declared = g.input_shape(node.params["name"])
    if declared is None:
        raise ShapeMismatch(node.id, f"unknown graph input {node.params['name']!r}")
    return (declared,)


_SHAPE_RULE: dict[OpKind, Callable] = {
    OpKind.INPUT: _shape_input, OpKind.CONV2D: _shape_conv, OpKind.MATMUL: _shape_matmul,
    OpKind.RELU: _shape_same, OpKind.IDENTITY: _shape_same, OpKind.BATCHNORM: _shape_bn,
    OpKind.ADD: _shape_add, OpKind.CONCAT: _shape_concat, OpKind.SPLIT: _shape_split,
    OpKind.MAXPOOL: _shape_pool, OpKind.AVGPOOL: _shape_pool,
}


def infer_shapes(g: Graph) -> dict[int, tuple[TensorShape, ...]]:
    out: dict[int, tuple[TensorShape, ...]] = {}
    for nid in topological_order(g):
        node = g.nodes[nid]
        ins = []
        for ref in node.inputs:
            produced = out[ref.node]
            if ref.port >= len(produced):
                raise ShapeMismatch(nid, f"reference to missing output port {ref.port} of node {ref.node}")
            ins.append(produced[ref.port])
        out[nid] = _SHAPE_RULE[node.kind](node, ins, g)
    return out


def validate(g: Graph) -> list[str]:
    """Every violated graph invariant, as text (empty list = valid)."""
    bad: list[str] = []
    names = [n for n, _ in g.inputs]
    if len(names) != len(set(names)):
        bad.append("duplicate graph input names")
    for nid, node in g.nodes.items():
        if nid != node.id:
            bad.append(f"node key {nid} != node id {node.id}")
        if node.kind is OpKind.CONCAT:
            if len(node.inputs) < 2:
                bad.append(f"node {nid}: concat needs >= 2 inputs")
        elif len(node.inputs) != _FIXED_ARITY[node.kind]:
            bad.append(f"node {nid}: {node.kind.value} expects {_FIXED_ARITY[node.kind]} inputs, "
                       f"has {len(node.inputs)}")
        bad += [f"node {nid}: missing param {p!r}" for p in _NEEDED_PARAMS.get(node.kind, ())
                if p not in node.params]
        bad += [f"node {nid}: missing weight {w!r}" for w in _NEEDED_WEIGHTS.get(node.kind, ())
                if w not in node.weights]
        for ref in node.inputs:
            if ref.node not in g.nodes:
                bad.append(f"node {nid}: dangling reference to node {ref.node}")
            elif not 0 <= ref.port < g.nodes[ref.node].n_outputs():
                bad.append(f"node {nid}: bad port {ref.port} on node {ref.node}")
        if node.kind is OpKind.CONV2D:
            p = node.params
            if "out_channels" in p and p["out_channels"] < 1:
                bad.append(f"node {nid}: out_channels must be >= 1")
            for key in ("kernel", "stride"):
                if key in p and any(v < 1 for v in p[key]):
                    bad.append(f"node {nid}: {key} entries must be >= 1")
            if "padding" in p and any(v < 0 for v in p["padding"]):
                bad.append(f"node {nid}: padding entries must be >= 0")
        if node.kind is OpKind.SPLIT and "sizes" in node.params:
            if any(s < 1 for s in node.params["sizes"]):
                bad.append(f"node {nid}: split sizes must be >= 1")
    if bad:
        return bad
    for ref in g.outputs:
        if ref.node not in g.nodes:
            bad.append(f"output references missing node {ref.node}")
        elif not 0 <= ref.port < g.nodes[ref.node].n_outputs():
            bad.append(f"output references bad port {ref.port} of node {ref.node}")
    if not g.outputs:
        bad.append("graph has no outputs")
    if bad:
        return bad
    try:
        topological_order(g)
    except ValueError as exc:
        return [str(exc)]
    try:
        infer_shapes(g)
    except ShapeMismatch as exc:
        return [f"shape inference failed: {exc}"]
    live = _reachable(g.nodes, g.outputs)
    bad += [f"node {nid} is not reachable from any output" for nid in sorted(set(g.nodes) - live)]
    for nid, node in g.nodes.items():
        if node.kind is OpKind.INPUT and g.input_shape(node.params["name"]) is None:
            bad.append(f"node {nid}: input name {node.params['name']!r} not declared")
    return bad


def _reachable(nodes: Mapping[int, Node], outputs) -> set[int]:
    seen: set[int] = set()
    todo = [r.node for r in outputs]
    while todo:
        nid = todo.pop()
        if nid not in seen:
            seen.add(nid)
            todo.extend(r.node for r in nodes[nid].inputs)
    return seen


# ---------------------------------------------------------------------------
# signatures
# ---------------------------------------------------------------------------

def _fmt(v: Any) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, (tuple, list)):
        return "x".join(str(int(x)) for x in v)
    return str(v)


def _norm(v: Any) -> Any:
    if isinstance(v, bool):
        return v
    if isinstance(v, (tuple, list)):
        return tuple(int(x) for x in v)
    if isinstance(v, int):
        return int(v)
    return v


@dataclass(frozen=True)
class NodeSignature:
    """Structural identity of a node (kind, input shapes, hyperparameters)."""

    kind: str
    input_shapes: tuple[tuple[int, ...], ...]
    params: tuple[tuple[str, Any], ...]

    @functools.cached_property
    def text(self) -> str:
        head = [self.kind]
        if self.input_shapes:
            head.append("in=" + ",".join("x".join(map(str, s)) for s in self.input_shapes))
        head += [f"{k}={_fmt(v)}" for k, v in self.params]
        return "|".join(head)

    def __str__(self) -> str:
        return self.text

    def param(self, key: str, default=None):
        return dict(self.params).get(key, default)


def signature_for(node: Node, in_shapes, g: Graph) -> NodeSignature:
    if node.kind is OpKind.INPUT:
        return NodeSignature("input", (), (("shape", g.input_shape(node.params["name"]).dims),))
    keys = SIG_KEYS.get(node.kind, ())
    return NodeSignature(node.kind.value, tuple(s.dims for s in in_shapes),
                         tuple((k, _norm(node.params[k])) for k in keys))


def signatures(g: Graph) -> dict[int, NodeSignature]:
    shapes = infer_shapes(g)
    return {nid: signature_for(g.nodes[nid], [shapes[r.node][r.port] for r in g.nodes[nid].inputs], g)
            for nid in sorted(g.nodes)}


def signature(node: Node, g: Graph) -> NodeSignature:
    return signatures(g)[node.id]


# ---------------------------------------------------------------------------
# float64 interpreter (test utility for rewrite soundness; not on any hot path)
# ---------------------------------------------------------------------------

def _windows(x, kernel, stride, padding, fill):
    kh, kw = kernel
    sh, sw = stride
    ph, pw = padding
    xp = np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)), constant_values=fill)
    win = np.lib.stride_tricks.sliding_window_view(xp, (kh, kw), axis=(2, 3))
    return win[:, :, ::sh, ::sw, :, :]


def _run_node(node: Node, args, feeds):
    k, p, w = node.kind, node.params, node.weights
    if k is OpKind.INPUT:
        return (feeds[p["name"]],)
    if k is OpKind.CONV2D:
        y = np.einsum("bcxykl,ockl->boxy",
                      _windows(args[0], w["weight"].shape[2:], _two(p["stride"]), _two(p["padding"]), 0.0),
                      w["weight"], optimize=True)
        if "bias" in w:
            y = y + w["bias"][None, :, None, None]
        return (np.maximum(y, 0.0) if p["has_activation"] else y,)
    if k is OpKind.MATMUL:
        return (args[0] @ w["weight"],)
    if k is OpKind.RELU:
        return (np.maximum(args[0], 0.0),)
    if k is OpKind.ADD:
        return (args[0] + args[1],)
    if k is OpKind.CONCAT:
        return (np.concatenate(args, axis=p["axis"]),)
    if k is OpKind.SPLIT:
        return tuple(np.split(args[0], np.cumsum(p["sizes"])[:-1], axis=p["axis"]))
    if k is OpKind.MAXPOOL:
        return (_windows(args[0], _two(p["kernel"]), _two(p["stride"]), _two(p["padding"]), -np.inf)
                .max(axis=(-2, -1)),)
    if k is OpKind.AVGPOOL:
        return (_windows(args[0], _two(p["kernel"]), _two(p["stride"]), _two(p["padding"]), 0.0)
                .mean(axis=(-2, -1)),)
    if k is OpKind.BATCHNORM:
        bshape = (1, -1) + (1,) * (args[0].ndim - 2)
        return (args[0] * w["scale"].reshape(bshape) + w["shift"].reshape(bshape),)
    if k is OpKind.IDENTITY:
        return (args[0],)
    raise ShapeMismatch(node.id, f"unhandled kind {k}")


def execute(g: Graph, feeds: Mapping[str, np.ndarray]) -> dict[str, np.ndarray]:
    declared = dict(g.inputs)
    for name in feeds:
        if name not in declared:
            raise MissingInput(name, "unknown input tensor")
    cast = {}
    for name, s in g.inputs:
        if name not in feeds:
            raise MissingInput(name)
        arr = np.asarray(feeds[name], dtype=np.float64)
        if arr.shape != s.dims:
            raise ShapeMismatch(-1, f"input {name!r} has shape {arr.shape}, declared {s}")
        cast[name] = arr
    vals: dict[tuple[int, int], np.ndarray] = {}
    for nid in topological_order(g):
        node = g.nodes[nid]
        outs = _run_node(node, [vals[(r.node, r.port)] for r in node.inputs], cast)
        for port, arr in enumerate(outs):
            vals[(nid, port)] = arr
    return {f"out{i}": vals[(r.node, r.port)] for i, r in enumerate(g.outputs)}


def equivalent(g1: Graph, g2: Graph, trials: int = 50, tol: float = 1e-4, seed: int = 0) -> bool:
    """Randomised refuter: False proves inequivalence, True means no counterexample."""
    if list(g1.inputs) != list(g2.inputs) or len(g1.outputs) != len(g2.outputs):
        return False
    rng = np.random.default_rng(seed)
    for _ in range(trials):
        feeds = {name: rng.standard_normal(s.dims) for name, s in g1.inputs}
        a, b = execute(g1, feeds), execute(g2, feeds)
        for key in a:
            if a[key].shape != b[key].shape or not np.allclose(a[key], b[key], rtol=tol, atol=1e-12):
                return False
    return True


# ---------------------------------------------------------------------------
# builder
# ---------------------------------------------------------------------------

class GraphBuilder:
    """Incremental construction; node ids are allocated 0, 1, 2, ..."""

    def __init__(self):
        self._nodes: dict[int, Node] = {}
        self._inputs: list[tuple[str, TensorShape]] = []
        self._outputs: list[EdgeRef] = []

    def _push(self, kind: OpKind, inputs, params, weights) -> int:
        nid = len(self._nodes)
        self._nodes[nid] = Node(nid, kind, tuple(inputs), params, weights)
        return nid

    def input(self, name: str, dims) -> EdgeRef:
        self._inputs.append((name, TensorShape(tuple(dims))))
        return EdgeRef(self._push(OpKind.INPUT, (), {"name": name}, {}))

    def conv2d(self, x: EdgeRef, weight, bias=None, stride=(1, 1), padding=(0, 0),
               has_activation: bool = False) -> EdgeRef:
        weight = np.asarray(weight, dtype=np.float64)
        params = {"out_channels": int(weight.shape[0]),
                  "kernel": (int(weight.shape[2]), int(weight.shape[3])),
                  "stride": _two(stride), "padding": _two(padding),
                  "has_activation": bool(has_activation)}
        weights = {"weight": weight}
        if bias is not None:
            weights["bias"] = np.asarray(bias, dtype=np.float64)
        return EdgeRef(self._push(OpKind.CONV2D, (x,), params, weights))

    def matmul(self, x: EdgeRef, weight) -> EdgeRef:
        weight = np.asarray(weight, dtype=np.float64)
        return EdgeRef(self._push(OpKind.MATMUL, (x,), {"out_features": int(weight.shape[1])},
                                  {"weight": weight}))

    def relu(self, x: EdgeRef) -> EdgeRef:
        return EdgeRef(self._push(OpKind.RELU, (x,), {}, {}))

    def add(self, x: EdgeRef, y: EdgeRef) -> EdgeRef:
        return EdgeRef(self._push(OpKind.ADD, (x, y), {}, {}))

    def identity(self, x: EdgeRef) -> EdgeRef:
        return EdgeRef(self._push(OpKind.IDENTITY, (x,), {}, {}))

    def batchnorm(self, x: EdgeRef, scale, shift) -> EdgeRef:
        return EdgeRef(self._push(OpKind.BATCHNORM, (x,), {},
                                  {"scale": np.asarray(scale, dtype=np.float64),
                                   "shift": np.asarray(shift, dtype=np.float64)}))

    def concat(self, xs, axis: int = 1) -> EdgeRef:
        return EdgeRef(self._push(OpKind.CONCAT, tuple(xs), {"axis": int(axis)}, {}))

    def split(self, x: EdgeRef, sizes, axis: int = 1) -> tuple[EdgeRef, ...]:
        sizes = tuple(int(s) for s in sizes)
        nid = self._push(OpKind.SPLIT, (x,), {"axis": int(axis), "sizes": sizes}, {})
        return tuple(EdgeRef(nid, p) for p in range(len(sizes)))

    def _pool(self, kind, x, kernel, stride, padding) -> EdgeRef:
        return EdgeRef(self._push(kind, (x,), {"kernel": _two(kernel), "stride": _two(stride),
                                               "padding": _two(padding)}, {}))

    def maxpool(self, x: EdgeRef, kernel=(2, 2), stride=(2, 2), padding=(0, 0)) -> EdgeRef:
        return self._pool(OpKind.MAXPOOL, x, kernel, stride, padding)

    def avgpool(self, x: EdgeRef, kernel=(2, 2), stride=(2, 2), padding=(0, 0)) -> EdgeRef:
        return self._pool(OpKind.AVGPOOL, x, kernel, stride, padding)

    def output(self, *refs: EdgeRef) -> None:
        self._outputs.extend(refs)

    def build(self, check: bool = True) -> Graph:
        g = Graph(dict(self._nodes), tuple(self._inputs), tuple(self._outputs))
        if check:
            problems = validate(g)
            if problems:
                raise GraphFormatError("invalid graph: " + "; ".join(problems))
        return g


# ---------------------------------------------------------------------------
# JSON schema (reference graph.py:785-875 documents the same layout)
# ---------------------------------------------------------------------------

_SEQ_PARAMS = {"kernel", "stride", "padding", "sizes", "shape"}


def _ref_out(ref: EdgeRef):
    return ref.node if ref.port == 0 else [ref.node, ref.port]


def _ref_in(obj, where: str) -> EdgeRef:
    if isinstance(obj, bool):
        raise GraphFormatError(f"{where}: bad edge reference {obj!r}")
    if isinstance(obj, int):
        return EdgeRef(obj)
    if isinstance(obj, list) and len(obj) == 2 and all(isinstance(v, int) for v in obj):
        return EdgeRef(obj[0], obj[1])
    raise GraphFormatError(f"{where}: bad edge reference {obj!r}")


def graph_to_json(g: Graph) -> dict:
    entries = []
    for nid in sorted(g.nodes):
        n = g.nodes[nid]
        item: dict[str, Any] = {
            "id": nid, "kind": n.kind.value,
            "params": {k: (list(v) if isinstance(v, tuple) else v) for k, v in sorted(n.params.items())},
            "inputs": [_ref_out(r) for r in n.inputs],
        }
        if n.weights:
            item["weights"] = {k: np.asarray(v, dtype=np.float64).tolist() for k, v in sorted(n.weights.items())}
        entries.append(item)
    return {"inputs": [{"name": name, "shape": list(s.dims)} for name, s in g.inputs],
            "nodes": entries, "outputs": [_ref_out(r) for r in g.outputs]}


def _weights_in(obj, nid: int) -> dict[str, np.ndarray]:
    out = {}
    for key, val in obj.items():
        try:
            if isinstance(val, dict):
                arr = np.frombuffer(base64.b64decode(val["b64"]), dtype=np.float64).reshape(val["shape"]).copy()
            else:
                arr = np.asarray(val, dtype=np.float64)
        except (KeyError, ValueError, TypeError) as exc:
            raise GraphFormatError(f"node {nid}: bad weight {key!r}: {exc}") from exc
        out[key] = arr
    return out


def graph_from_json(obj: dict) -> Graph:
    if not isinstance(obj, dict):
        raise GraphFormatError("graph document must be a JSON object")
    try:
        inputs = tuple((str(e["name"]), TensorShape(tuple(int(d) for d in e["shape"])))
                       for e in obj.get("inputs", []))
    except (KeyError, TypeError, ValueError) as exc:
        raise GraphFormatError(f"bad graph inputs: {exc}") from exc
    by_value = {k.value: k for k in OpKind}
    nodes: dict[int, Node] = {}
    for item in obj.get("nodes", []):
        nid = item.get("id")
        if not isinstance(nid, int) or isinstance(nid, bool) or nid < 0:
            raise GraphFormatError(f"bad node id {nid!r} (must be a non-negative integer)")
        if nid in nodes:
            raise GraphFormatError(f"node {nid}: duplicate id")
        kind = by_value.get(item.get("kind"))
        if kind is None:
            raise GraphFormatError(f"node {nid}: unknown kind {item.get('kind')!r}")
        params = {k: (tuple(int(x) for x in v) if k in _SEQ_PARAMS and isinstance(v, list) else v)
                  for k, v in item.get("params", {}).items()}
        refs = tuple(_ref_in(r, f"node {nid}") for r in item.get("inputs", []))
        nodes[nid] = Node(nid, kind, refs, params, _weights_in(item.get("weights", {}), nid))
    outputs = tuple(_ref_in(r, "outputs") for r in obj.get("outputs", []))
    return Graph(nodes, inputs, outputs)


def save_graph(g: Graph, path) -> None:
    with open(path, "w") as fh:
        json.dump(graph_to_json(g), fh, indent=2, sort_keys=True)
        fh.write("\n")


def load_graph(path) -> Graph:
    with open(path) as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise GraphFormatError(f"{path}: not valid JSON: {exc}") from exc
    return graph_from_json(doc)
