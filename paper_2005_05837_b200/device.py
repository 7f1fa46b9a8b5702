"""Host side of the B200 search: interning, graph records, and the step driver.

A `DeviceSession` owns one libef200 context on one GPU.  It

  * interns signature texts (id, ef_sig_desc, NodeSignature) and mirrors their
    cost rows into HBM (`ef_sig_put` / `ef_sig_costs`);
  * interns weight sets: original ones by the identity of the node's numpy
    arrays (uploaded once), derived ones by their derivation (op, a, b, s0) —
    the device computes derived tensors and every BLAKE2b digest;
  * converts a host `Graph` into a record (nodes in id order, CSR refs, a
    topological order) and back.

Misses: when a rewrite on the device creates a signature or a weight set that
is not interned yet, `ef_expand` returns EF_NEED_RESOLVE; `_resolve` interns
what the device asked for (profiling new signatures into a shadow database
that the search makes visible to the caller's database in the reference's
order) and the step is re-run.
"""

from __future__ import annotations

import ctypes as C
import os
import sys
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .costmodel import CostDatabase
from .errors import NativeUnavailable
from .ir import KIND_CODE, EdgeRef, Graph, Node, NodeSignature, OpKind, infer_shapes, signatures, topological_order
from .profiler import ProfilerSpec, profile_signature

_KIND_OF_CODE = {v: k for k, v in KIND_CODE.items()}
RULE_IDS = {"fuse-conv-relu": 0, "split-conv-activation": 1, "merge-parallel-convs": 2,
            "split-merged-conv": 3, "fold-identity": 4, "fuse-conv-batchnorm": 5}


def _dims4(dims) -> tuple[int, int, int, int]:
    d = list(dims)[:4]
    return tuple(d + [0] * (4 - len(d)))


def sig_desc_of(sig: NodeSignature, out0: tuple[int, ...] | None) -> tuple[N.SigDesc, bool]:
    """ef_sig_desc for a signature; exact for conv2d / relu / 2-way split (rank 4)."""
    d = N.SigDesc()
    kind = OpKind(sig.kind)
    d.kind = KIND_CODE[kind]
    exact = False
    if sig.input_shapes:
        s = sig.input_shapes[0]
        d.rank = len(s)
        d.in_[:] = _dims4(s)
    if out0 is not None:
        d.out[:] = _dims4(out0)
    p = dict(sig.params)
    rank_ok = d.rank == 4
    if kind is OpKind.CONV2D:
        d.oc = p["out_channels"]
        d.kh, d.kw = p["kernel"]
        d.sh, d.sw = p["stride"]
        d.ph, d.pw = p["padding"]
        d.act = int(bool(p["has_activation"]))
        exact = rank_ok
    elif kind is OpKind.RELU:
        exact = rank_ok
    elif kind is OpKind.SPLIT:
        sizes = p["sizes"]
        d.axis = p["axis"]
        d.nsizes = len(sizes)
        if len(sizes) == 2:
            d.s0, d.s1 = sizes
            exact = rank_ok
    return d, exact


def sig_from_desc(d: N.SigDesc) -> NodeSignature:
    """NodeSignature of a device-built descriptor (conv2d, relu or 2-way split)."""
    kind = _KIND_OF_CODE[d.kind]
    ins = (tuple(d.in_[: d.rank]),)
    if kind is OpKind.CONV2D:
        params = (("has_activation", bool(d.act)), ("kernel", (d.kh, d.kw)), ("out_channels", d.oc),
                  ("padding", (d.ph, d.pw)), ("stride", (d.sh, d.sw)))
    elif kind is OpKind.RELU:
        params = ()
    elif kind is OpKind.SPLIT:
        params = (("axis", d.axis), ("sizes", (d.s0, d.s1)))
    else:
        raise ValueError(f"device cannot create {kind}")
    return NodeSignature(kind.value, ins, params)


def _out_of_desc(d: N.SigDesc) -> tuple[int, ...]:
    return tuple(d.out[: d.rank])


@dataclass
class WsetInfo:
    kind: int
    oc: int
    w_shape: tuple | None
    has_bias: bool
    arrays: dict | None  # host arrays (original sets, or derived once downloaded)


def _hdr(key: str, shape: tuple) -> bytes:
    return key.encode() + str(tuple(int(x) for x in shape)).encode()


class DeviceSession:
    """One libef200 context bound to one CUDA device."""

    _default: "DeviceSession | None" = None
    _lock = threading.Lock()

    def __init__(self, device: int | None = None):
        self.L = N.lib()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        self.device = device
        self.ctx = self.L.ef_create(device)
        if not self.ctx:
            raise NativeUnavailable(f"ef_create({device}) failed")
        # held by users of the session's one geometry (rewrite.scratch_graph): the single-graph
        # entry points share the default session across threads
        self.lock = threading.RLock()
        # signatures
        self.sig_id: dict[str, int] = {}
        self.sig_list: list[NodeSignature] = []
        self.sig_out: list[tuple[int, ...] | None] = []
        self.sig_desc_key: dict[tuple, int] = {}
        self.rows_of: dict[int, list] = {}  # uploaded rows per sig id
        self.shadow = CostDatabase()         # rows profiled ahead of the reference's order
        # names
        self.name_id: dict[str, int] = {}
        # weight sets (0 = no weights)
        self.ws: list[WsetInfo] = [WsetInfo(0, 0, None, False, {})]
        self.ws_by_arrays: dict[tuple, int] = {}
        self.ws_keepalive: list = []
        self.ws_by_derive: dict[tuple, int] = {}
        self.geo: N.Geometry | None = None
        self.input_text = b""
        self.db: CostDatabase | None = None
        self.profiler: ProfilerSpec | None = None
        self._pinned, self._pinned_bytes = None, 0  # page-locked staging of step results
        self._apinned, self._apinned_bytes = None, 0  # the same for results_async

    @classmethod
    def reset_default(cls) -> None:
        """Destroy the process's default session (its tables, records and hashing scratch: a
        large-graph step sizes that scratch to most of the HBM); the next default() is fresh."""
        with cls._lock:
            if cls._default is not None:
                cls._default.close()
                cls._default = None

    @classmethod
    def default(cls) -> "DeviceSession":
        with cls._lock:
            if cls._default is None:
                cls._default = DeviceSession()
            return cls._default

    def close(self):
        if self._pinned:
            self.L.ef_host_free(self._pinned)
            self._pinned, self._pinned_bytes = None, 0
        if self._apinned:
            if self.ctx:
                self.results_wait()
            self.L.ef_host_free(self._apinned)
            self._apinned, self._apinned_bytes = None, 0
        if self.ctx:
            self.L.ef_destroy(self.ctx)
            self.ctx = None

    def _check(self, rc: int, what: str) -> int:
        return N.check(self.ctx, rc, what)

    # ------------------------------------------------------------------ interning

    def bind_costs(self, db: CostDatabase, profiler: ProfilerSpec | None) -> None:
        """Cost source for the next search: the caller's db, plus a shadow profiled eagerly."""
        if self.db is not db or self.profiler != profiler:
            self.shadow = CostDatabase()
        self.db, self.profiler = db, profiler
        for sid in range(len(self.sig_list)):
            self._upload_rows(sid)

    def _rows_for(self, sid: int) -> list:
        text = self.sig_list[sid].text
        if self.db is not None and self.db.has_signature(text):
            return self.db.rows_for(text)
        if self.sig_list[sid].kind == "input":
            return []
        if self.profiler is not None and not self.shadow.has_signature(text):
            profile_signature(self.sig_list[sid], self.shadow, self.profiler)
        return self.shadow.rows_for(text)

    def _upload_rows(self, sid: int) -> None:
        rows = self._rows_for(sid)
        if self.rows_of.get(sid) == rows:
            return
        n = len(rows)
        alg = (C.c_int32 * max(1, n))(*[r[0] for r in rows])
        t = (C.c_double * max(1, n))(*[r[1] for r in rows])
        e = (C.c_double * max(1, n))(*[r[2] for r in rows])
        self._check(self.L.ef_sig_costs(self.ctx, sid, n, alg, t, e), "ef_sig_costs")
        self.rows_of[sid] = rows

    def intern_sig(self, sig: NodeSignature, out0) -> int:
        sid = self.sig_id.get(sig.text)
        if sid is not None:
            return sid
        sid = len(self.sig_list)
        desc, exact = sig_desc_of(sig, out0)
        text = sig.text.encode()
        self._check(self.L.ef_sig_put(self.ctx, sid, C.byref(desc), text, len(text), int(exact)), "ef_sig_put")
        self.sig_id[sig.text] = sid
        self.sig_list.append(sig)
        self.sig_out.append(tuple(out0) if out0 is not None else None)
        if exact:
            self.sig_desc_key[desc.key()] = sid
        if self.db is not None or self.profiler is not None:
            self._upload_rows(sid)
        return sid

    def intern_name(self, name: str) -> int:
        nid = self.name_id.get(name)
        if nid is None:
            nid = len(self.name_id)
            raw = name.encode()
            self._check(self.L.ef_name_put(self.ctx, nid, raw, len(raw)), "ef_name_put")
            self.name_id[name] = nid
        return nid

    def intern_weights(self, node: Node) -> int:
        if not node.weights:
            return 0
        key = tuple((k, id(node.weights[k])) for k in sorted(node.weights))
        wid = self.ws_by_arrays.get(key)
        if wid is not None:
            return wid
        wid = len(self.ws)
        kind = KIND_CODE[node.kind]
        w = b = None
        hw = hb = b""
        if node.kind is OpKind.CONV2D:
            w = np.ascontiguousarray(node.weights["weight"], dtype=np.float64)
            hw = _hdr("weight", w.shape)
            if "bias" in node.weights:
                b = np.ascontiguousarray(node.weights["bias"], dtype=np.float64)
                hb = _hdr("bias", b.shape)
            oc = int(w.shape[0])
            info = WsetInfo(kind, oc, tuple(w.shape), b is not None, dict(node.weights))
        elif node.kind is OpKind.BATCHNORM:
            w = np.ascontiguousarray(node.weights["scale"], dtype=np.float64)
            b = np.ascontiguousarray(node.weights["shift"], dtype=np.float64)
            hw, hb = _hdr("scale", w.shape), _hdr("shift", b.shape)
            info = WsetInfo(kind, int(w.shape[0]), tuple(w.shape), True, dict(node.weights))
        elif node.kind is OpKind.MATMUL:
            w = np.ascontiguousarray(node.weights["weight"], dtype=np.float64)
            hw = _hdr("weight", w.shape)
            info = WsetInfo(kind, 0, tuple(w.shape), False, dict(node.weights))
        else:
            raise ValueError(f"node {node.id}: unexpected weights on a {node.kind.value} node")
        dp = C.POINTER(C.c_double)
        self._check(self.L.ef_wset_put(
            self.ctx, wid, kind, info.oc,
            w.ctypes.data_as(dp) if w is not None else None, 0 if w is None else w.size,
            b.ctypes.data_as(dp) if b is not None else None, 0 if b is None else b.size,
            hw, len(hw), hb, len(hb)), "ef_wset_put")
        self.ws.append(info)
        self.ws_by_arrays[key] = wid
        self.ws_keepalive.append(node.weights)
        return wid

    def _derive(self, op: int, a: int, b: int, s0: int) -> int:
        key = (op, a, b, s0)
        wid = self.ws_by_derive.get(key)
        if wid is not None:
            return wid
        A = self.ws[a]
        inner = A.w_shape[1:]
        if op == N.D_MERGE:
            oc = A.oc + self.ws[b].oc
        elif op == N.D_SLICE_LO:
            oc = s0
        elif op == N.D_SLICE_HI:
            oc = A.oc - s0
        else:
            oc = A.oc
        shape = (oc,) + tuple(inner)
        wid = len(self.ws)
        hw, hb = _hdr("weight", shape), _hdr("bias", (oc,))
        self._check(self.L.ef_wset_derive(self.ctx, wid, op, a, b, s0, hw, len(hw), hb, len(hb)), "ef_wset_derive")
        self.ws.append(WsetInfo(KIND_CODE[OpKind.CONV2D], oc, shape, True, None))
        self.ws_by_derive[key] = wid
        return wid

    def commit(self) -> None:
        self._check(self.L.ef_tables_commit(self.ctx), "ef_tables_commit")

    def last_commit_bytes(self) -> int:
        """Host->device bytes the last commit sent (incremental: only what changed)."""
        out = C.c_uint64(0)
        self._check(self.L.ef_commit_bytes(self.ctx, C.byref(out)), "ef_commit_bytes")
        return out.value

    def _pending_summary(self) -> str:
        ns, nd = C.c_uint32(0), C.c_uint32(0)
        self._check(self.L.ef_pending(self.ctx, None, 0, C.byref(ns), None, 0, C.byref(nd)), "ef_pending")
        sigs = (N.SigDesc * max(1, ns.value))()
        dvs = (C.c_int32 * max(4, 4 * nd.value))()
        self._check(self.L.ef_pending(self.ctx, sigs, ns.value, C.byref(ns), dvs, nd.value, C.byref(nd)), "ef_pending")
        return f"sigs={[sigs[i].key() for i in range(ns.value)]} known={list(self.sig_desc_key)[:8]} derives={list(dvs)[:4 * nd.value]}"

    def resolve_pending(self) -> bool:
        """Intern what the last ef_expand asked for, then commit.  -> whether anything new was
        interned."""
        ns, nd = C.c_uint32(0), C.c_uint32(0)
        self._check(self.L.ef_pending(self.ctx, None, 0, C.byref(ns), None, 0, C.byref(nd)), "ef_pending")
        sigs = (N.SigDesc * max(1, ns.value))()
        dvs = (C.c_int32 * max(4, 4 * nd.value))()
        self._check(self.L.ef_pending(self.ctx, sigs, ns.value, C.byref(ns), dvs, nd.value, C.byref(nd)), "ef_pending")
        n_sig, n_ws = len(self.sig_list), len(self.ws)
        for i in range(ns.value):
            d = sigs[i]
            if d.key() in self.sig_desc_key:
                continue
            sig = sig_from_desc(d)
            self.intern_sig(sig, _out_of_desc(d))
        seen = set()
        for i in range(nd.value):
            q = tuple(dvs[4 * i: 4 * i + 4])
            if q not in seen:
                seen.add(q)
                self._derive(*q)
        self.commit()
        return len(self.sig_list) != n_sig or len(self.ws) != n_ws

    # ------------------------------------------------------------------ records

    def set_geometry(self, g0: Graph, cap_nodes: int, cap_refs: int) -> None:
        self.input_text = "".join(f"{name}={s};" for name, s in g0.inputs).encode()
        geo = N.Geometry()
        self._check(self.L.ef_set_geometry(self.ctx, cap_nodes, cap_refs, max(1, len(g0.outputs)),
                                           self.input_text, len(self.input_text), C.byref(geo)), "ef_set_geometry")
        self.geo = geo

    def alloc(self) -> int:
        s = C.c_uint32(0)
        self._check(self.L.ef_record_alloc(self.ctx, C.byref(s)), "ef_record_alloc")
        return s.value

    def alloc_n(self, n: int) -> list[int]:
        out = (C.c_uint32 * max(1, n))()
        self._check(self.L.ef_records_alloc(self.ctx, n, out), "ef_records_alloc")
        return list(out)[:n]

    def free(self, slot: int) -> None:
        self._check(self.L.ef_record_free(self.ctx, slot), "ef_record_free")

    def free_n(self, slots: list[int]) -> None:
        if slots:
            self._check(self.L.ef_records_free(self.ctx, N.u32_array(slots), len(slots)), "ef_records_free")

    def _view(self, buf: np.ndarray, off: int, dtype, count: int) -> np.ndarray:
        return buf[off: off + np.dtype(dtype).itemsize * count].view(dtype)

    def encode(self, g: Graph) -> np.ndarray:
        """Flatten a graph into record bytes (interning its signatures and weights)."""
        G = self.geo
        ids = sorted(g.nodes)
        n = len(ids)
        if n > G.cap_nodes:
            raise ValueError(f"graph has {n} nodes, record capacity is {G.cap_nodes}")
        pos = {nid: i for i, nid in enumerate(ids)}
        sigs = signatures(g)
        shapes = infer_shapes(g)
        buf = np.zeros(G.record_bytes, dtype=np.uint8)
        nid_a = self._view(buf, G.off_nid, np.int32, n)
        sig_a = self._view(buf, G.off_sig, np.uint32, n)
        aux_a = self._view(buf, G.off_aux, np.uint32, n)
        nin_a = self._view(buf, G.off_nin, np.uint32, n)
        inoff_a = self._view(buf, G.off_inoff, np.uint32, n + 1)
        refs = []
        for i, nid in enumerate(ids):
            node = g.nodes[nid]
            nid_a[i] = nid
            sig_a[i] = self.intern_sig(sigs[nid], shapes[nid][0].dims)
            aux_a[i] = self.intern_name(node.params["name"]) if node.kind is OpKind.INPUT else self.intern_weights(node)
            nin_a[i] = len(node.inputs)
            inoff_a[i] = len(refs)
            refs += [(pos[r.node] << 8) | r.port for r in node.inputs]
        inoff_a[n] = len(refs)
        if len(refs) > G.cap_refs:
            raise ValueError("graph has more edges than the record capacity")
        self._view(buf, G.off_refs, np.uint32, len(refs))[:] = refs
        outs = [(pos[r.node] << 8) | r.port for r in g.outputs]
        self._view(buf, G.off_outs, np.uint32, len(outs))[:] = outs
        self._view(buf, G.off_topo, np.uint32, n)[:] = [pos[v] for v in topological_order(g)]
        hdr = self._view(buf, 0, np.int32, 4)
        hdr[:] = [n, len(refs), len(outs), len(g.compute_nodes())]
        return buf

    def upload(self, g: Graph) -> int:
        """Write g as a record and compute its node keys + sorted-key order on the device
        (every record must carry them before it can be expanded as a parent)."""
        buf = self.encode(g)
        self.commit()
        slot = self.alloc()
        self._check(self.L.ef_record_write(self.ctx, slot, buf.ctypes.data, buf.nbytes), "ef_record_write")
        self.hash_slots([slot])
        return slot

    def read_record(self, slot: int) -> np.ndarray:
        buf = np.zeros(self.geo.record_bytes, dtype=np.uint8)
        self._check(self.L.ef_record_read(self.ctx, slot, buf.ctypes.data, buf.nbytes), "ef_record_read")
        return buf

    def _weights_of(self, wid: int) -> dict:
        info = self.ws[wid]
        if info.arrays is None:
            wn, bn = C.c_uint64(0), C.c_uint64(0)
            self._check(self.L.ef_wset_read(self.ctx, wid, None, C.byref(wn), None, C.byref(bn)), "ef_wset_read")
            w = np.empty(wn.value, dtype=np.float64)
            b = np.empty(bn.value, dtype=np.float64)
            dp = C.POINTER(C.c_double)
            self._check(self.L.ef_wset_read(self.ctx, wid, w.ctypes.data_as(dp), C.byref(wn),
                                            b.ctypes.data_as(dp), C.byref(bn)), "ef_wset_read")
            info.arrays = {"weight": w.reshape(info.w_shape), "bias": b}
        return info.arrays

    def decode(self, buf: np.ndarray, g0: Graph) -> tuple[Graph, dict[int, int]]:
        """Record bytes -> (Graph, {node id: alg}) ; weights come from the host registry."""
        G = self.geo
        n, n_refs, n_out, _ = (int(x) for x in self._view(buf, 0, np.int32, 4))
        nid_a = self._view(buf, G.off_nid, np.int32, n)
        sig_a = self._view(buf, G.off_sig, np.uint32, n)
        aux_a = self._view(buf, G.off_aux, np.uint32, n)
        nin_a = self._view(buf, G.off_nin, np.uint32, n)
        inoff_a = self._view(buf, G.off_inoff, np.uint32, n + 1)
        refs = self._view(buf, G.off_refs, np.uint32, n_refs)
        outs = self._view(buf, G.off_outs, np.uint32, n_out)
        alg = self._view(buf, G.off_alg, np.uint8, n)
        names = {v: k for k, v in self.name_id.items()}
        nodes: dict[int, Node] = {}
        assign: dict[int, int] = {}
        for i in range(n):
            sig = self.sig_list[int(sig_a[i])]
            kind = OpKind(sig.kind)
            nid = int(nid_a[i])
            ins = tuple(EdgeRef(int(nid_a[int(r) >> 8]), int(r) & 255)
                        for r in refs[int(inoff_a[i]): int(inoff_a[i]) + int(nin_a[i])])
            if kind is OpKind.INPUT:
                params = {"name": names[int(aux_a[i])]}
                weights = {}
            else:
                params = {k: v for k, v in sig.params}
                weights = dict(self._weights_of(int(aux_a[i]))) if int(aux_a[i]) else {}
                assign[nid] = int(alg[i])
            nodes[nid] = Node(nid, kind, ins, params, weights)
        outputs = tuple(EdgeRef(int(nid_a[int(r) >> 8]), int(r) & 255) for r in outs)
        return Graph(nodes, g0.inputs, outputs), assign

    # ------------------------------------------------------------------ kernels

    def hash_slots(self, slots: list[int]) -> list[int]:
        n = len(slots)
        out = (C.c_uint64 * max(1, n))()
        self._check(self.L.ef_hash_records(self.ctx, N.u32_array(slots), n, out), "ef_hash_records")
        return [int(out[i]) for i in range(n)]

    def price_slots(self, slots: list[int], pp: N.PriceParams) -> list[N.CandResult]:
        n = len(slots)
        out = (N.CandResult * max(1, n))()
        self._check(self.L.ef_price_records(self.ctx, N.u32_array(slots), n, C.byref(pp), out), "ef_price_records")
        return [out[i] for i in range(n)]

    def expand(self, slots: list[int], rule_ids: list[int], pp: N.PriceParams,
               insert_visited: bool = True, results: bool = True):
        """One batched step (ef_expand).  -> the candidates' results (a view of a reused
        page-locked buffer), or with results=False only their count (read them with
        results_async / results_wait, overlapping the next step)."""
        parents = N.u32_array(slots)
        rules = N.i32_array(rule_ids)
        count = C.c_uint32(0)
        while True:
            rc = self.L.ef_expand(self.ctx, parents, len(slots), rules, len(rule_ids), C.byref(pp),
                                  int(insert_visited), C.byref(count))
            if rc == N.EF_NEED_RESOLVE:
                # a step records at most req_cap requests; retry while every round interns
                # something new (a round that interns nothing would loop forever)
                if not self.resolve_pending():
                    raise N.NativeError(f"ef_expand keeps asking for interning: {self._pending_summary()}")
                continue
            self._check(rc, "ef_expand")
            break
        return self._results(count.value) if results else count.value

    def results_async(self, n: int) -> np.ndarray:
        """Start copying the last step's n results to page-locked memory on the copy stream
        (ef_results_async); the returned view is valid after results_wait()."""
        need = max(1, n) * N.CAND_DTYPE.itemsize
        if self._apinned_bytes < need:
            self.results_wait()
            if self._apinned:
                self.L.ef_host_free(self._apinned)
            size = max(need, 2 * self._apinned_bytes)
            self._apinned = self.L.ef_host_alloc(size)
            if not self._apinned:
                raise N.NativeError("ef_host_alloc failed")
            self._apinned_bytes = size
        out = np.ctypeslib.as_array((C.c_uint8 * need).from_address(self._apinned)).view(N.CAND_DTYPE)[:n]
        if n:
            self._check(self.L.ef_results_async(self.ctx, self._apinned, n), "ef_results_async")
        return out

    def results_wait(self) -> None:
        self._check(self.L.ef_results_wait(self.ctx), "ef_results_wait")

    def _results(self, n: int) -> np.ndarray:
        """The last step's candidate results, copied into page-locked host memory (full D2H
        bandwidth).  The array is a view of a buffer the next step reuses: callers that keep
        results across steps copy them."""
        need = max(1, n) * N.CAND_DTYPE.itemsize
        if self._pinned_bytes < need:
            if self._pinned:
                self.L.ef_host_free(self._pinned)
            size = max(need, 2 * self._pinned_bytes)
            self._pinned = self.L.ef_host_alloc(size)
            if not self._pinned:
                raise N.NativeError("ef_host_alloc failed")
            self._pinned_bytes = size
        out = np.ctypeslib.as_array((C.c_uint8 * need).from_address(self._pinned)).view(N.CAND_DTYPE)[:n]
        if n:
            self._check(self.L.ef_results(self.ctx, self._pinned, n), "ef_results")
        return out

    # ---- hash-owner sharding (see shard.py) ------------------------------------------

    def expand_hashes(self, slots: list[int], rule_ids: list[int], pp: N.PriceParams | None = None) -> int:
        """Match, plan and hash the candidates of `slots` (no dedup).  With `pp`, large steps
        also price every candidate speculatively beside the hashing (ef_expand_hashes_spec);
        expand_finish* then keeps the survivors' prices."""
        parents = N.u32_array(slots)
        rules = N.i32_array(rule_ids)
        count = C.c_uint32(0)
        while True:
            if pp is not None:
                rc = self.L.ef_expand_hashes_spec(self.ctx, parents, len(slots), rules, len(rule_ids), C.byref(pp),
                                                  C.byref(count))
            else:
                rc = self.L.ef_expand_hashes(self.ctx, parents, len(slots), rules, len(rule_ids), C.byref(count))
            if rc == N.EF_NEED_RESOLVE:
                if not self.resolve_pending():
                    raise N.NativeError(f"ef_expand_hashes keeps asking for interning: {self._pending_summary()}")
                continue
            self._check(rc, "ef_expand_hashes")
            return count.value

    def route_owners(self, world: int, order_base: int, send) -> list[int]:
        """`send`: int64 CUDA tensor with room for 2 * candidates (hash, global order) pairs."""
        counts = (C.c_uint32 * max(1, world))()
        self._check(self.L.ef_route_owners(self.ctx, world, order_base, C.c_void_p(send.data_ptr()), counts),
                    "ef_route_owners")
        return [int(counts[i]) for i in range(world)]

    def owner_mark(self, recv, verdict, insert_visited: bool) -> None:
        """`recv`: int64 CUDA tensor of pairs from every rank; `verdict`: int32 CUDA tensor, one per pair."""
        self._check(self.L.ef_owner_mark(self.ctx, C.c_void_p(recv.data_ptr()), recv.numel() // 2,
                                         C.c_void_p(verdict.data_ptr()), int(insert_visited)), "ef_owner_mark")

    def expand_finish(self, verdict_back, pp: N.PriceParams, n: int) -> np.ndarray:
        self._check(self.L.ef_expand_finish(self.ctx, C.c_void_p(verdict_back.data_ptr()), C.byref(pp)),
                    "ef_expand_finish")
        return self._results(n)

    def route_owners_padded(self, world: int, order_base: int, cap: int, send, counts) -> None:
        """`send`: int64 CUDA tensor of world * cap * 2 (hash, global order) pairs by owner bucket;
        `counts`: int32 CUDA tensor of world pairs per owner (both written on the device)."""
        self._check(self.L.ef_route_owners_padded(self.ctx, world, order_base, cap, C.c_void_p(send.data_ptr()),
                                                  C.c_void_p(counts.data_ptr())), "ef_route_owners_padded")

    def owner_mark_padded(self, recv, recv_counts, world: int, cap: int, verdict, insert_visited: bool) -> None:
        self._check(self.L.ef_owner_mark_padded(self.ctx, C.c_void_p(recv.data_ptr()), C.c_void_p(recv_counts.data_ptr()),
                                                world, cap, C.c_void_p(verdict.data_ptr()), int(insert_visited)),
                    "ef_owner_mark_padded")

    def expand_finish_padded(self, verdict_back, world: int, cap: int, pp: N.PriceParams, n: int) -> np.ndarray:
        self._check(self.L.ef_expand_finish_padded(self.ctx, C.c_void_p(verdict_back.data_ptr()), world, cap,
                                                   C.byref(pp)), "ef_expand_finish_padded")
        return self._results(n)

    def stream_handle(self) -> int:
        """The library stream (cudaStream_t) as an integer, for torch.cuda.ExternalStream."""
        out = C.c_void_p(0)
        self._check(self.L.ef_stream(self.ctx, C.byref(out)), "ef_stream")
        return int(out.value or 0)

    def reprune(self, best: float, alpha: float) -> np.ndarray:
        """Recompute the last step's alpha-prune flags from `best` (ef_reprune); -> fresh results."""
        self._check(self.L.ef_reprune(self.ctx, float(best), float(alpha)), "ef_reprune")
        return self._results(self.last_stats()["candidates"])

    def upload_fence(self) -> None:
        """Later steps wait for every asynchronous upload issued so far."""
        self._check(self.L.ef_upload_fence(self.ctx), "ef_upload_fence")

    def materialise(self, parent_slots: list[int], rule_ids: list[int], cand_parent: list[int],
                    cand_local: list[int]) -> list[int]:
        """Records of rewrites named (index into parent_slots, rewrite index within that parent)
        (ef_materialise); -> their new slots."""
        slots = self.alloc_n(len(cand_parent))
        args = (N.u32_array(parent_slots), len(parent_slots), N.i32_array(rule_ids), len(rule_ids),
                N.u32_array(cand_parent), N.u32_array(cand_local), len(cand_parent), N.u32_array(slots))
        while True:
            rc = self.L.ef_materialise(self.ctx, *args)
            # a rewrite another rank's step interned (sharded closure / search): intern it here
            if rc == N.EF_NEED_RESOLVE:
                if not self.resolve_pending():
                    raise N.NativeError(f"ef_materialise keeps asking for interning: {self._pending_summary()}")
                continue
            self._check(rc, "ef_materialise")
            return slots

    def keep(self, cand_idx: list[int]) -> list[int]:
        slots = self.alloc_n(len(cand_idx))
        self._check(self.L.ef_keep(self.ctx, N.u32_array(cand_idx), len(cand_idx), N.u32_array(slots)), "ef_keep")
        return slots

    def visited_reset(self, capacity: int) -> None:
        self._check(self.L.ef_visited_reset(self.ctx, capacity), "ef_visited_reset")

    def visited_insert(self, hashes: list[int]) -> None:
        arr = (C.c_uint64 * max(1, len(hashes)))(*hashes)
        self._check(self.L.ef_visited_insert(self.ctx, arr, len(hashes)), "ef_visited_insert")

    STAGES = ("match", "plan", "dirty", "keys", "sort", "digest", "dedup", "price")

    def last_timing(self) -> list[float]:
        """Device ms of the last step per stage (STAGES), CUDA events on the library stream."""
        ms = (C.c_float * 9)()
        self.L.ef_last_timing(self.ctx, ms, 9)
        return list(ms)[:8]

    def last_step_ms(self) -> float:
        """Device ms of the whole last step, match to price (a sharded step: exchange included)."""
        ms = (C.c_float * 9)()
        self.L.ef_last_timing(self.ctx, ms, 9)
        return float(ms[8])

    def last_stats(self) -> dict:
        out = (C.c_uint64 * 5)()
        self.L.ef_last_stats(self.ctx, out, 5)
        return {"key_compressions": int(out[0]), "digest_compressions": int(out[1]), "candidates": int(out[2]),
                "priced": int(out[3]), "kernels": int(out[4])}

    def b2b_peak(self) -> float:
        """Measured BLAKE2b compressions/s of this GPU (the hash kernels' ALU roofline)."""
        r = C.c_double(0)
        self._check(self.L.ef_b2b_peak(self.ctx, C.byref(r)), "ef_b2b_peak")
        return r.value

    def pack(self, recs: list[np.ndarray]) -> tuple[np.ndarray, np.ndarray]:
        """Compact host form of full records (used bytes only) for ef_records_write_packed."""
        G = self.geo
        parts, offs, at = [], [], 0
        for buf in recs:
            n, n_refs, n_out, n_comp = (int(x) for x in buf[:16].view(np.int32))
            u32 = lambda off, cnt: buf[off: off + 4 * cnt].view(np.uint32)  # noqa: E731
            blob = np.concatenate([np.array([n, n_refs, n_out, n_comp], dtype=np.uint32), u32(G.off_nid, n),
                                   u32(G.off_sig, n), u32(G.off_aux, n), u32(G.off_nin, n), u32(G.off_inoff, n + 1),
                                   u32(G.off_topo, n), u32(G.off_refs, n_refs), u32(G.off_outs, n_out)])
            parts.append(blob)
            offs.append(at)
            at += 4 * blob.size
        return np.concatenate(parts), np.array(offs, dtype=np.uint64)

    def write_packed(self, slots: list[int], blob: np.ndarray, offsets: np.ndarray, asynchronous: bool = False) -> None:
        """Upload compact records (see pack); asynchronous=True queues the copy, unpacking and
        hashing on the upload stream, overlapping a step; call upload_fence() before a step reads
        them (blob must be page-locked and unchanged until then)."""
        fn = self.L.ef_records_write_packed_async if asynchronous else self.L.ef_records_write_packed
        self._check(fn(self.ctx, N.u32_array(slots), len(slots), blob.ctypes.data,
                       offsets.ctypes.data_as(C.POINTER(C.c_uint64)), blob.nbytes), "ef_records_write_packed")


def price_params(f, d: int, use_inner: bool, node_cap: int, alpha: float = 0.0,
                 best: float = float("inf"), per_parent: bool = False) -> N.PriceParams:
    """ef_price_params: the cost function, the inner search, the node cap and the step's alpha-prune
    (alpha = 0: no prune flags).  Start totals follow this interpreter's sum() (Neumaier from
    CPython 3.12 on, left to right before)."""
    kind, w, ct, ce, cp, tr, er, pr = f.device_params()
    return N.PriceParams(kind, int(d), int(bool(use_inner)), int(node_cap), w, ct, ce, cp, tr, er, pr,
                         float(best), float(alpha), int(sys.version_info < (3, 12)), int(per_parent))
