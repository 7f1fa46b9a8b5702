"""Hash-owner sharding of the frontier over ranks (one process per GPU).

The reference deduplicates every generated graph against one visited set and
keeps the first graph per hash in (rule, site) order (rules.py:79-88,
search.py:245-251).  Across ranks the frontier is split by parent, so the
global candidate order is rank-major, and deduplication is owned by hash: rank
`hash % world` receives every (hash, global order) pair it owns, decides first
occurrence (smallest global order) and membership in its shard of the visited
set, and sends the verdicts back.  The result on every rank is exactly the
single-rank result for the concatenated frontier (tests/test_shard.py,
tests/test_gpu_shard.py).

`OwnerExchange` is the collective layer (torch.distributed: NCCL over NVLink on
the GPUs, gloo in the CPU tests).  The exchange uses fixed-capacity buckets
(`cap` pairs per destination, cap = the largest candidate count of any rank, one
all-reduce), so the per-owner counts stay on the device and travel beside the
pairs; on the GPUs the all-to-alls run on the library's own stream
(torch.cuda.ExternalStream over ef_stream), so a sharded step has no host
round trip between its kernels and its collectives.  The per-rank work is the
device session's `expand_hashes` / `route_owners_padded` / `owner_mark_padded`
/ `expand_finish_padded` (libef200).

`gather_batch` is the all-gather the sharded search (frontier.outer_search with
`exchange=`) uses: every rank expands a contiguous slice of the batch, the
alpha-prune flags get the cross-rank exclusive minimum (the north_star
all-reduce for the global best), and the results are all-gathered so every rank
replays the same batch.
"""

from __future__ import annotations

import contextlib

import numpy as np
import torch
import torch.distributed as dist


def owner_of(h: int, world: int) -> int:
    """Rank owning a candidate hash (same rule as csrc/ef_step.cuh owner_of)."""
    return h % world


class OwnerExchange:
    """Collectives of the sharded step, closure and search."""

    def __init__(self, group=None, device: torch.device | None = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device if device is not None else torch.device("cpu")
        self._bufs: dict[str, torch.Tensor] = {}

    def buffer(self, name: str, numel: int, dtype) -> torch.Tensor:
        """A reusable buffer of at least `numel` elements (no allocator traffic per step)."""
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < numel or buf.dtype != dtype:
            buf = torch.empty(max(numel, 1024), dtype=dtype, device=self.device)
            self._bufs[name] = buf
        return buf[:numel]

    def on_stream(self, session):
        """Run the enclosed collectives on the session's library stream (CUDA), in order with
        its kernels; a no-op on CPU (gloo)."""
        if self.device.type != "cuda" or session is None:
            return contextlib.nullcontext()
        handle = session.stream_handle()
        return torch.cuda.stream(torch.cuda.ExternalStream(handle, device=self.device))

    def order_base(self) -> int:
        """Global order of this rank's first candidate: rank-major order needs no exchange,
        (rank << 40) + index is monotone in (rank, index)."""
        return self.rank << 40

    def max_int(self, x: int) -> int:
        t = torch.tensor([int(x)], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def to_owners(self, send: torch.Tensor, counts: torch.Tensor, cap: int, session=None):
        """`send`: [world][cap] (hash, order) pairs by owner, `counts`: [world] pairs per owner.
        -> ([world][cap] pairs this rank owns by source rank, [world] valid per source)."""
        recv = self.buffer("recv", send.numel(), torch.int64)
        rcounts = self.buffer("rcounts", self.world, torch.int32)
        with self.on_stream(session):
            dist.all_to_all_single(recv, send, group=self.group)
            dist.all_to_all_single(rcounts, counts, group=self.group)
        return recv, rcounts

    def back(self, verdict: torch.Tensor, cap: int, session=None) -> torch.Tensor:
        """Owner verdicts ([world][cap], by source) back to the senders ([world][cap], by owner)."""
        out = self.buffer("back", verdict.numel(), torch.int32)
        with self.on_stream(session):
            dist.all_to_all_single(out, verdict, group=self.group)
        return out

    def min(self, x: float) -> float:
        """Global best cost (all-reduce MIN)."""
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return float(t.item())

    def sum(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, group=self.group)
        return float(t.item())

    def all_gather_object(self, obj) -> list:
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out

    def exclusive_min(self, x: float, init: float) -> float:
        """min(init, x of every rank before this one): the best cost before this rank's first
        candidate in rank-major order."""
        t = torch.full((self.world,), float("inf"), dtype=torch.float64, device=self.device)
        t[self.rank] = x
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)  # each slot has one writer
        out = init
        for v in t[: self.rank].tolist():
            out = v if v < out else out
        return out


def sharded_expand(session, slots: list[int], rule_ids: list[int], pp, ex: OwnerExchange,
                   insert_visited: bool = False, phases: dict | None = None):
    """One frontier step over the parents of this rank with hash-owner deduplication.

    Returns this rank's candidate results (the layout of `DeviceSession.expand`); flags
    FIRST / VISITED are global, costs are those of this rank's survivors.  `phases` counts calls.
    """
    n = session.expand_hashes(slots, rule_ids, pp)
    cap = max(1, ex.max_int(n))  # the only host-visible size: every bucket of every rank fits
    world = ex.world
    send = ex.buffer("send", 2 * world * cap, torch.int64)
    counts = ex.buffer("counts", world, torch.int32)
    session.route_owners_padded(world, ex.order_base(), cap, send, counts)
    recv, rcounts = ex.to_owners(send, counts, cap, session)
    verdict = ex.buffer("verdict", world * cap, torch.int32)
    session.owner_mark_padded(recv, rcounts, world, cap, verdict, insert_visited)
    back = ex.back(verdict, cap, session)
    if phases is not None:
        phases["calls"] = phases.get("calls", 0) + 1
    return session.expand_finish_padded(back, world, cap, pp, n)


def _eligible_min(res: np.ndarray, priced: int, first: int) -> float:
    """Minimum cost over the candidates the device prune scans (PRICED and FIRST)."""
    if not len(res):
        return float("inf")
    m = (res["flags"] & (priced | first)) == (priced | first)
    return float(res["cost"][m].min()) if m.any() else float("inf")


def batch_slice(k: int, rank: int, world: int) -> tuple[int, int]:
    """The contiguous slice [lo, hi) of a k-parent batch rank `rank` expands."""
    return rank * k // world, (rank + 1) * k // world


def gather_batch(session, slots: list[int], rule_ids: list[int], pp, ex: OwnerExchange, expand=None) -> np.ndarray:
    """A batch expansion split over the ranks (frontier.outer_search with `exchange=`).

    Rank r expands the contiguous slice `batch_slice(len(slots), r, world)` of the batch (every
    rank holds every parent's record).  The device alpha-prune flags of a slice are recomputed
    from the minimum over the step's best and the candidates of all earlier slices (an
    exclusive scan over ranks: the cross-rank form of search.py:258-267's `best` before each
    candidate).  The results are then all-gathered, with parent indices made batch-global and
    the touched-signature ids translated into this rank's interning (ranks intern in their own
    order), so every rank holds the batch exactly as one GPU would have produced it.
    """
    from . import _native as N

    expand = expand or (lambda sl: session.expand(sl, rule_ids, pp, insert_visited=False))
    lo, hi = batch_slice(len(slots), ex.rank, ex.world)
    res = expand(slots[lo:hi]).copy() if hi > lo else np.empty(0, dtype=N.CAND_DTYPE)
    if pp.alpha > 0.0 and ex.world > 1:
        carry = ex.exclusive_min(_eligible_min(res, N.F_PRICED, N.F_FIRST), pp.best)
        if hi > lo and carry != pp.best:
            res = session.reprune(carry, pp.alpha).copy()
    res["parent"] += lo
    touched = sorted({int(x) for x in res["touched_sig"].ravel().tolist()} - {0xFFFFFFFF})
    sigs = {sid: (session.sig_list[sid], session.sig_out[sid]) for sid in touched}
    parts = ex.all_gather_object((res, sigs))
    out = []
    added = False
    for r, (part, psigs) in enumerate(parts):
        part = part.copy()
        if r != ex.rank and psigs:
            remap = {}
            for sid, (sig, out0) in psigs.items():
                before = len(session.sig_list)
                remap[sid] = session.intern_sig(sig, out0)
                added = added or len(session.sig_list) != before
            ts = part["touched_sig"]
            for i in range(ts.shape[0]):
                for k in range(ts.shape[1]):
                    v = int(ts[i, k])
                    if v != 0xFFFFFFFF:
                        ts[i, k] = remap[v]
        out.append(part)
    if added:
        session.commit()
    return np.concatenate(out) if out else np.empty(0, dtype=N.CAND_DTYPE)
