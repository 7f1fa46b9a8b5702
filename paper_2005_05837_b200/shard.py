"""Hash-owner sharding of the frontier step over ranks (one process per GPU).

The reference deduplicates every generated graph against one visited set and
keeps the first graph per hash in (rule, site) order (rules.py:79-88,
search.py:245-251).  Across ranks the frontier is split by parent, so the
global candidate order is rank-major, and deduplication is owned by hash: rank
`hash % world` receives every (hash, global order) pair it owns, decides first
occurrence (smallest global order) and membership in its shard of the visited
set, and sends the verdicts back.  The result on every rank is exactly the
single-rank result for the concatenated frontier (tests/test_shard.py).

`OwnerExchange` is the collective layer (torch.distributed: NCCL over NVLink on
the GPUs, gloo in the CPU tests); the per-rank work is the device session's
`expand_hashes` / `route_owners` / `owner_mark` / `expand_finish` (libef200).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def owner_of(h: int, world: int) -> int:
    """Rank owning a candidate hash (same rule as csrc/ef_step.cuh owner_of)."""
    return h % world


class OwnerExchange:
    """All-to-all of (hash, order) pairs to their owners and of verdicts back."""

    def __init__(self, group=None, device: torch.device | None = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device if device is not None else torch.device("cpu")
        self._bufs: dict[str, torch.Tensor] = {}

    def buffer(self, name: str, numel: int, dtype) -> torch.Tensor:
        """A reusable device buffer of at least `numel` elements (no allocator traffic per step)."""
        buf = self._bufs.get(name)
        if buf is None or buf.numel() < numel or buf.dtype != dtype:
            buf = torch.empty(max(numel, 1024), dtype=dtype, device=self.device)
            self._bufs[name] = buf
        return buf[:numel]

    def _sync(self):
        if self.device.type == "cuda":
            torch.cuda.current_stream(self.device).synchronize()

    def order_base(self) -> int:
        """Global order of this rank's first candidate: rank-major order needs no exchange,
        (rank << 40) + index is monotone in (rank, index)."""
        return self.rank << 40

    def to_owners(self, send: torch.Tensor, counts: list[int]) -> tuple[torch.Tensor, list[int]]:
        """`send` holds sum(counts) pairs grouped by owner; returns the pairs this rank owns
        (grouped by source rank) and how many came from each source."""
        c = torch.tensor(counts, dtype=torch.int64, device=self.device)
        rc = torch.empty_like(c)
        dist.all_to_all_single(rc, c, group=self.group)
        recv_counts = [int(x) for x in rc.tolist()]
        recv = torch.empty(2 * sum(recv_counts), dtype=torch.int64, device=self.device)
        dist.all_to_all_single(recv, send[: 2 * sum(counts)].contiguous(), [2 * x for x in recv_counts],
                               [2 * x for x in counts], group=self.group)
        self._sync()
        return recv, recv_counts

    def back(self, verdict: torch.Tensor, recv_counts: list[int], counts: list[int]) -> torch.Tensor:
        """Owner verdicts (in receive order) back to the senders (in send order)."""
        out = torch.empty(max(sum(counts), 1), dtype=torch.int32, device=self.device)
        dist.all_to_all_single(out[: sum(counts)], verdict[: sum(recv_counts)].contiguous(), counts, recv_counts,
                               group=self.group)
        self._sync()
        return out

    def min(self, x: float) -> float:
        """Global best cost for the alpha rule (all-reduce MIN)."""
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return float(t.item())

    def sum(self, x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, group=self.group)
        return float(t.item())


def sharded_expand(session, slots: list[int], rule_ids: list[int], pp, ex: OwnerExchange,
                   insert_visited: bool = False, phases: dict | None = None):
    """One frontier step over the parents of this rank with hash-owner deduplication.

    Returns this rank's candidate results (the layout of `DeviceSession.expand`);
    flags FIRST / VISITED are global, costs are those of this rank's survivors.
    `phases`, when given, accumulates host wall seconds per phase.
    """
    import time

    t = [time.perf_counter()]

    def mark():
        t.append(time.perf_counter())

    n = session.expand_hashes(slots, rule_ids)
    mark()
    base = ex.order_base()
    send = ex.buffer("send", max(2 * n, 2), torch.int64)
    counts = session.route_owners(ex.world, base, send)
    mark()
    recv, recv_counts = ex.to_owners(send, counts)
    mark()
    verdict = ex.buffer("verdict", max(recv.numel() // 2, 1), torch.int32)
    if recv.numel():
        session.owner_mark(recv, verdict, insert_visited)
    mark()
    back = ex.back(verdict, recv_counts, counts)
    mark()
    out = session.expand_finish(back, pp, n)
    mark()
    if phases is not None:
        phases["calls"] = phases.get("calls", 0) + 1
        for name, a, b in zip(("hash", "route", "to_owners", "mark", "back", "finish"), t, t[1:]):
            phases[name] = phases.get(name, 0.0) + (b - a)
    return out
