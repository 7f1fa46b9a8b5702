"""Hash-owner sharding protocol over world_size-2 gloo on CPU.

Each rank holds a slice of a frontier's candidate hashes (rank-major global
order, with duplicates inside and across ranks) and a shard of a visited set.
The product's exchange layer (paper_2005_05837_b200.shard: OwnerExchange +
sharded_expand) routes (hash, order) pairs to their owner ranks and the
verdicts back; the per-rank device work is stood in for by `HostRank`, a plain
restatement of what ef_route_owners / ef_owner_mark / ef_expand_finish compute.
The verdicts must equal single-process deduplication of the concatenated
frontier: first occurrence in global order (rules.py:79-88) and visited
membership (search.py:247-251), with first occurrences inserted afterwards.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_05837_b200.shard import OwnerExchange, owner_of, sharded_expand

F_FIRST, F_VISITED = 1, 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class HostRank:
    """Per-rank work of the device session, restated on host tensors."""

    def __init__(self, hashes, visited_shard):
        self.hashes = [int(h) for h in hashes]
        self.visited = set(visited_shard)

    def expand_hashes(self, slots, rule_ids):
        return len(self.hashes)

    def route_owners(self, world, base, send):
        order = sorted(range(len(self.hashes)), key=lambda c: owner_of(self.hashes[c], world))
        counts = [0] * world
        pairs = []
        for c in order:
            counts[owner_of(self.hashes[c], world)] += 1
            pairs += [self.hashes[c], base + c]
        self.perm = order
        if pairs:
            send[: len(pairs)] = torch.from_numpy(np.array(pairs, dtype=np.uint64).view(np.int64))
        return counts

    def owner_mark(self, recv, verdict, insert_visited):
        pairs = recv.numpy().view(np.uint64).reshape(-1, 2)
        first = {}
        for h, o in pairs.tolist():
            first[h] = min(first.get(h, o), o)
        for i, (h, o) in enumerate(pairs.tolist()):
            verdict[i] = (F_FIRST if first[h] == o else 0) | (F_VISITED if h in self.visited else 0)
        if insert_visited:
            for i, (h, _) in enumerate(pairs.tolist()):
                if int(verdict[i]) == F_FIRST:
                    self.visited.add(h)

    def expand_finish(self, back, pp, n):
        flags = [0] * n
        for pos, c in enumerate(self.perm):
            flags[c] = int(back[pos])
        return flags


def _frontier(seed):
    rng = np.random.default_rng(seed)
    pool = rng.integers(0, 2**64, size=300, dtype=np.uint64)
    pool[0] = 0  # hash 0 is a legal digest
    cands = rng.choice(pool, size=1000)  # duplicates inside and across ranks
    visited = set(int(x) for x in rng.choice(pool, size=60, replace=False))
    return [int(x) for x in cands], visited


def _expected(cands, visited):
    seen, out = set(), []
    for h in cands:
        f = 0
        if h not in seen:
            f |= F_FIRST
            seen.add(h)
        if h in visited:
            f |= F_VISITED
        out.append(f)
    return out


def _worker(rank, world, port, q, seed, splits):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cands, visited = _frontier(seed)
        lo, hi = splits[rank], splits[rank + 1]
        mine = HostRank(cands[lo:hi], {h for h in visited if owner_of(h, world) == rank})
        ex = OwnerExchange()
        flags = sharded_expand(mine, [], [], None, ex, insert_visited=True)
        # second step over the same frontier: everything is now visited somewhere
        flags2 = sharded_expand(mine, [], [], None, ex, insert_visited=False)
        best = ex.min(float(rank + 3))
        q.put((rank, flags, flags2, best))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,splits", [(1, [0, 400, 1000]), (2, [0, 1000, 1000]), (3, [0, 0, 1000])])
def test_sharded_dedup_equals_single_rank(seed, splits):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, seed, splits)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        rank, flags, flags2, best = q.get(timeout=120)
        got[rank] = (flags, flags2, best)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cands, visited = _frontier(seed)
    want = _expected(cands, visited)
    assert got[0][0] + got[1][0] == want
    # after inserting the first occurrences every candidate is visited
    seen_after = visited | set(cands)
    want2 = [(F_FIRST if i == cands.index(h) else 0) | F_VISITED for i, h in enumerate(cands)]
    assert got[0][1] + got[1][1] == want2 and all(h in seen_after for h in cands)
    assert got[0][2] == got[1][2] == 3.0
