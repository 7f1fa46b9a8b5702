"""Hash-owner sharding protocol and the sharded search's batch gather over world_size-2 gloo on CPU.

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
    """Per-rank work of the device session, restated on host tensors (the padded protocol)."""

    def __init__(self, hashes, visited_shard):
        self.hashes = [int(h) for h in hashes]
        self.visited = set(visited_shard)

    def expand_hashes(self, slots, rule_ids, pp=None):
        return len(self.hashes)

    def route_owners_padded(self, world, base, cap, send, counts):
        assert cap >= len(self.hashes)
        cnt = [0] * world
        self.perm = {}
        for c, h in enumerate(self.hashes):
            o = owner_of(h, world)
            pos = o * cap + cnt[o]
            cnt[o] += 1
            send[2 * pos] = torch.tensor(np.array([h], dtype=np.uint64).view(np.int64))[0]
            send[2 * pos + 1] = base + c
            self.perm[pos] = c
        counts[:] = torch.tensor(cnt, dtype=torch.int32)

    def owner_mark_padded(self, recv, rcounts, world, cap, verdict, insert_visited):
        pairs = recv.numpy().view(np.uint64).reshape(-1, 2)
        rc = rcounts.tolist()
        valid = [i for i in range(world * cap) if i % cap < rc[i // cap]]
        first = {}
        for i in valid:
            h, o = int(pairs[i, 0]), int(pairs[i, 1])
            first[h] = min(first.get(h, o), o)
        verdict.zero_()
        for i in valid:
            h, o = int(pairs[i, 0]), int(pairs[i, 1])
            verdict[i] = (F_FIRST if first[h] == o else 0) | (F_VISITED if h in self.visited else 0)
        if insert_visited:
            for i in valid:
                if int(verdict[i]) == F_FIRST:
                    self.visited.add(int(pairs[i, 0]))

    def expand_finish_padded(self, back, world, cap, pp, n):
        flags = [0] * n
        for pos, c in self.perm.items():
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


# ---- the sharded search's batch gather (shard.gather_batch) --------------------------------

F_PRICED, F_BEST, F_ENQUEUE = 8, 64, 128


def _batch(seed, k):
    """A batch of k parents' candidates as one GPU returns them: (parent, flags, cost, touched)."""
    rng = np.random.default_rng(seed)
    from paper_2005_05837_b200 import _native as N

    n = int(rng.integers(3 * k, 6 * k))
    res = np.zeros(n, dtype=N.CAND_DTYPE)
    res["parent"] = np.sort(rng.integers(0, k, n))
    res["hash"] = rng.integers(0, 2**63, n, dtype=np.int64).astype(np.uint64)
    res["cost"] = rng.uniform(10.0, 20.0, n)
    res["flags"] = np.where(rng.random(n) < 0.8, F_FIRST | F_PRICED, F_PRICED)
    res["touched_sig"] = 0xFFFFFFFF
    res["touched_sig"][:, 0] = rng.integers(0, 6, n)  # signature by name "sig<k>"
    return res


def _prune(res, best, alpha):
    """k_prune_*: BEST / ENQUEUE from the minimum before each eligible candidate."""
    out = res.copy()
    prev = best
    for i in range(len(out)):
        f = int(out["flags"][i])
        if (f & (F_PRICED | F_FIRST)) == (F_PRICED | F_FIRST):
            c = float(out["cost"][i])
            f &= ~(F_BEST | F_ENQUEUE)
            f |= (F_BEST if c < prev else 0) | (F_ENQUEUE if c < alpha * prev else 0)
            out["flags"][i] = f
            prev = c if c < prev else prev
    return out


class FakeSession:
    """What gather_batch uses of a DeviceSession: the expansion of a slice of the batch, the
    re-prune, and signature interning (each rank interns in its own order)."""

    def __init__(self, full, rank, best, alpha):
        self.full, self.best, self.alpha = full, best, alpha
        self.sig_list, self.sig_out, self.by_text = [], [], {}
        self.committed = 0
        order = list(range(6)) if rank == 0 else list(range(5, -1, -1))  # rank-specific interning
        for k in order:
            self.intern_sig(f"sig{k}", (k,))
        self.last = None

    def intern_sig(self, sig, out0):
        if sig not in self.by_text:
            self.by_text[sig] = len(self.sig_list)
            self.sig_list.append(sig)
            self.sig_out.append(out0)
        return self.by_text[sig]

    def commit(self):
        self.committed += 1

    def expand(self, parents):
        lo, hi = parents[0], parents[-1] + 1
        part = self.full[(self.full["parent"] >= lo) & (self.full["parent"] < hi)].copy()
        part["parent"] -= lo
        ts = part["touched_sig"]
        ts[:, 0] = [self.by_text[f"sig{int(v)}"] for v in ts[:, 0]]  # this rank's ids
        self.last = _prune(part, self.best, self.alpha)
        return self.last

    def reprune(self, best, alpha):
        self.last = _prune(self.last, best, alpha)
        return self.last


class PP:
    def __init__(self, best, alpha):
        self.best, self.alpha = best, alpha


def _gather_worker(rank, world, port, q, seed, k):
    from paper_2005_05837_b200.shard import gather_batch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _batch(seed, k)
        sess = FakeSession(full, rank, 15.0, 1.05)
        got = gather_batch(sess, list(range(k)), [0], PP(15.0, 1.05), OwnerExchange(), expand=sess.expand)
        names = [[sess.sig_list[int(v)] for v in row if int(v) != 0xFFFFFFFF] for row in got["touched_sig"]]
        q.put((rank, got["parent"].tolist(), got["flags"].tolist(), got["cost"].tolist(), names))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed,k", [(5, 7), (6, 2), (7, 1)])
def test_gather_batch_equals_single_gpu_batch(seed, k):
    """Every rank ends with the batch one GPU produces: global parent indices, prune flags
    with the best carried across ranks, signature ids in its own interning."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q, seed, k)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, par, flags, cost, names = q.get(timeout=120)
        got[rank] = (par, flags, cost, names)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _prune(_batch(seed, k), 15.0, 1.05)
    want = (full["parent"].tolist(), full["flags"].tolist(), full["cost"].tolist(),
            [[f"sig{int(v)}"] for v in full["touched_sig"][:, 0]])
    assert got[0] == want and got[1] == want
