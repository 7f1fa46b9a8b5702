"""Graphs the search runs on.

* The reference's bundled instances (reference models.py): the three-conv
  micro-benchmark with its measured cost table, toy graphs, the alpha-valley
  and coordinated-move instances, and the seeded random graphs used by the
  reference's test-suite.  These consume the seeded numpy stream in the same
  order as the reference, so a seed names the same graph in both packages
  (tests/golden pins this).
* The paper's evaluation models at their real layer shapes, batch 1, random
  float64 weights: SqueezeNet 1.1, ResNet-50 (v1: stride on the first 1x1 of
  each bottleneck, so each stage's projection and first 1x1 are mergeable
  parallel convolutions), Inception-v3 and a NASNet-A-style cell stack
  (separable convolutions expressed as conv pairs: the IR has no grouped conv).
  Fully-connected heads are 1x1 convolutions over the pooled 1x1 map (the IR
  has no flatten).
* `random_dag`: synthetic conv/matmul DAGs of 1k-20k operators for the
  candidates/sec sweep.
"""

from __future__ import annotations

import numpy as np

from .costmodel import CostDatabase, CostRecord
from .ir import EdgeRef, Graph, GraphBuilder, Node, NodeSignature, signatures, validate


def _conv_w(rng, oc: int, ic: int, kh: int, kw: int) -> np.ndarray:
    return rng.standard_normal((oc, ic, kh, kw)) / np.sqrt(ic * kh * kw)


# ---------------------------------------------------------------------------
# reference instances (reference models.py)
# ---------------------------------------------------------------------------

# Table 1 of the paper: (time ms, power W, energy J/1000) per algorithm label
MICROBENCH_COSTS = {
    "conv1": {"a": (0.0195, 144.5, 2.81), "b": (0.0209, 84.0, 1.75)},
    "conv2": {"a": (0.00941, 58.0, 0.545), "b": (0.0175, 47.0, 0.822)},
    "conv3": {"a": (0.165, 190.8, 31.4), "b": (0.146, 116.0, 16.9), "c": (0.083, 144.0, 11.9)},
}


def microbench_graph() -> Graph:
    rng = np.random.default_rng(12)
    b = GraphBuilder()
    x = b.input("x", (1, 3, 16, 16))
    c1 = b.conv2d(x, _conv_w(rng, 8, 3, 3, 3), padding=(1, 1))
    c2 = b.conv2d(c1, _conv_w(rng, 8, 8, 1, 1))
    c3 = b.conv2d(c2, _conv_w(rng, 16, 8, 3, 3), stride=(2, 2), padding=(1, 1))
    b.output(c3)
    return b.build()


def microbench_signatures() -> dict[str, str]:
    g = microbench_graph()
    sigs = signatures(g)
    return {f"conv{i + 1}": sigs[n.id].text for i, n in enumerate(g.compute_nodes())}


def microbench_database() -> CostDatabase:
    """Table 1 as a database; power stored as energy/time so energies are exact."""
    sig_of = microbench_signatures()
    db = CostDatabase()
    for row, algs in MICROBENCH_COSTS.items():
        for label, (t, _p, e) in sorted(algs.items()):
            db.add(sig_of[row], ord(label) - ord("a"), CostRecord(time_ms=t, power_w=e / t))
    return db


def chain_graph(n: int, seed: int = 0) -> Graph:
    if n < 1:
        raise ValueError("chain length must be >= 1")
    rng = np.random.default_rng(seed)
    b = GraphBuilder()
    cur = b.input("x", (1, 3, 8, 8))
    ch = 3
    for _ in range(n):
        cur = b.relu(b.conv2d(cur, _conv_w(rng, 4, ch, 3, 3), padding=(1, 1)))
        ch = 4
    b.output(cur)
    return b.build()


def toy_squeeze(seed: int = 0) -> Graph:
    rng = np.random.default_rng(seed)
    b = GraphBuilder()
    x = b.input("x", (1, 3, 16, 16))
    sq = b.conv2d(x, _conv_w(rng, 4, 3, 1, 1), has_activation=True)
    e1 = b.relu(b.conv2d(sq, _conv_w(rng, 6, 4, 3, 3), padding=(1, 1)))
    e2 = b.relu(b.conv2d(sq, _conv_w(rng, 6, 4, 3, 3), padding=(1, 1)))
    e3 = b.relu(b.conv2d(sq, _conv_w(rng, 4, 4, 1, 1)))
    head = b.relu(b.conv2d(b.concat([e1, e2, e3], axis=1), _conv_w(rng, 8, 16, 3, 3), padding=(1, 1)))
    b.output(b.maxpool(head, kernel=(2, 2), stride=(2, 2)))
    return b.build()


def toy_resnet(seed: int = 0) -> Graph:
    rng = np.random.default_rng(seed)
    b = GraphBuilder()
    x = b.input("x", (1, 3, 8, 8))
    stem = b.conv2d(x, _conv_w(rng, 4, 3, 3, 3), padding=(1, 1))
    c1 = b.conv2d(stem, _conv_w(rng, 4, 4, 3, 3), padding=(1, 1))
    r1 = b.relu(b.batchnorm(c1, rng.uniform(0.5, 1.5, 4), rng.standard_normal(4)))
    c2 = b.conv2d(r1, _conv_w(rng, 4, 4, 3, 3), padding=(1, 1))
    bn2 = b.batchnorm(c2, rng.uniform(0.5, 1.5, 4), rng.standard_normal(4))
    tail = b.identity(b.relu(b.add(stem, bn2)))
    b.output(b.avgpool(tail, kernel=(2, 2), stride=(2, 2)))
    return b.build()


def valley_instance():
    """Three-graph chain whose middle graph is the most expensive (reference models.py:131-169).

    g0 = fused conv + (conv, relu); fusing gives g1 (two fused convs), merging gives g2.
    energy(g1)=5 > energy(g0)=4.5 > energy(g2)=2, so alpha=1 stops at g0 and alpha=1.5 reaches g2.
    """
    from .rewrite import default_rules

    rng = np.random.default_rng(7)
    b = GraphBuilder()
    x = b.input("x", (1, 2, 4, 4))
    fused = b.conv2d(x, _conv_w(rng, 2, 2, 3, 3), padding=(1, 1), has_activation=True)
    after = b.relu(b.conv2d(x, _conv_w(rng, 2, 2, 3, 3), padding=(1, 1)))
    b.output(fused, after)
    g0 = b.build()

    def conv(act: bool, oc: int) -> str:
        return NodeSignature("conv2d", ((1, 2, 4, 4),), (("has_activation", act), ("kernel", (3, 3)),
                                                         ("out_channels", oc), ("padding", (1, 1)),
                                                         ("stride", (1, 1)))).text

    db = CostDatabase()
    db.add(conv(True, 2), 0, CostRecord(1.0, 2.5))
    db.add(conv(False, 2), 0, CostRecord(1.0, 1.0))
    db.add(NodeSignature("relu", ((1, 2, 4, 4),), ()).text, 0, CostRecord(1.0, 1.0))
    db.add(conv(True, 4), 0, CostRecord(1.0, 1.5))
    db.add(NodeSignature("split", ((1, 4, 4, 4),), (("axis", 1), ("sizes", (2, 2)))).text, 0, CostRecord(1.0, 0.5))
    rules = [r for r in default_rules() if r.name in ("fuse-conv-relu", "merge-parallel-convs")]
    return g0, db, rules


def coordinated_witness():
    """Two nodes where only a joint move improves product(0.5) (reference models.py:172-198)."""
    b = GraphBuilder()
    x = b.input("x", (1, 2, 4, 4))
    r = b.relu(x)
    i = b.identity(r)
    b.output(i)
    g = b.build()
    sigs = signatures(g)
    db = CostDatabase()
    db.add(sigs[r.node].text, 0, CostRecord(5.0, 9.95 / 5.0))
    db.add(sigs[r.node].text, 1, CostRecord(995.0, 0.0501 / 995.0))
    db.add(sigs[i.node].text, 0, CostRecord(5.0, 0.05 / 5.0))
    db.add(sigs[i.node].text, 1, CostRecord(5.2, 0.031 / 5.2))
    return g, db


def random_graph(seed: int, ops: int | None = None, max_ops: int = 8) -> Graph:
    """Seeded random graph biased toward rewrite sites.

    Consumes the numpy stream exactly as reference models.py:205-333 does, so
    the same seed yields the same graph (including weights) in both packages.
    """
    rng = np.random.default_rng(seed)
    target = int(ops) if ops is not None else int(rng.integers(3, max_ops + 1))
    b = GraphBuilder()
    c0 = int(rng.choice([2, 3]))
    hw = int(rng.choice([4, 6, 8]))
    live: list[tuple[EdgeRef, tuple]] = [(b.input("x", (1, c0, hw, hw)), (1, c0, hw, hw))]
    made = 0
    while made < target:
        left = target - made
        menu = [("conv", 0.30), ("relu", 0.12), ("identity", 0.08), ("batchnorm", 0.12)]
        if left >= 2:
            menu += [("conv_relu", 0.16), ("parallel_convs", 0.14), ("conv_bn", 0.10)]
        if len(live) >= 2:
            menu += [("add", 0.10), ("concat", 0.06)]
        if any(s[1] >= 2 for _, s in live):
            menu += [("split", 0.04)]
        if any(s[2] >= 2 and s[3] >= 2 for _, s in live):
            menu += [("pool", 0.06)]
        names = [m for m, _ in menu]
        wts = np.asarray([w for _, w in menu])
        move = str(rng.choice(names, p=wts / sum(w for _, w in menu)))
        if move in ("conv", "conv_relu", "conv_bn", "parallel_convs"):
            idx = int(rng.integers(len(live)))
            ref, (bn, c, h, w) = live[idx]
            k = int(rng.choice([1, 3]))
            k = 1 if k > min(h, w) else k
            pad = int(rng.integers(0, 2)) if k == 3 else 0
            oc = int(rng.integers(2, 6))
            act = bool(rng.integers(0, 2)) if move == "conv" else False
            live.pop(idx)
            out = b.conv2d(ref, _conv_w(rng, oc, c, k, k), padding=(pad, pad), has_activation=act)
            shp = (bn, oc, h + 2 * pad - k + 1, w + 2 * pad - k + 1)
            if move == "conv_relu":
                out = b.relu(out)
                made += 1
            elif move == "conv_bn":
                out = b.batchnorm(out, rng.uniform(0.5, 1.5, oc), rng.standard_normal(oc))
                made += 1
            elif move == "parallel_convs":
                twin = b.conv2d(ref, _conv_w(rng, oc, c, k, k), padding=(pad, pad), has_activation=act)
                live.append((twin, shp))
                made += 1
            live.append((out, shp))
            made += 1
        elif move in ("relu", "identity"):
            ref, s = live.pop(int(rng.integers(len(live))))
            live.append((b.relu(ref) if move == "relu" else b.identity(ref), s))
            made += 1
        elif move == "batchnorm":
            ref, s = live.pop(int(rng.integers(len(live))))
            live.append((b.batchnorm(ref, rng.uniform(0.5, 1.5, s[1]), rng.standard_normal(s[1])), s))
            made += 1
        elif move in ("add", "concat"):
            groups: dict[tuple, list[int]] = {}
            for i, (_, s) in enumerate(live):
                groups.setdefault(s if move == "add" else (s[0], s[2], s[3]), []).append(i)
            cands = [v for v in groups.values() if len(v) >= 2]
            if not cands:
                continue
            pick = cands[int(rng.integers(len(cands)))]
            rj, sj = live.pop(pick[1])
            ri, si = live.pop(pick[0])
            if move == "add":
                live.append((b.add(ri, rj), sj))
            else:
                live.append((b.concat([ri, rj], axis=1), (si[0], si[1] + sj[1], si[2], si[3])))
            made += 1
        elif move == "split":
            opts = [i for i, (_, s) in enumerate(live) if s[1] >= 2]
            ref, (bn, c, h, w) = live.pop(opts[int(rng.integers(len(opts)))])
            c1 = int(rng.integers(1, c))
            p0, p1 = b.split(ref, (c1, c - c1), axis=1)
            live += [(p0, (bn, c1, h, w)), (p1, (bn, c - c1, h, w))]
            made += 1
        elif move == "pool":
            opts = [i for i, (_, s) in enumerate(live) if s[2] >= 2 and s[3] >= 2]
            ref, (bn, c, h, w) = live.pop(opts[int(rng.integers(len(opts)))])
            pool = b.maxpool if rng.integers(0, 2) else b.avgpool
            live.append((pool(ref, kernel=(2, 2), stride=(2, 2)), (bn, c, h // 2, w // 2)))
            made += 1
    b.output(*[ref for ref, _ in live])
    return b.build()


# ---------------------------------------------------------------------------
# the paper's evaluation models (batch 1, real layer shapes, random weights)
# ---------------------------------------------------------------------------

class _Net:
    """Builder helper tracking channel counts; conv weights are He-scaled normals."""

    def __init__(self, seed: int, name: str, dims):
        self.rng = np.random.default_rng(seed)
        self.b = GraphBuilder()
        self.x = self.b.input(name, dims)

    def conv(self, x, cin, cout, k, stride=1, pad=0, bias=False, act=False):
        kh, kw = (k, k) if isinstance(k, int) else k
        sh, sw = (stride, stride) if isinstance(stride, int) else stride
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        w = _conv_w(self.rng, cout, cin, kh, kw)
        bias_v = self.rng.standard_normal(cout) * 0.01 if bias else None
        return self.b.conv2d(x, w, bias=bias_v, stride=(sh, sw), padding=(ph, pw), has_activation=act)

    def bn(self, x, c):
        return self.b.batchnorm(x, self.rng.uniform(0.5, 1.5, c), self.rng.standard_normal(c) * 0.1)

    def cbr(self, x, cin, cout, k, stride=1, pad=0):
        """conv -> batchnorm -> relu (torchvision BasicConv2d)."""
        return self.b.relu(self.bn(self.conv(x, cin, cout, k, stride, pad), cout))


def squeezenet(seed: int = 0, hw: int = 224) -> Graph:
    """SqueezeNet 1.1: conv/relu stem, 8 fire modules, conv classifier, global pool."""
    n = _Net(seed, "x", (1, 3, hw, hw))
    b = n.b

    def fire(x, cin, sq, e1, e3):
        s = b.relu(n.conv(x, cin, sq, 1, bias=True))
        a = b.relu(n.conv(s, sq, e1, 1, bias=True))
        c = b.relu(n.conv(s, sq, e3, 3, pad=1, bias=True))
        return b.concat([a, c], axis=1), e1 + e3

    x = b.relu(n.conv(n.x, 3, 64, 3, stride=2, bias=True))
    x = b.maxpool(x, (3, 3), (2, 2))
    x, c = fire(x, 64, 16, 64, 64)
    x, c = fire(x, c, 16, 64, 64)
    x = b.maxpool(x, (3, 3), (2, 2))
    x, c = fire(x, c, 32, 128, 128)
    x, c = fire(x, c, 32, 128, 128)
    x = b.maxpool(x, (3, 3), (2, 2))
    for sq, e in ((48, 192), (48, 192), (64, 256), (64, 256)):
        x, c = fire(x, c, sq, e, e)
    x = b.relu(n.conv(x, c, 1000, 1, bias=True))
    spatial = ((((hw - 3) // 2 + 1 - 3) // 2 + 1 - 3) // 2 + 1 - 3) // 2 + 1
    b.output(b.avgpool(x, (spatial, spatial), (1, 1)))
    return b.build()


def resnet50(seed: int = 0, hw: int = 224) -> Graph:
    """ResNet-50 v1 (stride on the first 1x1 of a bottleneck), BN after every conv."""
    n = _Net(seed, "x", (1, 3, hw, hw))
    b = n.b
    x = n.cbr(n.x, 3, 64, 7, stride=2, pad=3)
    x = b.maxpool(x, (3, 3), (2, 2), (1, 1))
    cin = 64
    size = (hw + 6 - 7) // 2 + 1
    size = (size + 2 - 3) // 2 + 1
    for width, blocks, stride in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
        for i in range(blocks):
            s = stride if i == 0 else 1
            if i == 0:
                short = n.bn(n.conv(x, cin, 4 * width, 1, stride=s), 4 * width)
            else:
                short = x
            y = n.cbr(x, cin, width, 1, stride=s)
            y = n.cbr(y, width, width, 3, pad=1)
            y = n.bn(n.conv(y, width, 4 * width, 1), 4 * width)
            x = b.relu(b.add(y, short))
            cin = 4 * width
        size = (size - 1) // stride + 1 if stride > 1 else size
    x = b.avgpool(x, (size, size), (1, 1))
    b.output(n.conv(x, cin, 1000, 1, bias=True))
    return b.build()


def inception_v3(seed: int = 0, hw: int = 299) -> Graph:
    """Inception-v3 (torchvision layout, no auxiliary head)."""
    n = _Net(seed, "x", (1, 3, hw, hw))
    b = n.b
    cbr = n.cbr
    x = cbr(n.x, 3, 32, 3, stride=2)
    x = cbr(x, 32, 32, 3)
    x = cbr(x, 32, 64, 3, pad=1)
    x = b.maxpool(x, (3, 3), (2, 2))
    x = cbr(x, 64, 80, 1)
    x = cbr(x, 80, 192, 3)
    x = b.maxpool(x, (3, 3), (2, 2))
    c = 192

    def block_a(x, c, pool):
        b1 = cbr(x, c, 64, 1)
        b5 = cbr(cbr(x, c, 48, 1), 48, 64, 5, pad=2)
        b3 = cbr(cbr(cbr(x, c, 64, 1), 64, 96, 3, pad=1), 96, 96, 3, pad=1)
        bp = cbr(b.avgpool(x, (3, 3), (1, 1), (1, 1)), c, pool, 1)
        return b.concat([b1, b5, b3, bp], axis=1), 224 + pool

    def block_b(x, c):
        b3 = cbr(x, c, 384, 3, stride=2)
        bd = cbr(cbr(cbr(x, c, 64, 1), 64, 96, 3, pad=1), 96, 96, 3, stride=2)
        return b.concat([b3, bd, b.maxpool(x, (3, 3), (2, 2))], axis=1), 384 + 96 + c

    def block_c(x, c, c7):
        b1 = cbr(x, c, 192, 1)
        b7 = cbr(cbr(cbr(x, c, c7, 1), c7, c7, (1, 7), pad=(0, 3)), c7, 192, (7, 1), pad=(3, 0))
        d = cbr(x, c, c7, 1)
        d = cbr(d, c7, c7, (7, 1), pad=(3, 0))
        d = cbr(d, c7, c7, (1, 7), pad=(0, 3))
        d = cbr(d, c7, c7, (7, 1), pad=(3, 0))
        d = cbr(d, c7, 192, (1, 7), pad=(0, 3))
        bp = cbr(b.avgpool(x, (3, 3), (1, 1), (1, 1)), c, 192, 1)
        return b.concat([b1, b7, d, bp], axis=1), 768

    def block_d(x, c):
        b3 = cbr(cbr(x, c, 192, 1), 192, 320, 3, stride=2)
        b7 = cbr(cbr(cbr(cbr(x, c, 192, 1), 192, 192, (1, 7), pad=(0, 3)), 192, 192, (7, 1), pad=(3, 0)),
                 192, 192, 3, stride=2)
        return b.concat([b3, b7, b.maxpool(x, (3, 3), (2, 2))], axis=1), 320 + 192 + c

    def block_e(x, c):
        b1 = cbr(x, c, 320, 1)
        t = cbr(x, c, 384, 1)
        b3 = b.concat([cbr(t, 384, 384, (1, 3), pad=(0, 1)), cbr(t, 384, 384, (3, 1), pad=(1, 0))], axis=1)
        d = cbr(cbr(x, c, 448, 1), 448, 384, 3, pad=1)
        bd = b.concat([cbr(d, 384, 384, (1, 3), pad=(0, 1)), cbr(d, 384, 384, (3, 1), pad=(1, 0))], axis=1)
        bp = cbr(b.avgpool(x, (3, 3), (1, 1), (1, 1)), c, 192, 1)
        return b.concat([b1, b3, bd, bp], axis=1), 2048

    for pool in (32, 64, 64):
        x, c = block_a(x, c, pool)
    x, c = block_b(x, c)
    for c7 in (128, 160, 160, 192):
        x, c = block_c(x, c, c7)
    x, c = block_d(x, c)
    x, c = block_e(x, c)
    x, c = block_e(x, c)
    size = 8 if hw == 299 else max(1, hw // 37)
    x = b.avgpool(x, (size, size), (1, 1))
    b.output(n.conv(x, c, 1000, 1, bias=True))
    return b.build()


def nasnet_a(seed: int = 0, hw: int = 224, filters: int = 44, cells: int = 4) -> Graph:
    """NASNet-A-style stack: `cells` normal cells per stage, 2 reduction cells.

    Separable convolutions are written relu -> conv kxk -> bn -> relu -> conv
    kxk -> bn (no grouped conv in the IR); the relu of a cell input is shared by
    the branches reading it, so same-kernel branches are parallel convs.
    """
    n = _Net(seed, "x", (1, 3, hw, hw))
    b = n.b

    def sep(x, c, k, stride=1):
        y = n.bn(n.conv(x, c, c, k, stride=stride, pad=k // 2), c)
        return n.bn(n.conv(b.relu(y), c, c, k, pad=k // 2), c)

    def adjust(x, cin, cout, stride=1):
        return n.bn(n.conv(b.relu(x), cin, cout, 1, stride=stride), cout)

    def normal(h, hp, ch, chp, f, hp_stride=1):
        a = adjust(h, ch, f)
        p = adjust(hp, chp, f, hp_stride)
        ra, rp = b.relu(a), b.relu(p)
        b0 = b.add(sep(ra, f, 3), b.identity(a))
        b1 = b.add(sep(rp, f, 3), sep(ra, f, 5))
        b2 = b.add(b.avgpool(a, (3, 3), (1, 1), (1, 1)), b.identity(p))
        b3 = b.add(b.avgpool(p, (3, 3), (1, 1), (1, 1)), b.avgpool(p, (3, 3), (1, 1), (1, 1)))
        b4 = b.add(sep(rp, f, 5), sep(rp, f, 3))
        return b.concat([p, b0, b1, b2, b3, b4], axis=1), 6 * f

    def reduction(h, hp, ch, chp, f, hp_stride=1):
        a = adjust(h, ch, f)
        p = adjust(hp, chp, f, hp_stride)
        ra, rp = b.relu(a), b.relu(p)
        b0 = b.add(sep(ra, f, 5, 2), sep(rp, f, 7, 2))
        b1 = b.add(b.maxpool(a, (3, 3), (2, 2), (1, 1)), sep(rp, f, 7, 2))
        b2 = b.add(b.avgpool(a, (3, 3), (2, 2), (1, 1)), sep(rp, f, 5, 2))
        b3 = b.add(b.avgpool(b0, (3, 3), (1, 1), (1, 1)), b.identity(b1))
        b4 = b.add(sep(b.relu(b0), f, 3), b.maxpool(a, (3, 3), (2, 2), (1, 1)))
        return b.concat([b1, b2, b3, b4], axis=1), 4 * f

    stem = n.bn(n.conv(n.x, 3, 32, 3, stride=2, pad=1), 32)
    h, ch, hp, chp = stem, 32, stem, 32
    f = filters
    pending_stride = 1
    for stage in range(3):
        if stage > 0:
            f *= 2
            nh, nch = reduction(h, hp, ch, chp, f, pending_stride)
            hp, chp, h, ch = h, ch, nh, nch
            pending_stride = 2  # hp is still at the previous resolution
        for _ in range(cells):
            nh, nch = normal(h, hp, ch, chp, f, pending_stride)
            hp, chp, h, ch = h, ch, nh, nch
            pending_stride = 1
    x = b.relu(h)
    size = (hw + 2 - 3) // 2 + 1
    for _ in range(2):
        size = (size + 2 - 3) // 2 + 1
    x = b.avgpool(x, (size, size), (1, 1))
    b.output(n.conv(x, ch, 1000, 1, bias=True))
    return b.build()


def random_dag(n_ops: int, seed: int = 0, channels=(2, 8), hw: int = 8, max_live: int = 24) -> Graph:
    """Synthetic conv/matmul DAG with about `n_ops` operators, dense in rewrite sites.

    Two inputs: an image tensor feeding conv / relu / batchnorm / identity /
    add / concat / split / pool moves (the reference's random-graph move set,
    scaled up), and a feature vector feeding a matmul/relu/add chain.  The live
    set is bounded so concats stay narrow and the DAG stays wide instead of deep.
    """
    rng = np.random.default_rng(seed)
    b = GraphBuilder()
    c_lo, c_hi = channels
    img: list[tuple[EdgeRef, tuple]] = [(b.input("x", (1, c_lo, hw, hw)), (1, c_lo, hw, hw))]
    feat_dim = 16
    vec: list[EdgeRef] = [b.input("y", (1, feat_dim))]
    retired: list[EdgeRef] = []
    made = 0
    moves = ["conv", "conv_relu", "conv_bn", "parallel", "relu", "identity", "bn", "add", "concat", "split",
             "pool", "matmul"]
    probs = np.array([0.16, 0.14, 0.12, 0.12, 0.06, 0.05, 0.05, 0.10, 0.04, 0.04, 0.02, 0.10])
    probs = probs / probs.sum()
    while made < n_ops:
        move = moves[int(rng.choice(len(moves), p=probs))]
        if move == "matmul":
            i = int(rng.integers(len(vec)))
            y = b.matmul(vec[i], rng.standard_normal((feat_dim, feat_dim)) / 4.0)
            made += 1
            if rng.random() < 0.5:
                y = b.relu(y)
                made += 1
            if len(vec) >= 2 and rng.random() < 0.3:
                j = int(rng.integers(len(vec)))
                y = b.add(y, vec.pop(j))
                made += 1
            vec.append(y)
            if len(vec) > 4:
                vec.pop(0)
            continue
        idx = int(rng.integers(len(img)))
        ref, (bn, c, h, w) = img[idx]
        if move in ("conv", "conv_relu", "conv_bn", "parallel"):
            k = 3 if (rng.random() < 0.5 and min(h, w) >= 3) else 1
            pad = 1 if k == 3 else 0
            oc = int(rng.integers(c_lo, c_hi + 1))
            act = move == "conv" and rng.random() < 0.3
            out = b.conv2d(ref, _conv_w(rng, oc, c, k, k), padding=(pad, pad), has_activation=act)
            shp = (bn, oc, h, w)
            made += 1
            if move == "conv_relu":
                out = b.relu(out)
                made += 1
            elif move == "conv_bn":
                out = b.batchnorm(out, rng.uniform(0.5, 1.5, oc), rng.standard_normal(oc))
                made += 1
            elif move == "parallel":
                for _ in range(int(rng.integers(1, 3))):
                    oc2 = int(rng.integers(c_lo, c_hi + 1))
                    twin = b.conv2d(ref, _conv_w(rng, oc2, c, k, k), padding=(pad, pad))
                    img.append((twin, (bn, oc2, h, w)))
                    made += 1
            img.append((out, shp))
            if rng.random() < 0.5:
                img.pop(idx)
        elif move in ("relu", "identity", "bn"):
            if move == "relu":
                out = b.relu(ref)
            elif move == "identity":
                out = b.identity(ref)
            else:
                out = b.batchnorm(ref, rng.uniform(0.5, 1.5, c), rng.standard_normal(c))
            img[idx] = (out, (bn, c, h, w))
            made += 1
        elif move in ("add", "concat"):
            same = [i for i, (_, s) in enumerate(img) if i != idx and (s == (bn, c, h, w) if move == "add"
                                                                      else s[2:] == (h, w))]
            if not same:
                continue
            j = same[int(rng.integers(len(same)))]
            rj, sj = img[j]
            if move == "add":
                out, shp = b.add(ref, rj), (bn, c, h, w)
            else:
                if c + sj[1] > 4 * c_hi:
                    continue
                out, shp = b.concat([ref, rj], axis=1), (bn, c + sj[1], h, w)
            for k in sorted((idx, j), reverse=True):
                img.pop(k)
            img.append((out, shp))
            made += 1
        elif move == "split" and c >= 2:
            c1 = int(rng.integers(1, c))
            p0, p1 = b.split(ref, (c1, c - c1), axis=1)
            img.pop(idx)
            img += [(p0, (bn, c1, h, w)), (p1, (bn, c - c1, h, w))]
            made += 1
        elif move == "pool" and h >= 4:
            out = b.maxpool(ref, (2, 2), (2, 2)) if rng.random() < 0.5 else b.avgpool(ref, (2, 2), (2, 2))
            img[idx] = (out, (bn, c, h // 2, w // 2))
            made += 1
        if len(img) > max_live:
            retired.append(img.pop(0)[0])
    outs = retired + [r for r, _ in img] + vec
    b.output(*outs)
    g = b.build(check=False)
    # drop dead nodes (edges popped by the live-set bound): keep what reaches an output
    live = set()
    todo = [r.node for r in g.outputs]
    while todo:
        v = todo.pop()
        if v not in live:
            live.add(v)
            todo.extend(r.node for r in g.nodes[v].inputs)
    return _compact(g, live)


def _compact(g: Graph, keep: set[int]) -> Graph:
    """Renumber kept nodes 0..n-1 in id order (ids stay topological)."""
    ids = sorted(keep)
    new = {old: i for i, old in enumerate(ids)}
    b_nodes = {}
    for old in ids:
        v = g.nodes[old]
        b_nodes[new[old]] = Node(new[old], v.kind, tuple(EdgeRef(new[r.node], r.port) for r in v.inputs),
                                 v.params, v.weights)
    out = Graph(b_nodes, g.inputs, tuple(EdgeRef(new[r.node], r.port) for r in g.outputs))
    bad = validate(out)
    if bad:
        raise ValueError("random_dag produced an invalid graph: " + "; ".join(bad[:3]))
    return out


MODELS = {
    "squeezenet": squeezenet, "resnet50": resnet50, "inception_v3": inception_v3, "nasnet_a": nasnet_a,
    "toy-squeeze": toy_squeeze, "toy-resnet": toy_resnet, "microbench": lambda seed=0: microbench_graph(),
}


def generate(name: str, seed: int = 0) -> Graph:
    if name in MODELS:
        return MODELS[name](seed)
    if name.startswith("chain:"):
        return chain_graph(int(name.split(":", 1)[1]), seed)
    if name.startswith("dag:"):
        return random_dag(int(name.split(":", 1)[1]), seed)
    raise ValueError(f"unknown model name {name!r}")
