"""The pricing's division by a normalisation reference (div_pre: RN(1/y) once, then two FMA
residual corrections, Markstein) is the correctly rounded IEEE quotient the reference's float
`/` computes (cost.py:284-296): checked bit for bit against the device's IEEE division on
2^27 random dividends per divisor -- the refs of the golden searches, divisors with all-ones /
all-zeros significands, powers of two and random ones."""

import ctypes as C
import random
import struct

import pytest

import paper_2005_05837_b200 as ef
from paper_2005_05837_b200 import zoo
from paper_2005_05837_b200.device import DeviceSession

pytestmark = pytest.mark.gpu


def _f(bits):
    return struct.unpack("<d", struct.pack("<Q", bits))[0]


def test_division_by_reference_is_correctly_rounded():
    ys = []
    for model in ("inception_v3", "resnet50"):
        g = zoo.generate(model, 0)
        db = ef.CostDatabase()
        ef.ensure_profiled(g, db, ef.SyntheticProfiler(0))
        ys += [float(v) for v in ef.normalization_refs(g, db)]
    ys += [1.0, 2.0, 0.5, 3.0, 0.1, 1e-3, 7e5, _f(0x3FFFFFFFFFFFFFFF), _f(0x3FF0000000000001), _f(0x43EFFFFFFFFFFFFF)]
    rng = random.Random(7)
    for _ in range(22):
        e = rng.randrange(1023 - 400, 1023 + 400)
        ys.append(_f((e << 52) | rng.getrandbits(52)) * rng.choice((1.0, -1.0)))
    s = DeviceSession(0)
    try:
        arr = (C.c_double * len(ys))(*ys)
        bad = C.c_uint64(0)
        s._check(s.L.ef_check_division(s.ctx, arr, len(ys), 1 << 27, 12345, C.byref(bad)), "ef_check_division")
        assert bad.value == 0
    finally:
        s.close()
