"""ctypes binding of libef200.so (the C ABI in include/ef200.h).

The library is built in-tree by `build.py` (nvcc, sm_100a).  There is no CPU
fallback anywhere in this package: if the library or a CUDA device is missing,
`lib()` raises NativeUnavailable and every GPU entry point fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeUnavailable

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EF_LIB") or os.path.join(HERE, "libef200.so")  # EF_LIB: an alternative build (experiments)

EF_OK = 0
EF_NEED_RESOLVE = 1

# flags of ef_cand_result (ef200.h)
F_FIRST, F_VISITED, F_CAPPED, F_PRICED, F_MISSING, F_INCOMPLETE, F_BEST, F_ENQUEUE, F_PFIRST = (
    1, 2, 4, 8, 16, 32, 64, 128, 256)

# weight-set derivations
D_MERGE, D_SLICE_LO, D_SLICE_HI, D_FOLD = 1, 2, 3, 4


class SigDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("rank", C.c_int32), ("in_", C.c_int32 * 4), ("out", C.c_int32 * 4),
                ("oc", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("sh", C.c_int32), ("sw", C.c_int32),
                ("ph", C.c_int32), ("pw", C.c_int32), ("act", C.c_int32),
                ("axis", C.c_int32), ("nsizes", C.c_int32), ("s0", C.c_int32), ("s1", C.c_int32)]

    def key(self) -> tuple:
        return (self.kind, self.rank, tuple(self.in_), tuple(self.out), self.oc, self.kh, self.kw, self.sh,
                self.sw, self.ph, self.pw, self.act, self.axis, self.nsizes, self.s0, self.s1)


class Geometry(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in (
        "cap_nodes", "cap_refs", "cap_outs", "record_bytes", "off_nid", "off_sig", "off_aux", "off_nin",
        "off_inoff", "off_topo", "off_refs", "off_outs", "off_keys", "off_alg", "off_sperm", "off_skeys",
        "off_srank")]


class PriceParams(C.Structure):
    _fields_ = [("kind", C.c_int32), ("d", C.c_int32), ("use_inner", C.c_int32), ("node_cap", C.c_int32),
                ("w", C.c_double), ("ct", C.c_double), ("ce", C.c_double), ("cp", C.c_double),
                ("t_ref", C.c_double), ("e_ref", C.c_double), ("p_ref", C.c_double),
                ("best", C.c_double), ("alpha", C.c_double), ("naive_sum", C.c_int32), ("per_parent", C.c_int32)]


class CandResult(C.Structure):
    _fields_ = [("hash", C.c_uint64), ("cost", C.c_double), ("time_ms", C.c_double), ("energy", C.c_double),
                ("evals", C.c_int64), ("sweeps", C.c_int32), ("n_compute", C.c_int32),
                ("flags", C.c_uint32), ("parent", C.c_uint32), ("rule", C.c_uint32),
                ("site_a", C.c_uint32), ("site_b", C.c_uint32), ("touched_sig", C.c_uint32 * 2),
                ("n_nodes", C.c_uint32)]


import numpy as _np

# numpy view of ef_cand_result (same layout; checked against ctypes at import)
CAND_DTYPE = _np.dtype([("hash", "<u8"), ("cost", "<f8"), ("time_ms", "<f8"), ("energy", "<f8"),
                        ("evals", "<i8"), ("sweeps", "<i4"), ("n_compute", "<i4"), ("flags", "<u4"),
                        ("parent", "<u4"), ("rule", "<u4"), ("site_a", "<u4"), ("site_b", "<u4"),
                        ("touched_sig", "<u4", (2,)), ("n_nodes", "<u4")])
assert CAND_DTYPE.itemsize == C.sizeof(CandResult)

_P = C.c_void_p
_U32P = C.POINTER(C.c_uint32)
_I32P = C.POINTER(C.c_int32)
_U64P = C.POINTER(C.c_uint64)
_DP = C.POINTER(C.c_double)

_PROTOS = {
    "ef_create": (_P, [C.c_int]),
    "ef_destroy": (None, [_P]),
    "ef_error": (C.c_char_p, [_P]),
    "ef_device_count": (C.c_int, []),
    "ef_sig_put": (C.c_int, [_P, C.c_uint32, C.POINTER(SigDesc), C.c_char_p, C.c_uint32, C.c_int]),
    "ef_sig_costs": (C.c_int, [_P, C.c_uint32, C.c_uint32, _I32P, _DP, _DP]),
    "ef_name_put": (C.c_int, [_P, C.c_uint32, C.c_char_p, C.c_uint32]),
    "ef_wset_put": (C.c_int, [_P, C.c_uint32, C.c_int32, C.c_int32, _DP, C.c_uint64, _DP, C.c_uint64,
                              C.c_char_p, C.c_uint32, C.c_char_p, C.c_uint32]),
    "ef_wset_derive": (C.c_int, [_P, C.c_uint32, C.c_int32, C.c_uint32, C.c_uint32, C.c_int32,
                                 C.c_char_p, C.c_uint32, C.c_char_p, C.c_uint32]),
    "ef_wset_read": (C.c_int, [_P, C.c_uint32, _DP, _U64P, _DP, _U64P]),
    "ef_wset_digest": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_uint8)]),
    "ef_tables_commit": (C.c_int, [_P]),
    "ef_set_geometry": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_char_p, C.c_uint32,
                                  C.POINTER(Geometry)]),
    "ef_record_alloc": (C.c_int, [_P, _U32P]),
    "ef_record_free": (C.c_int, [_P, C.c_uint32]),
    "ef_records_alloc": (C.c_int, [_P, C.c_uint32, _U32P]),
    "ef_records_free": (C.c_int, [_P, _U32P, C.c_uint32]),
    "ef_record_write": (C.c_int, [_P, C.c_uint32, C.c_void_p, C.c_uint64]),
    "ef_record_read": (C.c_int, [_P, C.c_uint32, C.c_void_p, C.c_uint64]),
    "ef_records_write": (C.c_int, [_P, _U32P, C.c_uint32, C.c_void_p, C.c_uint64, C.c_uint64]),
    "ef_host_alloc": (C.c_void_p, [C.c_uint64]),
    "ef_host_free": (None, [C.c_void_p]),
    "ef_hash_records": (C.c_int, [_P, _U32P, C.c_uint32, _U64P]),
    "ef_price_records": (C.c_int, [_P, _U32P, C.c_uint32, C.POINTER(PriceParams), C.POINTER(CandResult)]),
    "ef_visited_reset": (C.c_int, [_P, C.c_uint64]),
    "ef_visited_insert": (C.c_int, [_P, _U64P, C.c_uint32]),
    "ef_visited_count": (C.c_int, [_P, _U64P]),
    "ef_visited_capacity": (C.c_int, [_P, _U64P]),
    "ef_expand": (C.c_int, [_P, _U32P, C.c_uint32, _I32P, C.c_uint32, C.POINTER(PriceParams), C.c_int, _U32P]),
    "ef_pending": (C.c_int, [_P, C.POINTER(SigDesc), C.c_uint32, _U32P, _I32P, C.c_uint32, _U32P]),
    "ef_results": (C.c_int, [_P, C.c_void_p, C.c_uint32]),
    "ef_results_async": (C.c_int, [_P, C.c_void_p, C.c_uint32]),
    "ef_results_wait": (C.c_int, [_P]),
    "ef_keep": (C.c_int, [_P, _U32P, C.c_uint32, _U32P]),
    "ef_materialise": (C.c_int, [_P, _U32P, C.c_uint32, C.POINTER(C.c_int32), C.c_uint32, _U32P, _U32P,
                                 C.c_uint32, _U32P]),
    "ef_last_timing": (C.c_int, [_P, C.POINTER(C.c_float), C.c_uint32]),
    "ef_last_stats": (C.c_int, [_P, _U64P, C.c_uint32]),
    "ef_records_write_packed": (C.c_int, [_P, _U32P, C.c_uint32, C.c_void_p, _U64P, C.c_uint64]),
    "ef_records_write_packed_async": (C.c_int, [_P, _U32P, C.c_uint32, C.c_void_p, _U64P, C.c_uint64]),
    "ef_upload_fence": (C.c_int, [_P]),
    "ef_b2b_peak": (C.c_int, [_P, C.POINTER(C.c_double)]),
    "ef_expand_hashes": (C.c_int, [_P, _U32P, C.c_uint32, _I32P, C.c_uint32, _U32P]),
    "ef_route_owners": (C.c_int, [_P, C.c_uint32, C.c_uint64, C.c_void_p, _U32P]),
    "ef_owner_mark": (C.c_int, [_P, C.c_void_p, C.c_uint32, C.c_void_p, C.c_int]),
    "ef_expand_finish": (C.c_int, [_P, C.c_void_p, C.POINTER(PriceParams)]),
    "ef_expand_hashes_spec": (C.c_int, [_P, _U32P, C.c_uint32, _I32P, C.c_uint32, C.POINTER(PriceParams), _U32P]),
    "ef_route_owners_padded": (C.c_int, [_P, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]),
    "ef_owner_mark_padded": (C.c_int, [_P, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_int]),
    "ef_expand_finish_padded": (C.c_int, [_P, C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(PriceParams)]),
    "ef_stream": (C.c_int, [_P, C.POINTER(C.c_void_p)]),
    "ef_commit_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "ef_check_division": (C.c_int, [_P, C.POINTER(C.c_double), C.c_uint32, C.c_uint64, C.c_uint64,
                                    C.POINTER(C.c_uint64)]),
    "ef_reprune": (C.c_int, [_P, C.c_double, C.c_double]),
}

EXPORTED = tuple(_PROTOS)

_LIB = None


def load_library(path: str = LIB_PATH):
    """Load the shared library and bind every prototype (no device needed)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} is missing: run `python build.py` (nvcc, sm_100a)")
        lib = C.CDLL(path)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def lib():
    """The library, after checking a CUDA device is visible."""
    L = load_library()
    if L.ef_device_count() < 1:
        raise NativeUnavailable("no CUDA device visible: the B200 path has no CPU fallback")
    return L


class NativeError(RuntimeError):
    pass


def check(ctx, rc: int, what: str) -> int:
    if rc < 0:
        msg = _LIB.ef_error(ctx).decode(errors="replace") if ctx else ""
        raise NativeError(f"{what} failed ({rc}): {msg}")
    return rc


def u32_array(values):
    """uint32 buffer for a C call (numpy-backed: no per-element ctypes conversion)."""
    arr = _np.ascontiguousarray(_np.asarray(values if len(values) else [0], dtype=_np.uint32))
    return arr.ctypes.data_as(_U32P)  # the pointer keeps a reference to `arr`


def i32_array(values):
    arr = _np.ascontiguousarray(_np.asarray(values if len(values) else [0], dtype=_np.int32))
    return arr.ctypes.data_as(_I32P)
