"""paper_2301_00806_b200 -- B200-native enumeration of weak pseudo-manifolds.

Python mirror of the reference's enumeration API for this one path
(``plseeds``, /root/reference/proj/include/plseeds), bound to the C-ABI
library ``libwpm_b200.so`` (include/wpm_b200.h).  Names and argument meaning
follow the reference:

    idcm_orbits(n, p)            charmap.hpp:212-281
    charmap_of_dcm(rows, p)      charmap.hpp:155-204
    matroid_universe(rows, p)    pipeline.hpp:33-35 (kernel 1 on the GPU)
    cyclic_facet_bound(n)        affine_property.hpp:35-45
    ubt_property(n, M)           affine_property.hpp:49-54
    SearchJob                    search.hpp:46-55
    enumerate_wpm(job)           search.hpp:141-258 (kernels 2-3 + canonical sort)
    write_complexes(...)         complex_io.hpp:21-39

Errors mirror the reference's exception types (errors.hpp): ``PurityError``,
``CapExceededError`` and ``ValueError`` (std::invalid_argument).  There is
no CPU fallback: if the CUDA library is missing the import fails, and every
compute call raises ``RuntimeError`` when no B200 is present.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# WPM_DEBUG_LIB=debug|traps|<variant> selects a diagnostic build of the same sources
_VARIANT = os.environ.get("WPM_DEBUG_LIB", "")
LIB_PATH = os.path.join(_HERE, {"": "libwpm_b200.so", "debug": "libwpm_b200_dbg.so"}.get(
    _VARIANT, f"libwpm_b200_{_VARIANT}.so"))

WPM_OK = 0
WPM_EINTERNAL = 1
WPM_EINVAL = 2
WPM_EINFEASIBLE = 3
WPM_ECAP = 5
WPM_CAP_NONE = -1
WPM_CAP_UBT = -2
WPM_MAX_M = 16


class PurityError(RuntimeError):
    """errors.hpp:10-13 (purity_error)."""


class CapExceededError(RuntimeError):
    """errors.hpp:28-31 (cap_exceeded_error)."""


class WpmError(RuntimeError):
    """Internal / CUDA failure of the B200 path (status 1)."""


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(the B200 path has no CPU fallback)"
    )

_lib = ctypes.CDLL(LIB_PATH)

_i32, _i64, _u32p, _u64p, _i32p = (
    ctypes.c_int32,
    ctypes.c_int64,
    ctypes.POINTER(ctypes.c_uint32),
    ctypes.POINTER(ctypes.c_uint64),
    ctypes.POINTER(ctypes.c_int32),
)


class _Result(ctypes.Structure):
    _fields_ = [
        ("num_maps", ctypes.c_int32),
        ("words", ctypes.c_int32),
        ("total", ctypes.c_int64),
        ("counts", ctypes.POINTER(ctypes.c_int64)),
        ("offsets", ctypes.POINTER(ctypes.c_int64)),
        ("bits", ctypes.POINTER(ctypes.c_uint64)),
        ("nodes", ctypes.c_int64),
        ("duplicates", ctypes.c_int64),
        ("ms_search", ctypes.c_double),
        ("ms_sort", ctypes.c_double),
        ("tasks", ctypes.c_int64),
        ("ms_total", ctypes.c_double),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
    ]


class _Job(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("num_facets", ctypes.c_int32),
        ("facets", _u64p),
        ("facet_cap", ctypes.c_int64),
        ("required", _i32p),
        ("num_required", ctypes.c_int32),
        ("forbidden", _i32p),
        ("num_forbidden", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("shard_index", ctypes.c_int32),
        ("shard_count", ctypes.c_int32),
        ("progress", ctypes.c_void_p),
        ("progress_user", ctypes.c_void_p),
        ("devices", _i32p),
        ("num_devices", ctypes.c_int32),
    ]


# progress(done, total, user) -- SearchJob::progress (search.hpp:54)
_PROGRESS = ctypes.CFUNCTYPE(None, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p)


class _Complexes(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("count", ctypes.c_int64),
        ("offsets", ctypes.POINTER(ctypes.c_int64)),
        ("facets", ctypes.POINTER(ctypes.c_uint64)),
        ("words", ctypes.c_int32),
        ("bits", ctypes.POINTER(ctypes.c_uint64)),
        ("line7", ctypes.c_int64),
        ("line13", ctypes.c_int64),
        ("ms_union", ctypes.c_double),
        ("ms_filter", ctypes.c_double),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("line15", ctypes.c_int64),
        ("ms_canon", ctypes.c_double),
        ("ms_dedupe", ctypes.c_double),
    ]


_ResultP = ctypes.POINTER(_Result)
_ComplexesP = ctypes.POINTER(_Complexes)
_PlanP = ctypes.c_void_p

_SIGS = {
    "wpm_last_error": (ctypes.c_char_p, []),
    "wpm_device_count": (ctypes.c_int, []),
    "wpm_cyclic_facet_bound": (_i64, [_i32]),
    "wpm_idcm_orbits": (_i32, [_i32, _i32, _u32p, _i32]),
    "wpm_charmap_of_dcm": (_i32, [_i32, _i32, _u32p, _u32p]),
    "wpm_plan_create_orbits": (ctypes.c_int, [_i32, _i32, _i64, _i32, ctypes.POINTER(_PlanP)]),
    "wpm_plan_create_charmaps": (ctypes.c_int, [_i32, _i32, _i32, _u32p, _i64, _i32, ctypes.POINTER(_PlanP)]),
    "wpm_plan_create_universes": (
        ctypes.c_int,
        [_i32, _i32, _i32, _i32p, _u64p, _i64, _i32p, _i32, _i32p, _i32, _i32, ctypes.POINTER(_PlanP)],
    ),
    "wpm_plan_num_maps": (ctypes.c_int, [_PlanP]),
    "wpm_plan_universe": (_i32, [_PlanP, _i32, _u64p, _i32]),
    "wpm_plan_incidence": (_i32, [_PlanP, _i32, _u64p, _i32, _i32p, _i32p]),
    "wpm_plan_run": (ctypes.c_int, [_PlanP, _i32, _i32, ctypes.POINTER(_i64)]),
    "wpm_plan_fetch": (ctypes.c_int, [_PlanP, ctypes.POINTER(_ResultP)]),
    "wpm_plan_stats": (
        ctypes.c_int,
        [_PlanP, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64),
         ctypes.POINTER(_i64)],
    ),
    "wpm_plan_timing": (ctypes.c_int, [_PlanP, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i32)]),
    "wpm_plan_device_result": (
        ctypes.c_int,
        [_PlanP, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_i64),
         ctypes.POINTER(_i32)],
    ),
    "wpm_canonical_sort_device": (
        ctypes.c_int,
        [_i32, ctypes.c_void_p, ctypes.c_void_p, _i64, _i32, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(_i64),
         ctypes.c_void_p],
    ),
    "wpm_int_peak": (ctypes.c_int, [_i32, ctypes.POINTER(ctypes.c_double)]),
    "wpm_plan_destroy": (None, [_PlanP]),
    "wpm_enumerate": (ctypes.c_int, [ctypes.POINTER(_Job), ctypes.POINTER(_ResultP)]),
    "wpm_enumerate_orbits": (ctypes.c_int, [_i32, _i32, _i64, _i32, ctypes.POINTER(_ResultP)]),
    "wpm_result_free": (None, [_ResultP]),
    "wpm_write_cplx": (_i64, [_ResultP, _i32, _i32, _i32, _u64p, ctypes.c_char_p, _i64]),
    "wpm_plan_line13": (ctypes.c_int, [_PlanP, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "wpm_plan_line13_timing": (ctypes.c_int, [_PlanP, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(ctypes.c_double)]),
    "wpm_plan_fetch_complexes": (ctypes.c_int, [_PlanP, _i32, ctypes.POINTER(_ComplexesP)]),
    "wpm_complexes_free": (None, [_ComplexesP]),
    "wpm_write_complexes": (_i64, [_ComplexesP, ctypes.c_char_p, _i64]),
    "wpm_seed_flags": (ctypes.c_int, [_i32, _i32, _i64, ctypes.POINTER(_i64), _u64p, _i32,
                                      ctypes.POINTER(ctypes.c_uint8)]),
    "wpm_pipeline_line13": (ctypes.c_int, [_i32, _i32, _i64, _i32, ctypes.POINTER(_ComplexesP)]),
    "wpm_plan_line15": (ctypes.c_int, [_PlanP, ctypes.POINTER(_i64)]),
    "wpm_plan_line15_stats": (ctypes.c_int, [_PlanP, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                                             ctypes.POINTER(_i64)]),
    "wpm_plan_set_node_budget": (ctypes.c_int, [_PlanP, _i64]),
    "wpm_plan_truncated": (ctypes.c_int, [_PlanP]),
    "wpm_plan_line15_costs": (_i64, [_PlanP, ctypes.POINTER(_i64), _i64]),
    "wpm_canonical_forms": (ctypes.c_int, [_i32, _i32, _i64, ctypes.POINTER(_i64), _u64p, _i32, _u64p,
                                           ctypes.POINTER(ctypes.c_int8)]),
    "wpm_pipeline_line15": (ctypes.c_int, [_i32, _i32, _i64, _i32, ctypes.POINTER(_ComplexesP)]),
    "wpm_plan_run_kernel_basis": (ctypes.c_int, [_PlanP, ctypes.c_uint64, ctypes.POINTER(_i64)]),
    "wpm_plan_kernel_basis_stats": (ctypes.c_int, [_PlanP, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                                   ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "wpm_plan_set_devices": (ctypes.c_int, [_PlanP, _i32p, _i32]),
    "wpm_plan_create_orbits_multi": (ctypes.c_int, [_i32, _i32, _i64, _i32p, _i32, ctypes.POINTER(_PlanP)]),
    "wpm_plan_device_stats": (ctypes.c_int, [_PlanP, _i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)]),
    "wpm_plan_set_split": (ctypes.c_int, [_PlanP, _i32]),
    "wpm_plan_set_progress": (ctypes.c_int, [_PlanP, ctypes.c_void_p, ctypes.c_void_p]),
    "wpm_plan_split": (ctypes.c_int, [_PlanP, _i32, _i32, _i32, _i64, ctypes.POINTER(_i64)]),
    "wpm_plan_frontier": (ctypes.c_int, [_PlanP, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(_i64),
                                         ctypes.POINTER(_i32)]),
    "wpm_plan_load_frontier": (ctypes.c_int, [_PlanP, ctypes.c_void_p, _i64]),
    "wpm_claim_counter_create": (ctypes.c_int, [_i32, ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]),
    "wpm_claim_counter_open": (ctypes.c_int, [_i32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "wpm_claim_counter_reset": (ctypes.c_int, [_i32, ctypes.c_void_p]),
    "wpm_claim_counter_close": (ctypes.c_int, [_i32, ctypes.c_void_p, _i32]),
    "wpm_plan_run_claim": (ctypes.c_int, [_PlanP, ctypes.c_void_p, ctypes.POINTER(_i64)]),
    "wpm_plan_set_root_stats": (ctypes.c_int, [_PlanP, _i32]),
    "wpm_plan_root_nodes": (_i64, [_PlanP, ctypes.POINTER(_i64), _i64, ctypes.POINTER(_i64)]),
    "wpm_plan_run_kernel_basis_prefix": (ctypes.c_int, [_PlanP, _i32, _i32, _i32p, ctypes.c_uint64,
                                                        ctypes.POINTER(_i64)]),
    "wpm_plan_space_blocks": (_i32, [_PlanP, _i32, _i32p, _i32]),
    "wpm_plan_verify": (ctypes.c_int, [_PlanP, _i32, ctypes.POINTER(_i64), ctypes.POINTER(_i64), _u64p]),
    "wpm_plan_combination_space": (ctypes.c_int, [_PlanP, _i32, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(_i32),
                                                  ctypes.POINTER(_i32)]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED_SYMBOLS = tuple(_SIGS)


def _check(rc: int) -> None:
    if rc == WPM_OK:
        return
    msg = (_lib.wpm_last_error() or b"").decode()
    if rc == WPM_ECAP:
        raise CapExceededError(msg)
    if rc == WPM_EINVAL:
        if "purity" in msg or "empty facet set" in msg:
            raise PurityError(msg)
        raise ValueError(msg)
    if rc == WPM_EINFEASIBLE:
        raise ValueError(msg)
    raise WpmError(msg or f"status {rc}")


def _u32(a) -> "ctypes.Array":
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return arr, arr.ctypes.data_as(_u32p)


def _u64(a):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.uint64))
    return arr, arr.ctypes.data_as(_u64p)


def _i32a(a):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return arr, arr.ctypes.data_as(_i32p)


# ----------------------------------------------------------------- host side

def device_count() -> int:
    return int(_lib.wpm_device_count())


def int_peak(device: int = 0) -> float:
    """Measured INT32 issue peak (lane-ops/s) of `device` (roofline denominator)."""
    v = ctypes.c_double()
    _check(_lib.wpm_int_peak(device, ctypes.byref(v)))
    return v.value


def enumerate_orbits(n: int, p: int = 4, facet_cap: int = WPM_CAP_UBT, device: int = 0) -> "Result":
    """One-shot Algorithm-2 loop for one n (wpm_enumerate_orbits)."""
    rp = _ResultP()
    _check(_lib.wpm_enumerate_orbits(n, p, facet_cap, device, ctypes.byref(rp)))
    return Result(rp)


def canonical_sort_device(device: int, bits32_ptr: int, map_ptr: int, count: int, words32: int, out_bits_ptr: int,
                          out_map_ptr: int, stream: int = 0) -> int:
    """Canonical sort of device-resident rows (e.g. shards gathered over NCCL); returns duplicates."""
    d = _i64()
    _check(_lib.wpm_canonical_sort_device(device, bits32_ptr, map_ptr, count, words32, out_bits_ptr, out_map_ptr,
                                          ctypes.byref(d), stream or None))
    return int(d.value)


def claim_counter_create(device: int = 0):
    """(device pointer, 64-byte CUDA IPC handle) of a new shared claim counter."""
    p = ctypes.c_void_p()
    h = (ctypes.c_uint8 * 64)()
    _check(_lib.wpm_claim_counter_create(device, ctypes.byref(p), h))
    return p.value, bytes(h)


def claim_counter_open(device: int, handle: bytes) -> int:
    p = ctypes.c_void_p()
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    _check(_lib.wpm_claim_counter_open(device, h, ctypes.byref(p)))
    return p.value


def claim_counter_reset(device: int, ptr: int) -> None:
    _check(_lib.wpm_claim_counter_reset(device, ptr))


def claim_counter_close(device: int, ptr: int, opened: bool) -> None:
    _check(_lib.wpm_claim_counter_close(device, ptr, 1 if opened else 0))


def cyclic_facet_bound(n: int) -> int:
    """affine_property.hpp:35-45."""
    return int(_lib.wpm_cyclic_facet_bound(n))


@dataclass
class AffineProperty:
    """affine_property.hpp:16-31 (only count caps reach the device)."""

    weights: List[int]
    constant: int

    def is_count_cap(self) -> bool:
        return all(w == -1 for w in self.weights)


def ubt_property(n: int, universe_size: int) -> AffineProperty:
    """affine_property.hpp:49-54: g(K) = cap + 1 - |K| > 0."""
    return AffineProperty([-1] * universe_size, cyclic_facet_bound(n) + 1)


@dataclass
class DualCharMatrix:
    """charmap.hpp:64-87: one p-bit row per vertex."""

    m: int
    p: int
    rows: List[int]


def idcm_orbits(n: int, p: int = 4) -> List[DualCharMatrix]:
    """charmap.hpp:212-281 (host C++ in the library)."""
    k = int(_lib.wpm_idcm_orbits(n, p, None, 0))
    if k < 0:
        _check(-k)
    m = n + p
    buf = np.zeros(k * m, dtype=np.uint32)
    _lib.wpm_idcm_orbits(n, p, buf.ctypes.data_as(_u32p), k)
    return [DualCharMatrix(m, p, [int(x) for x in buf[i * m:(i + 1) * m]]) for i in range(k)]


def charmap_of_dcm(d: DualCharMatrix) -> List[int]:
    """charmap.hpp:155-204: lambda columns (n-bit ints)."""
    rows, rp = _u32(d.rows)
    cols = np.zeros(d.m, dtype=np.uint32)
    r = int(_lib.wpm_charmap_of_dcm(d.m, d.p, rp, cols.ctypes.data_as(_u32p)))
    if r < 0:
        _check(-r)
    return [int(c) for c in cols]


# ----------------------------------------------------------------- plans

class Plan:
    """A device-resident batch of characteristic maps / universes.

    Owns the kernel-1 universes, kernel-2 incidence tables, the work queue
    and the result buffers on one GPU.  ``run()`` is the hot path (kernel 3 +
    canonical sort, inputs and outputs resident in HBM); ``fetch()`` copies
    the result to the host.
    """

    def __init__(self, handle, n: int, m: int):
        self._h = ctypes.c_void_p(handle)
        self.n = n
        self.m = m
        self.num_maps = int(_lib.wpm_plan_num_maps(self._h))

    @classmethod
    def orbits(cls, n: int, p: int = 4, facet_cap: int = WPM_CAP_UBT, device: int = 0,
               devices: Optional[Sequence[int]] = None) -> "Plan":
        """devices: one job over several GPUs (wpm_plan_create_orbits_multi)."""
        h = _PlanP()
        if devices and len(devices) > 1:
            arr, ap = _i32a(list(devices))
            _check(_lib.wpm_plan_create_orbits_multi(n, p, facet_cap, ap, len(devices), ctypes.byref(h)))
        else:
            _check(_lib.wpm_plan_create_orbits(n, p, facet_cap, device, ctypes.byref(h)))
        return cls(h.value, n, n + p)

    def set_devices(self, devices: Sequence[int]) -> None:
        arr, ap = _i32a(list(devices) or [0])
        _check(_lib.wpm_plan_set_devices(self._h, ap, len(devices)))

    def set_split(self, depth: int) -> None:
        """Split the tree below the root at this branch depth before the search (0 = off)."""
        _check(_lib.wpm_plan_set_split(self._h, depth))

    def set_progress(self, fn) -> None:
        """fn(done, total) while runs are in flight (SearchJob::progress); None = off."""
        self._progress = _PROGRESS(lambda d, t, u: fn(int(d), int(t))) if fn else None
        _check(_lib.wpm_plan_set_progress(self._h, ctypes.cast(self._progress, ctypes.c_void_p) if fn else None,
                                          None))

    def device_stats(self):
        """[(kernel-3 ms, nodes)] per device of the last multi-GPU run."""
        ms = (ctypes.c_double * 64)()
        nd = (_i64 * 64)()
        k = int(_lib.wpm_plan_device_stats(self._h, 64, ms, nd))
        return [(ms[i], int(nd[i])) for i in range(max(k, 0))]

    def set_root_stats(self, on: bool = True) -> None:
        _check(_lib.wpm_plan_set_root_stats(self._h, 1 if on else 0))

    def root_nodes(self):
        """(per-root node counts of the last run's main phase, split-phase nodes)."""
        sp = _i64()
        k = int(_lib.wpm_plan_root_nodes(self._h, None, 0, ctypes.byref(sp)))
        if k < 0:
            _check(-k)
        out = np.zeros(max(k, 1), dtype=np.int64)
        _lib.wpm_plan_root_nodes(self._h, out.ctypes.data_as(ctypes.POINTER(_i64)), k, ctypes.byref(sp))
        return out[:k], int(sp.value)

    # -- the cross-process protocol (one process per GPU, see dist.py)
    def split(self, depth: int = 0, target: int = 0, shard_index: int = 0, shard_count: int = 1) -> int:
        """Split this plan's share of the root tasks (t % shard_count ==
        shard_index) below the root (depth 0: the library's choice); returns
        the frontier record count."""
        c = _i64()
        _check(_lib.wpm_plan_split(self._h, shard_index, shard_count, depth, target, ctypes.byref(c)))
        return int(c.value)

    def frontier(self):
        """(device pointer, records, uint32 words per record) of the last split."""
        p, c, w = ctypes.c_void_p(), _i64(), _i32()
        _check(_lib.wpm_plan_frontier(self._h, ctypes.byref(p), ctypes.byref(c), ctypes.byref(w)))
        return p.value or 0, int(c.value), int(w.value)

    def load_frontier(self, ptr: int, count: int) -> None:
        _check(_lib.wpm_plan_load_frontier(self._h, ptr or None, count))

    def run_claim(self, counter: int) -> int:
        tot = _i64()
        _check(_lib.wpm_plan_run_claim(self._h, counter, ctypes.byref(tot)))
        return int(tot.value)

    @classmethod
    def charmaps(cls, n: int, m: int, cols: Sequence[Sequence[int]], facet_cap: int = WPM_CAP_UBT,
                 device: int = 0) -> "Plan":
        flat, fp = _u32([c for cs in cols for c in cs])
        h = _PlanP()
        _check(_lib.wpm_plan_create_charmaps(n, m, len(cols), fp, facet_cap, device, ctypes.byref(h)))
        return cls(h.value, n, m)

    @classmethod
    def universes(cls, m: int, n: int, universes: Sequence[Sequence[int]], facet_cap: int = WPM_CAP_NONE,
                  required: Sequence[int] = (), forbidden: Sequence[int] = (), device: int = 0) -> "Plan":
        counts, cp = _i32a([len(u) for u in universes])
        flat, fp = _u64([f for u in universes for f in u])
        req, rp = _i32a(list(required) or [0])
        forb, fbp = _i32a(list(forbidden) or [0])
        h = _PlanP()
        _check(_lib.wpm_plan_create_universes(m, n, len(universes), cp, fp, facet_cap, rp, len(required), fbp,
                                              len(forbidden), device, ctypes.byref(h)))
        return cls(h.value, n, m)

    def universe(self, i: int) -> List[int]:
        buf = np.zeros(1 << 12, dtype=np.uint64)
        M = int(_lib.wpm_plan_universe(self._h, i, buf.ctypes.data_as(_u64p), len(buf)))
        if M < 0:
            _check(-M)
        return [int(x) for x in buf[:M]]

    def incidence(self, i: int):
        """(ridges, cols[M][n], parents[N][<=8]) of map i, from kernel 2."""
        M = len(self.universe(i))
        ridges = np.zeros(1 << 13, dtype=np.uint64)
        cols = np.zeros(M * self.n, dtype=np.int32)
        par = np.zeros((1 << 13) * 8, dtype=np.int32)
        N = int(_lib.wpm_plan_incidence(self._h, i, ridges.ctypes.data_as(_u64p), len(ridges),
                                        cols.ctypes.data_as(_i32p), par.ctypes.data_as(_i32p)))
        if N < 0:
            _check(-N)
        parents = [[int(g) for g in par[r * 8:(r + 1) * 8] if g >= 0] for r in range(N)]
        return [int(x) for x in ridges[:N]], cols.reshape(M, self.n).tolist(), parents

    def run(self, shard_index: int = 0, shard_count: int = 1) -> int:
        tot = _i64()
        _check(_lib.wpm_plan_run(self._h, shard_index, shard_count, ctypes.byref(tot)))
        return int(tot.value)

    def timing(self) -> dict:
        v, w = ctypes.c_double(), _i32()
        _check(_lib.wpm_plan_timing(self._h, ctypes.byref(v), ctypes.byref(w)))
        return {"ms_total": v.value, "warps": int(w.value)}

    def device_result(self):
        """(bits32_ptr, map_ptr, count, words32) of the resident canonical result."""
        b, mp, c, w = ctypes.c_void_p(), ctypes.c_void_p(), _i64(), _i32()
        _check(_lib.wpm_plan_device_result(self._h, ctypes.byref(b), ctypes.byref(mp), ctypes.byref(c),
                                           ctypes.byref(w)))
        return b.value or 0, mp.value or 0, int(c.value), int(w.value)

    def stats(self) -> dict:
        a, b, c, d = ctypes.c_double(), ctypes.c_double(), _i64(), _i64()
        _check(_lib.wpm_plan_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(d)))
        return {"ms_search": a.value, "ms_sort": b.value, "nodes": c.value, "tasks": d.value}

    def fetch(self) -> "Result":
        rp = _ResultP()
        _check(_lib.wpm_plan_fetch(self._h, ctypes.byref(rp)))
        return Result(rp)

    def run_kernel_basis(self, candidate_cap: int = (1 << 64) - 1) -> int:
        """Algorithm 1 as the reference runs it (search.hpp:141-258): the
        reference's kernel basis on the host, EVERY combination-space leaf on
        the device (k6_odometer.cu); same result layout as run()."""
        tot = _i64()
        _check(_lib.wpm_plan_run_kernel_basis(self._h, ctypes.c_uint64(candidate_cap), ctypes.byref(tot)))
        return int(tot.value)

    def run_kernel_basis_prefix(self, map_index: int, cand: Sequence[int], candidate_cap: int = (1 << 64) - 1) -> int:
        """Algorithm 1 over one map with its first len(cand) blocks fixed to
        the given candidates (the reference's inner odometer over the rest)."""
        arr, ap = _i32a(list(cand) or [0])
        tot = _i64()
        _check(_lib.wpm_plan_run_kernel_basis_prefix(self._h, map_index, len(cand), ap, ctypes.c_uint64(candidate_cap),
                                                     ctypes.byref(tot)))
        return int(tot.value)

    def space_blocks(self, map_index: int) -> List[int]:
        """Widths of the map's combination-space blocks, widest first."""
        buf = np.zeros(4096, dtype=np.int32)
        k = int(_lib.wpm_plan_space_blocks(self._h, map_index, buf.ctypes.data_as(_i32p), len(buf)))
        if k < 0:
            _check(-k)
        return [int(x) for x in buf[:k]]

    def verify(self, reach: bool = False, coords: bool = False):
        """Kernel 8 on the last run: (unsound rows, unreachable rows or -1,
        coordinates per row or None)."""
        a, b = _i64(), _i64()
        out = np.zeros(max(self.stats_total(), 1), dtype=np.uint64) if coords else None
        _check(_lib.wpm_plan_verify(self._h, 1 if reach else 0, ctypes.byref(a), ctypes.byref(b),
                                    out.ctypes.data_as(_u64p) if coords else None))
        return int(a.value), int(b.value), (out[: self.stats_total()] if coords else None)

    def stats_total(self) -> int:
        return int(self.device_result()[2])

    def kernel_basis_stats(self) -> dict:
        a, b, c, d = _i64(), _i64(), ctypes.c_double(), ctypes.c_double()
        _check(_lib.wpm_plan_kernel_basis_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                                ctypes.byref(d)))
        return {"leaves": int(a.value), "checked": int(b.value), "ms_prep": c.value, "ms_leaves": d.value}

    def combination_space(self, i: int) -> dict:
        sp, s, nb = ctypes.c_uint64(), _i32(), _i32()
        _check(_lib.wpm_plan_combination_space(self._h, i, ctypes.byref(sp), ctypes.byref(s), ctypes.byref(nb)))
        return {"space": int(sp.value), "s": int(s.value), "blocks": int(nb.value)}

    def line13(self) -> Tuple[int, int]:
        """Algorithm 2 lines 7 and 13 (pipeline.hpp:58-89) on the last run, on
        the device: (union size, survivors of the support + seedness filters)."""
        a, b = _i64(), _i64()
        _check(_lib.wpm_plan_line13(self._h, ctypes.byref(a), ctypes.byref(b)))
        return int(a.value), int(b.value)

    def line13_timing(self) -> dict:
        a, b = ctypes.c_double(), ctypes.c_double()
        _check(_lib.wpm_plan_line13_timing(self._h, ctypes.byref(a), ctypes.byref(b)))
        return {"ms_union": a.value, "ms_filter": b.value}

    def set_node_budget(self, budget: int) -> None:
        """Stop later runs after `budget` search nodes (0 = enumerate all);
        a stopped run has .truncated() True (stress runs, BASELINE configs[4])."""
        _check(_lib.wpm_plan_set_node_budget(self._h, int(budget)))

    def truncated(self) -> bool:
        return bool(_lib.wpm_plan_truncated(self._h))

    def line15(self) -> int:
        """Algorithm 2 line 15 (pipeline.hpp:91-103) on the last line-13
        result, on the device: canonical_form of every survivor, then one
        representative per isomorphism class; returns the class count."""
        a = _i64()
        _check(_lib.wpm_plan_line15(self._h, ctypes.byref(a)))
        return int(a.value)

    def line15_stats(self) -> dict:
        a, b = ctypes.c_double(), ctypes.c_double()
        c, d, e, h = _i64(), _i64(), _i32(), _i64()
        _check(_lib.wpm_plan_line15_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                                          ctypes.byref(d), ctypes.byref(e), ctypes.byref(h)))
        return {"ms_canon": a.value, "ms_dedupe": b.value, "labelings": int(c.value), "placements": int(d.value),
                "launches": int(e.value), "cache_hits": int(h.value)}

    def line15_costs(self) -> np.ndarray:
        """placements of each line-13 survivor's canonical-labeling search"""
        n = _lib.wpm_plan_line15_costs(self._h, None, 0)
        if n < 0:
            _check(-n)
        out = np.zeros(max(n, 1), dtype=np.int64)
        _lib.wpm_plan_line15_costs(self._h, out.ctypes.data_as(ctypes.POINTER(_i64)), n)
        return out[:n]

    def fetch_complexes(self, which: int = 13) -> "Complexes":
        """The line-7 union (which=7), the line-13 survivors (13), the
        canonical form of every survivor in survivor order (14), or the
        line-15 class representatives in order of first appearance (15)."""
        cp = _ComplexesP()
        _check(_lib.wpm_plan_fetch_complexes(self._h, which, ctypes.byref(cp)))
        return Complexes(cp)

    def close(self) -> None:
        if self._h:
            _lib.wpm_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class Result:
    """Host copy of an enumeration (wpm_result_t): per-map canonical lists."""

    def __init__(self, rp):
        r = rp.contents
        self.num_maps = r.num_maps
        self.words = r.words
        self.total = r.total
        self.nodes = r.nodes
        self.duplicates = r.duplicates
        self.ms_search = r.ms_search
        self.ms_sort = r.ms_sort
        self.tasks = r.tasks
        self.ms_total = r.ms_total
        self.h2d_bytes = r.h2d_bytes
        self.d2h_bytes = r.d2h_bytes
        self.counts = [int(r.counts[i]) for i in range(r.num_maps)]
        self.offsets = [int(r.offsets[i]) for i in range(r.num_maps + 1)]
        n = r.total * r.words
        # zero-copy view of the library's (page-locked) result rows; the
        # block goes back to the library cache when this object dies
        self._rp = rp
        self.bits = (np.ctypeslib.as_array(r.bits, shape=(max(n, 1),))[:n].reshape(r.total, r.words)
                     if n else np.zeros((0, r.words), dtype=np.uint64))

    def __del__(self):
        rp = getattr(self, "_rp", None)
        if rp is not None:
            self._rp = None
            self.bits = None
            _lib.wpm_result_free(rp)

    def map_bits(self, i: int) -> np.ndarray:
        return self.bits[self.offsets[i]:self.offsets[i + 1]]


class Complexes:
    """Host copy of a labeled complex list (wpm_complexes_t): `facets[offsets[i]:
    offsets[i+1]]` are the facet masks of complex i (bit v = vertex v), `bits`
    the characteristic rows over all n-subsets of [m] (ascending masks)."""

    def __init__(self, cp):
        c = cp.contents
        self.m, self.n, self.count = c.m, c.n, c.count
        self.line7, self.line13, self.line15 = c.line7, c.line13, c.line15
        self.ms_canon, self.ms_dedupe = c.ms_canon, c.ms_dedupe
        self.ms_union, self.ms_filter = c.ms_union, c.ms_filter
        self.h2d_bytes, self.d2h_bytes = c.h2d_bytes, c.d2h_bytes
        self.words = c.words
        self._cp = cp
        self.offsets = np.ctypeslib.as_array(c.offsets, shape=(c.count + 1,))
        nf = int(self.offsets[-1])
        self.facets = (np.ctypeslib.as_array(c.facets, shape=(max(nf, 1),))[:nf] if nf
                       else np.zeros(0, dtype=np.uint64))
        nb = c.count * c.words
        self.bits = (np.ctypeslib.as_array(c.bits, shape=(max(nb, 1),))[:nb].reshape(c.count, c.words) if nb
                     else np.zeros((0, c.words), dtype=np.uint64))

    def __len__(self) -> int:
        return int(self.count)

    def complex(self, i: int) -> List[int]:
        return [int(x) for x in self.facets[self.offsets[i]:self.offsets[i + 1]]]

    def cplx_bytes(self) -> bytes:
        """write_complexes (complex_io.hpp:34-39) of the whole list."""
        need = _lib.wpm_write_complexes(self._cp, None, 0)
        if need < 0:
            _check(-need)
        buf = ctypes.create_string_buffer(int(need) + 1)
        _lib.wpm_write_complexes(self._cp, buf, need)
        return buf.raw[:need]

    def __del__(self):
        cp = getattr(self, "_cp", None)
        if cp is not None:
            self._cp = None
            self.offsets = self.facets = self.bits = None
            _lib.wpm_complexes_free(cp)


def seed_flags(m: int, n: int, complexes: Sequence[Sequence[int]], device: int = 0) -> np.ndarray:
    """is_seed (classify.hpp:51) and full support (complex.hpp:64) of a batch
    of pure complexes on the device: uint8 flags, bit 0 = seed, bit 1 = full
    support.  Raises like PureComplex's validation (complex.hpp:37-55)."""
    off = np.zeros(len(complexes) + 1, dtype=np.int64)
    for i, K in enumerate(complexes):
        off[i + 1] = off[i] + len(K)
    fac = np.zeros(max(int(off[-1]), 1), dtype=np.uint64)
    k = 0
    for K in complexes:
        for f in K:
            fac[k] = int(f)
            k += 1
    flags = np.zeros(max(len(complexes), 1), dtype=np.uint8)
    _check(_lib.wpm_seed_flags(m, n, len(complexes), off.ctypes.data_as(ctypes.POINTER(_i64)),
                               fac.ctypes.data_as(_u64p), device, flags.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
    return flags[:len(complexes)]


def is_seed(m: int, n: int, facets: Sequence[int], device: int = 0) -> bool:
    """classify.hpp:51 for one complex (device)."""
    return bool(seed_flags(m, n, [facets], device)[0] & 1)


def pipeline_line13(n: int, p: int = 4, facet_cap: int = WPM_CAP_UBT, device: int = 0) -> Complexes:
    """Algorithm 2 lines 1-13 for one n (pipeline.hpp:52-89), one call."""
    cp = _ComplexesP()
    _check(_lib.wpm_pipeline_line13(n, p, facet_cap, device, ctypes.byref(cp)))
    return Complexes(cp)


def pipeline_line15(n: int, p: int = 4, facet_cap: int = WPM_CAP_UBT, device: int = 0) -> Complexes:
    """Algorithm 2 lines 1-15 for one n (pipeline.hpp:52-103), one call: the
    line-15 class representatives (canonical forms, first-appearance order)."""
    cp = _ComplexesP()
    _check(_lib.wpm_pipeline_line15(n, p, facet_cap, device, ctypes.byref(cp)))
    return Complexes(cp)


def _csr(complexes: Sequence[Sequence[int]]):
    off = np.zeros(len(complexes) + 1, dtype=np.int64)
    for i, K in enumerate(complexes):
        off[i + 1] = off[i] + len(K)
    fac = np.zeros(max(int(off[-1]), 1), dtype=np.uint64)
    k = 0
    for K in complexes:
        for f in K:
            fac[k] = int(f)
            k += 1
    return off, fac


def canonical_forms(m: int, n: int, complexes: Sequence[Sequence[int]], device: int = 0,
                    with_classes: bool = False):
    """canonical_form (isomorphism.hpp:228-303) of a batch of pure complexes
    on the device: one ascending facet-mask list per complex; with_classes
    also returns detail::refine_classes (isomorphism.hpp:162-218) per vertex
    1..m.  Raises like PureComplex's validation (complex.hpp:37-55)."""
    off, fac = _csr(complexes)
    out = np.zeros_like(fac)
    cls = np.zeros(max(len(complexes) * m, 1), dtype=np.int8)
    _check(_lib.wpm_canonical_forms(m, n, len(complexes), off.ctypes.data_as(ctypes.POINTER(_i64)),
                                    fac.ctypes.data_as(_u64p), device, out.ctypes.data_as(_u64p),
                                    cls.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)) if with_classes else None))
    forms = [[int(x) for x in out[off[i]:off[i + 1]]] for i in range(len(complexes))]
    if with_classes:
        return forms, [[int(x) for x in cls[i * m:(i + 1) * m]] for i in range(len(complexes))]
    return forms


def canonical_form(m: int, n: int, facets: Sequence[int], device: int = 0) -> List[int]:
    """isomorphism.hpp:228-303 for one complex (device)."""
    return canonical_forms(m, n, [facets], device)[0]


# ----------------------------------------------------------------- the drop-in

@dataclass
class SearchJob:
    """search.hpp:46-55.  ``basis`` is not needed by the ridge-driven search;
    pins are given directly as facet indices (apply_link_constraints
    semantics, kernel_basis.hpp:248-321).  ``facets`` may be in any order (the
    reference's incidence_matrix indexes by hash); results come back in
    canonical order.  ``progress(done, total)`` is SearchJob::progress;
    ``devices`` (several GPUs for one job) replaces ``threads``;
    ``candidate_cap`` is accepted for API compatibility (the device search
    has no combination space to cap)."""

    m: int
    n: int
    facets: List[int]
    properties: List[AffineProperty] = field(default_factory=list)
    required: List[int] = field(default_factory=list)
    forbidden: List[int] = field(default_factory=list)
    threads: int = 1
    candidate_cap: int = 1 << 48
    device: int = 0
    progress: Optional[object] = None
    devices: Optional[List[int]] = None


def _facet_cap(job: SearchJob) -> int:
    """search.hpp:181-187: a pure count cap becomes the device cap."""
    cap = WPM_CAP_NONE
    for g in job.properties:
        if not g.is_count_cap():
            raise ValueError("general affine properties are not supported by the B200 path (count caps only)")
        c = g.constant - 1
        cap = c if cap < 0 else min(cap, c)
    return cap


def bits_to_facets(bits_row: np.ndarray, universe: Sequence[int]) -> List[int]:
    out = []
    for w, word in enumerate(bits_row):
        x = int(word)
        while x:
            b = (x & -x).bit_length() - 1
            out.append(universe[w * 64 + b])
            x &= x - 1
    return out


def enumerate_wpm_bits(job: SearchJob) -> Result:
    """enumerate_wpm returning the canonical bitsets over the universe in
    ascending (canonical) order (no PureComplex build)."""
    facets = list(job.facets)
    if not facets:
        raise PurityError("incidence of an empty facet set")
    dev0 = job.devices[0] if job.devices else job.device
    with Plan.universes(job.m, job.n, [facets], _facet_cap(job), job.required, job.forbidden, dev0) as p:
        if job.progress is not None:
            p.set_progress(job.progress)
        if job.devices and len(job.devices) > 1:
            p.set_devices(job.devices)
        p.run()
        return p.fetch()


def enumerate_wpm(job: SearchJob) -> List[List[int]]:
    """search.hpp:141-258: every nonempty WPM inside job.facets satisfying the
    properties, canonical order; each as its ascending facet-mask list."""
    res = enumerate_wpm_bits(job)
    uni = sorted(job.facets)
    return [bits_to_facets(row, uni) for row in res.map_bits(0)]


def matroid_universe(d: DualCharMatrix) -> List[int]:
    """pipeline.hpp:33-35 via kernel 1."""
    cols = charmap_of_dcm(d)
    with Plan.charmaps(d.m - d.p, d.m, [cols], WPM_CAP_UBT, 0) as p:
        return p.universe(0)


def write_complex(m: int, n: int, facets: Sequence[int]) -> str:
    """complex_io.hpp:21-32."""
    lines = [f"{m} {n}"]
    for f in facets:
        lines.append(" ".join(str(v) for v in range(1, 64) if (f >> v) & 1))
    return "\n".join(lines) + "\n"


def write_complexes(m: int, n: int, complexes: Sequence[Sequence[int]]) -> str:
    """complex_io.hpp:34-39."""
    return "\n".join(write_complex(m, n, K) for K in complexes)


def write_cplx_bytes(res: Result, i: int, m: int, n: int, universe: Sequence[int]) -> bytes:
    """Serialise map i of a result through the C-ABI writer (byte-exact .cplx)."""
    uni, up = _u64(universe)
    # rebuild a transient wpm_result_t view for the writer
    rr = _Result()
    rr.num_maps = res.num_maps
    rr.words = res.words
    rr.total = res.total
    counts = (ctypes.c_int64 * max(res.num_maps, 1))(*res.counts)
    offsets = (ctypes.c_int64 * (res.num_maps + 1))(*res.offsets)
    bits = np.ascontiguousarray(res.bits.reshape(-1) if res.bits.size else np.zeros(1, dtype=np.uint64))
    rr.counts = counts
    rr.offsets = offsets
    rr.bits = bits.ctypes.data_as(_u64p)
    need = int(_lib.wpm_write_cplx(ctypes.byref(rr), i, m, n, up, None, 0))
    if need < 0:
        _check(-need)
    buf = ctypes.create_string_buffer(max(need, 1))
    _lib.wpm_write_cplx(ctypes.byref(rr), i, m, n, up, buf, need)
    return buf.raw[:need]
