"""ctypes binding of oracle/liboracle.so -- TEST INFRASTRUCTURE ONLY.

The oracle (oracle/plseeds_port.c: the reference algorithm restated in C;
oracle/dfs_port.c: the device search restated in C) is the checker.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Sequence, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
LIB = os.path.join(ORACLE_DIR, "liboracle.so")

_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i32p = ctypes.POINTER(ctypes.c_int32)


class _PoResult(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("words", ctypes.c_int), ("bits", _u64p), ("space", ctypes.c_uint64),
                ("s", ctypes.c_int), ("nblocks", ctypes.c_int)]


class _DfsResult(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("words", ctypes.c_int), ("bits", _u64p), ("nodes", ctypes.c_int64)]


def build_oracle() -> str:
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
    return LIB


def _arr(a, dt):
    x = np.ascontiguousarray(np.asarray(a, dtype=dt))
    if x.size == 0:
        x = np.zeros(1, dtype=dt)
    return x


class Oracle:
    def __init__(self):
        self.lib = ctypes.CDLL(build_oracle())
        L = self.lib
        L.po_idcm_orbits.argtypes = [ctypes.c_int, ctypes.c_int, _u32p, ctypes.c_int]
        L.po_charmap_of_dcm.argtypes = [ctypes.c_int, ctypes.c_int, _u32p, _u32p]
        L.po_binary_matroid.argtypes = [ctypes.c_int, ctypes.c_int, _u32p, _u64p, ctypes.c_int]
        L.po_all_subsets_universe.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_int]
        L.po_cyclic_facet_bound.argtypes = [ctypes.c_int]
        L.po_cyclic_facet_bound.restype = ctypes.c_int64
        L.po_incidence.argtypes = [_u64p, ctypes.c_int, _u64p, ctypes.c_int, _i32p, _i32p, _i32p]
        L.po_enumerate_wpm.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int64, _i32p,
                                       ctypes.c_int, _i32p, ctypes.c_int, ctypes.c_uint64,
                                       ctypes.POINTER(_PoResult)]
        L.po_result_free.argtypes = [ctypes.POINTER(_PoResult)]
        L.po_brute_force_count.argtypes = [_u64p, ctypes.c_int, _i32p, ctypes.c_int, _i32p, ctypes.c_int,
                                           ctypes.c_int64]
        L.po_brute_force_count.restype = ctypes.c_int64
        L.po_is_wpm_direct.argtypes = [_u64p, ctypes.c_int]
        L.po_write_cplx.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_int, _u64p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_char_p, ctypes.c_int64]
        L.po_write_cplx.restype = ctypes.c_int64
        L.po_bits_cmp.argtypes = [_u64p, _u64p, ctypes.c_int]
        L.dfs_enumerate.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int64, _i32p, ctypes.c_int, _i32p,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(_DfsResult)]
        L.dfs_result_free.argtypes = [ctypes.POINTER(_DfsResult)]
        L.po_minimal_nonfaces.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, _u64p, ctypes.c_int]
        L.po_wedge_witness.argtypes = [_u64p, ctypes.c_int, _u64p, ctypes.c_int, _i32p, _i32p]
        L.po_is_seed.argtypes = [ctypes.c_int, _u64p, ctypes.c_int]
        L.po_is_seed_swap.argtypes = [ctypes.c_int, _u64p, ctypes.c_int]
        L.po_line13.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_int64, ctypes.c_int,
                                ctypes.POINTER(ctypes.c_int64), _u64p, ctypes.POINTER(ctypes.c_int64)]
        L.po_line13.restype = ctypes.c_int64
        L.po_refine_classes.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, _i32p]
        L.po_canonical_form.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, _u64p, ctypes.POINTER(ctypes.c_longlong)]
        L.dfs_enumerate_shard.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int, ctypes.POINTER(_DfsResult)]

    # -- characteristic maps
    def idcm_orbits(self, n: int, p: int = 4) -> List[List[int]]:
        m = n + p
        buf = np.zeros(64 * m, dtype=np.uint32)
        k = self.lib.po_idcm_orbits(n, p, buf.ctypes.data_as(_u32p), 64)
        if k < 0:
            raise ValueError("invalid (n, p)")
        return [[int(x) for x in buf[i * m:(i + 1) * m]] for i in range(k)]

    def charmap_of_dcm(self, rows: Sequence[int], p: int = 4) -> List[int]:
        r = _arr(rows, np.uint32)
        cols = np.zeros(len(rows), dtype=np.uint32)
        n = self.lib.po_charmap_of_dcm(len(rows), p, r.ctypes.data_as(_u32p), cols.ctypes.data_as(_u32p))
        if n < 0:
            raise ValueError("rank deficient")
        return [int(c) for c in cols]

    def binary_matroid(self, n: int, cols: Sequence[int]) -> List[int]:
        c = _arr(cols, np.uint32)
        out = np.zeros(1 << 14, dtype=np.uint64)
        M = self.lib.po_binary_matroid(n, len(cols), c.ctypes.data_as(_u32p), out.ctypes.data_as(_u64p), len(out))
        if M < 0:
            raise ValueError("matrix is rank deficient")
        return [int(x) for x in out[:M]]

    def matroid_universe(self, rows: Sequence[int], p: int = 4) -> List[int]:
        return self.binary_matroid(len(rows) - p, self.charmap_of_dcm(rows, p))

    def all_subsets_universe(self, m: int, n: int) -> List[int]:
        out = np.zeros(1 << 16, dtype=np.uint64)
        M = self.lib.po_all_subsets_universe(m, n, out.ctypes.data_as(_u64p), len(out))
        return [int(x) for x in out[:M]]

    def cyclic_facet_bound(self, n: int) -> int:
        return int(self.lib.po_cyclic_facet_bound(n))

    # -- incidence
    def incidence(self, facets: Sequence[int]):
        f = _arr(facets, np.uint64)
        M = len(facets)
        n = bin(int(facets[0])).count("1")
        ridges = np.zeros(M * n, dtype=np.uint64)
        cols = np.zeros(M * n, dtype=np.int32)
        po = np.zeros(M * n + 1, dtype=np.int32)
        pa = np.zeros(M * n, dtype=np.int32)
        N = self.lib.po_incidence(f.ctypes.data_as(_u64p), M, ridges.ctypes.data_as(_u64p), M * n,
                                  cols.ctypes.data_as(_i32p), po.ctypes.data_as(_i32p), pa.ctypes.data_as(_i32p))
        if N < 0:
            raise ValueError("impure")
        parents = [[int(x) for x in pa[po[r]:po[r + 1]]] for r in range(N)]
        return [int(x) for x in ridges[:N]], cols.reshape(M, n).tolist(), parents

    # -- the reference algorithm (kernel-basis odometer)
    def enumerate_ref(self, m: int, n: int, facets: Sequence[int], cap: int = -1, required=(), forbidden=(),
                      candidate_cap: int = (1 << 64) - 1):
        f = _arr(facets, np.uint64)
        rq = _arr(list(required), np.int32)
        fb = _arr(list(forbidden), np.int32)
        res = _PoResult()
        rc = self.lib.po_enumerate_wpm(m, n, f.ctypes.data_as(_u64p), len(facets), cap, rq.ctypes.data_as(_i32p),
                                       len(required), fb.ctypes.data_as(_i32p), len(forbidden),
                                       ctypes.c_uint64(candidate_cap), ctypes.byref(res))
        if rc != 0:
            return rc, None
        cnt, w = res.count, res.words
        bits = (np.ctypeslib.as_array(res.bits, shape=(cnt * w,)).copy().reshape(cnt, w) if cnt
                else np.zeros((0, w), dtype=np.uint64))
        out = {"count": cnt, "bits": bits, "space": res.space, "s": res.s, "nblocks": res.nblocks}
        self.lib.po_result_free(ctypes.byref(res))
        return 0, out

    # -- the device search restated
    def dfs(self, n: int, facets: Sequence[int], cap: int = -1, required=(), forbidden=(), want_bits=True,
            root_lo: int = 0, root_hi: int = -1) -> Tuple[int, int, np.ndarray]:
        f = _arr(facets, np.uint64)
        rq = _arr(list(required), np.int32)
        fb = _arr(list(forbidden), np.int32)
        res = _DfsResult()
        M = len(facets)
        rc = self.lib.dfs_enumerate(n, f.ctypes.data_as(_u64p), M, cap, rq.ctypes.data_as(_i32p), len(required),
                                    fb.ctypes.data_as(_i32p), len(forbidden), 1 if want_bits else 0, root_lo,
                                    M if root_hi < 0 else root_hi, ctypes.byref(res))
        if rc != 0:
            raise ValueError("bad universe")
        cnt, w = res.count, res.words
        bits = (np.ctypeslib.as_array(res.bits, shape=(cnt * w,)).copy().reshape(cnt, w) if cnt and want_bits
                else np.zeros((0, w), dtype=np.uint64))
        nodes = res.nodes
        self.lib.dfs_result_free(ctypes.byref(res))
        return cnt, nodes, bits

    def dfs_shard(self, n: int, facets: Sequence[int], cap: int, shard_index: int, shard_count: int):
        f = _arr(facets, np.uint64)
        res = _DfsResult()
        rc = self.lib.dfs_enumerate_shard(n, f.ctypes.data_as(_u64p), len(facets), cap, 1, shard_index, shard_count,
                                          ctypes.byref(res))
        if rc != 0:
            raise ValueError("bad universe")
        cnt, w = res.count, res.words
        bits = (np.ctypeslib.as_array(res.bits, shape=(cnt * w,)).copy().reshape(cnt, w) if cnt
                else np.zeros((0, w), dtype=np.uint64))
        nodes = res.nodes
        self.lib.dfs_result_free(ctypes.byref(res))
        return cnt, nodes, bits

    def brute_force_count(self, facets, required=(), forbidden=(), cap: int = -1) -> int:
        f = _arr(facets, np.uint64)
        rq = _arr(list(required), np.int32)
        fb = _arr(list(forbidden), np.int32)
        return int(self.lib.po_brute_force_count(f.ctypes.data_as(_u64p), len(facets), rq.ctypes.data_as(_i32p),
                                                 len(required), fb.ctypes.data_as(_i32p), len(forbidden), cap))

    def is_wpm_direct(self, facets: Sequence[int]) -> bool:
        f = _arr(facets, np.uint64)
        return bool(self.lib.po_is_wpm_direct(f.ctypes.data_as(_u64p), len(facets)))

    def write_cplx(self, m: int, n: int, universe: Sequence[int], bits: np.ndarray) -> bytes:
        u = _arr(universe, np.uint64)
        b = np.ascontiguousarray(bits, dtype=np.uint64)
        cnt = b.shape[0]
        w = b.shape[1] if b.ndim == 2 else 1
        if cnt == 0:
            return b""
        bp = b.ctypes.data_as(_u64p)
        need = self.lib.po_write_cplx(m, n, u.ctypes.data_as(_u64p), len(universe), bp, cnt, w, None, 0)
        buf = ctypes.create_string_buffer(int(need))
        self.lib.po_write_cplx(m, n, u.ctypes.data_as(_u64p), len(universe), bp, cnt, w, buf, need)
        return buf.raw[:need]

    def bits_cmp(self, a: np.ndarray, b: np.ndarray) -> int:
        x = np.ascontiguousarray(a, dtype=np.uint64)
        y = np.ascontiguousarray(b, dtype=np.uint64)
        return int(self.lib.po_bits_cmp(x.ctypes.data_as(_u64p), y.ctypes.data_as(_u64p), len(x)))

    # -- Algorithm 2 lines 7 and 13 (oracle/line13_port.c)
    def minimal_nonfaces(self, m: int, facets: Sequence[int]) -> List[int]:
        f = _arr(facets, np.uint64)
        out = np.zeros(1 << 16, dtype=np.uint64)
        k = self.lib.po_minimal_nonfaces(m, f.ctypes.data_as(_u64p), len(facets), out.ctypes.data_as(_u64p),
                                         len(out))
        if k < 0:
            raise ValueError("bad complex")
        return [int(x) for x in out[:k]]

    def wedge_witness(self, m: int, facets: Sequence[int]):
        mnf = _arr(self.minimal_nonfaces(m, facets), np.uint64)
        f = _arr(facets, np.uint64)
        u = ctypes.c_int32(0)
        v = ctypes.c_int32(0)
        w = self.lib.po_wedge_witness(f.ctypes.data_as(_u64p), len(facets), mnf.ctypes.data_as(_u64p),
                                      len(self.minimal_nonfaces(m, facets)), ctypes.byref(u), ctypes.byref(v))
        return (u.value, v.value) if w == 1 else None

    def is_seed(self, m: int, facets: Sequence[int], literal: bool = True) -> bool:
        f = _arr(sorted(facets), np.uint64)
        fn = self.lib.po_is_seed if literal else self.lib.po_is_seed_swap
        r = fn(m, f.ctypes.data_as(_u64p), len(facets))
        if r < 0:
            raise ValueError("bad complex")
        return bool(r)

    def line13(self, m: int, n: int, rows: np.ndarray, literal: bool = False):
        """pipeline.hpp:58-89 on complexes given as bitsets over the
        all-subsets universe of (m, n): (line7, line13, survivor rows)."""
        r = np.ascontiguousarray(rows, dtype=np.uint64)
        cnt = r.shape[0]
        w = r.shape[1]
        if cnt == 0:
            r = np.zeros((1, w), dtype=np.uint64)
        surv = np.zeros((max(cnt, 1), w), dtype=np.uint64)
        l7 = ctypes.c_int64(0)
        k = self.lib.po_line13(m, n, w, r.ctypes.data_as(_u64p), cnt, 1 if literal else 0, ctypes.byref(l7),
                               surv.ctypes.data_as(_u64p), None)
        if k < 0:
            raise ValueError("line13 failed")
        return int(l7.value), int(k), surv[:k].copy()

    # -- Algorithm 2 line 15 (oracle/line15_port.c)
    def refine_classes(self, m: int, facets: Sequence[int]) -> List[int]:
        """isomorphism.hpp:162-218: refined class of vertices 1..m."""
        f = _arr(facets, np.uint64)
        cls = np.zeros(m, dtype=np.int32)
        r = self.lib.po_refine_classes(m, f.ctypes.data_as(_u64p), len(facets), cls.ctypes.data_as(_i32p))
        if r < 0:
            raise ValueError("bad complex")
        return [int(x) for x in cls]

    def canonical_form(self, m: int, facets: Sequence[int]) -> Tuple[List[int], int]:
        """isomorphism.hpp:228-303: (canonical facets ascending, labelings visited)."""
        f = _arr(sorted(facets), np.uint64)
        out = np.zeros(max(len(facets), 1), dtype=np.uint64)
        leaves = ctypes.c_longlong(0)
        k = self.lib.po_canonical_form(m, f.ctypes.data_as(_u64p), len(facets), out.ctypes.data_as(_u64p),
                                       ctypes.byref(leaves))
        if k < 0:
            raise ValueError("bad complex")
        return [int(x) for x in out[:k]], int(leaves.value)

    def line15(self, m: int, n: int, rows: np.ndarray):
        """pipeline.hpp:91-103 on line-13 survivors given as bitsets over the
        all-subsets universe: (canonical rows per survivor, first-appearance
        representative indices)."""
        all_sub = np.asarray(self.all_subsets_universe(m, n), dtype=np.uint64)
        r = np.ascontiguousarray(rows, dtype=np.uint64)
        canon = np.zeros_like(r)
        seen = {}
        reps = []
        for i in range(r.shape[0]):
            facets = [int(all_sub[j]) for j in _bits_of(r[i])]
            cf, _ = self.canonical_form(m, facets)
            idx = np.searchsorted(all_sub, np.asarray(cf, dtype=np.uint64))
            for j in idx:
                canon[i, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
            key = canon[i].tobytes()
            if key not in seen:
                seen[key] = i
                reps.append(i)
        return canon, reps


def _bits_of(row: np.ndarray) -> List[int]:
    out = []
    for w, x in enumerate(row.tolist()):
        while x:
            b = x & -x
            out.append(w * 64 + b.bit_length() - 1)
            x ^= b
    return out


def read_cplx(data: bytes):
    """complex_io.hpp:41-89 reader: list of (m, n, [facet masks])."""
    out = []
    for block in data.decode().strip().split("\n\n"):
        lines = block.strip().split("\n")
        if not lines or not lines[0]:
            continue
        m, n = map(int, lines[0].split())
        fs = []
        for ln in lines[1:]:
            mask = 0
            for v in ln.split():
                mask |= 1 << int(v)
            fs.append(mask)
        out.append((m, n, fs))
    return out
