"""CPU tests of the Algorithm 2 line-7/13 oracle (oracle/line13_port.c).

Pins: the seedness cases of test_classify.cpp:24-31 and :205-220, the
reference's own is_seed (oracle/_ref/plseeds_ref seed) on random complexes,
and the reference pipeline's line7/line13 counts (107 / 1676 /
44572 / 202984 and 28 / 858 / 30490 / 121712, re-measured by
tests/golden/make_golden_line13.py into golden.json["line13"]).
"""
import hashlib
import os
import random
import subprocess
import tempfile

import numpy as np
import pytest

import catalog as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")


def test_seedness_catalog(oracle):
    # test_classify.cpp:24-31
    cases = [(C.s0(), True), (C.simplex_boundary(2), False), (C.square(), True),
             (C.wedge(C.square(), 1), False), (C.hexagon(), True), (C.octahedron(), True)]
    for (m, n, fs), want in cases:
        assert oracle.is_seed(m, fs, literal=True) == want, (m, n, fs)
        assert oracle.is_seed(m, fs, literal=False) == want, (m, n, fs)


def test_minimal_nonfaces_known(oracle):
    # square: the two diagonals; boundary of the triangle: the triangle itself
    m, _, fs = C.square()
    assert oracle.minimal_nonfaces(m, fs) == sorted([C.mask(1, 3), C.mask(2, 4)])
    m, _, fs = C.simplex_boundary(2)
    assert oracle.minimal_nonfaces(m, fs) == [C.mask(1, 2, 3)]
    m, _, fs = C.pentagon()
    assert len(oracle.minimal_nonfaces(m, fs)) == 5
    # a ghost vertex is a singleton candidate (complex.hpp:199-202) but never
    # survives the minimality check (:210-217): face_set has no empty face
    # (faces_by_card erases it, :185) -- what the compiled reference returns
    assert oracle.minimal_nonfaces(5, C.square()[2]) == sorted([C.mask(1, 3), C.mask(2, 4)])
    # wedging the square at 1 turns the diagonal {1, 3} into {1, 3, 5}, so the
    # minimal non-faces are {1, 3, 5}, {2, 4}; the first witness edge in
    # canonical order is {1, 3} (classify.hpp:36-46)
    m, _, fs = C.wedge(C.square(), 1)
    assert oracle.minimal_nonfaces(m, fs) == sorted([C.mask(1, 3, 5), C.mask(2, 4)])
    assert oracle.wedge_witness(m, fs) == (1, 3)


def test_suspension_preserves_seedness(oracle):
    # test_classify.cpp:205-220 on random small complexes
    rng = random.Random(7)
    for _ in range(60):
        K = C.random_pure(rng, rng.randint(3, 6), rng.randint(1, 3), 0.5)
        if not K[2]:
            continue
        S = C.suspension(K)
        assert oracle.is_seed(S[0], S[2]) == oracle.is_seed(K[0], K[2])


def _random_cases(seed, count):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        m = rng.randint(2, 8)
        n = rng.randint(1, min(m - 1, 5))
        K = C.random_pure(rng, m, n, rng.choice([0.2, 0.4, 0.6, 0.8, 1.0]))
        if rng.random() < 0.35 and K[2]:  # wedges are non-seeds: exercise witnesses
            v = rng.choice([v for v in range(1, m + 1) if any(f >> v & 1 for f in K[2])] or [1])
            if any(f >> v & 1 for f in K[2]) and K[0] < 9:
                K = C.wedge(K, v)
        if rng.random() < 0.5:
            perm = list(range(K[0] + 1))
            tail = perm[1:]
            rng.shuffle(tail)
            K = C.relabel(K, [0] + tail)
        out.append(K)
    return out


def test_literal_and_swap_forms_agree(oracle):
    seeds = 0
    for m, n, fs in _random_cases(11, 600):
        a = oracle.is_seed(m, fs, literal=True)
        b = oracle.is_seed(m, fs, literal=False)
        assert a == b, (m, n, fs)
        seeds += a
    assert 50 < seeds < 590  # both outcomes exercised


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="reference driver not built")
def test_is_seed_matches_reference_binary(oracle):
    cases = [c for c in _random_cases(23, 300) if c[2]]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "k.cplx")
        with open(path, "w") as f:
            for i, (m, n, fs) in enumerate(cases):
                if i:
                    f.write("\n")
                f.write(f"{m} {n}\n")
                for x in fs:
                    f.write(" ".join(str(v) for v in range(1, m + 1) if x >> v & 1) + "\n")
        out = subprocess.run([REF_BIN, "seed", path], check=True, capture_output=True, text=True).stdout.split()
    assert len(out) == 2 * len(cases)
    for i, (m, n, fs) in enumerate(cases):
        sup = int(out[2 * i])
        seed = int(out[2 * i + 1])
        got_sup = 1 if (np.bitwise_or.reduce(np.array(fs, dtype=np.uint64)) == C.full(m)) else 0
        assert sup == got_sup
        assert seed == int(oracle.is_seed(m, fs, literal=True)), (m, n, fs)


def _global_rows(oracle, n):
    """every UBT-capped WPM of every orbit map, as bitsets over all n-subsets"""
    m = n + 4
    all_sub = np.array(oracle.all_subsets_universe(m, n), dtype=np.uint64)
    gw = (len(all_sub) + 63) // 64
    rows = []
    for r in oracle.idcm_orbits(n):
        uni = oracle.matroid_universe(r)
        _, _, bits = oracle.dfs(n, uni, oracle.cyclic_facet_bound(n))
        gidx = np.searchsorted(all_sub, np.array(uni, dtype=np.uint64))
        out = np.zeros((bits.shape[0], gw), dtype=np.uint64)
        for j, g in enumerate(gidx):
            hit = (bits[:, j >> 6] >> np.uint64(j & 63)) & np.uint64(1)
            out[:, g >> 6] |= hit << np.uint64(int(g) & 63)
        rows.append(out)
    return m, all_sub, np.concatenate(rows)


@pytest.mark.parametrize("n", [2, 3, 4])
def test_line13_counts_match_reference(oracle, golden, n):
    m, all_sub, rows = _global_rows(oracle, n)
    want = golden["line13"][str(n)]
    for literal in (True, False):
        l7, l13, surv = oracle.line13(m, n, rows, literal=literal)
        assert (l7, l13) == (want["line7"], want["line13"])
        data = oracle.write_cplx(m, n, list(all_sub), surv)
        assert hashlib.sha256(data).hexdigest() == want["sha256"]


def test_line13_golden_counts_survey(golden):
    # the reference pipeline's own line7/line13 for n = 2..5
    g = golden["line13"]
    assert [g[str(n)]["line7"] for n in (2, 3, 4, 5)] == [107, 1676, 44572, 202984]
    assert [g[str(n)]["line13"] for n in (2, 3, 4, 5)] == [28, 858, 30490, 121712]
    assert all(str(n) in g for n in range(2, 12))
