"""GPU parity of Algorithm 2 lines 7 and 13 (k5_line13.cu) through the C-ABI.

* line7 / line13 counts and the SHA-256 of the line-13 survivors written with
  write_complexes, n = 2..11, against golden.json["line13"] (the reference
  pipeline for n <= 7, the oracle for n >= 8 -- see make_golden_line13.py);
* the line-7 union against the oracle's union of the same per-map lists;
* wpm_seed_flags (is_seed + support) against the literal oracle restatement
  on the catalog complexes of test_classify.cpp:24-31 and random complexes;
* PureComplex validation errors (complex.hpp:37-55).
"""
import hashlib
import random

import numpy as np
import pytest

import catalog as C

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8, 9, 10, 11])
def test_line13_counts_and_digest(wpm, golden, n):
    want = golden["line13"][str(n)]
    with wpm.Plan.orbits(n) as p:
        p.run()
        l7, l13 = p.line13()
        assert (l7, l13) == (want["line7"], want["line13"])
        surv = p.fetch_complexes(13)
        assert len(surv) == l13 and surv.line7 == l7
        assert hashlib.sha256(surv.cplx_bytes()).hexdigest() == want["sha256"]
        # every survivor: full support, pure, facets ascending
        full = C.full(n + 4)
        for i in range(0, len(surv), max(1, len(surv) // 50)):
            fs = surv.complex(i)
            assert fs == sorted(fs) and all(bin(f).count("1") == n for f in fs)
            assert np.bitwise_or.reduce(np.array(fs, dtype=np.uint64)) == full


@pytest.mark.parametrize("n", [3, 4])
def test_line7_union_matches_oracle(wpm, oracle, n):
    m = n + 4
    all_sub = np.array(oracle.all_subsets_universe(m, n), dtype=np.uint64)
    with wpm.Plan.orbits(n) as p:
        p.run()
        p.line13()
        union = p.fetch_complexes(7)
    rows = []
    for r in oracle.idcm_orbits(n):
        uni = oracle.matroid_universe(r)
        _, _, bits = oracle.dfs(n, uni, oracle.cyclic_facet_bound(n))
        gidx = np.searchsorted(all_sub, np.array(uni, dtype=np.uint64))
        out = np.zeros((bits.shape[0], union.words), dtype=np.uint64)
        for j, g in enumerate(gidx):
            hit = (bits[:, j >> 6] >> np.uint64(j & 63)) & np.uint64(1)
            out[:, g >> 6] |= hit << np.uint64(int(g) & 63)
        rows.append(out)
    allr = np.concatenate(rows)
    l7, l13, surv = oracle.line13(m, n, allr)
    assert len(union) == l7
    # the union's rows, in order, are the oracle's sorted unique rows
    uniq = np.unique(allr, axis=0)
    assert uniq.shape[0] == l7
    got = {tuple(r) for r in union.bits.tolist()}
    assert got == {tuple(r) for r in uniq.tolist()}
    for i in range(len(union) - 1):
        assert oracle.bits_cmp(union.bits[i], union.bits[i + 1]) < 0


def test_seed_flags_catalog(wpm):
    cases = [(C.s0(), True), (C.simplex_boundary(2), False), (C.square(), True),
             (C.wedge(C.square(), 1), False), (C.hexagon(), True), (C.octahedron(), True),
             (C.pentagon(), True), (C.simplex_boundary(5), False)]
    for (m, n, fs), want in cases:
        assert wpm.is_seed(m, n, fs) == want, (m, n, fs)


def test_seed_flags_random_vs_oracle(wpm, oracle):
    rng = random.Random(5)
    by_shape = {}
    for _ in range(1500):
        m = rng.randint(2, 12)
        n = rng.randint(1, min(m - 1, 7))
        K = C.random_pure(rng, m, n, rng.choice([0.1, 0.3, 0.6, 0.9, 1.0]))
        if K[2] and rng.random() < 0.4 and m < 12:
            vs = [v for v in range(1, m + 1) if any(f >> v & 1 for f in K[2])]
            K = C.wedge(K, rng.choice(vs))
        if rng.random() < 0.5:
            tail = list(range(1, K[0] + 1))
            rng.shuffle(tail)
            K = C.relabel(K, [0] + tail)
        by_shape.setdefault((K[0], K[1]), []).append(K[2])
    seeds = total = 0
    for (m, n), ks in by_shape.items():
        flags = wpm.seed_flags(m, n, ks)
        for fs, fl in zip(ks, flags):
            want_seed = oracle.is_seed(m, fs, literal=True)
            want_sup = (np.bitwise_or.reduce(np.array(fs, dtype=np.uint64)) == C.full(m)) if fs else False
            assert bool(fl & 1) == want_seed, (m, n, fs)
            assert bool(fl & 2) == bool(want_sup), (m, n, fs)
            seeds += want_seed
            total += 1
    assert 0 < seeds < total


def test_seed_flags_unsorted_input_and_empty(wpm):
    m, n, fs = C.octahedron()
    assert wpm.seed_flags(m, n, [list(reversed(fs)), []]).tolist() == [3, 1]


def test_seed_flags_validation(wpm):
    with pytest.raises(wpm.PurityError):
        wpm.seed_flags(4, 2, [[C.mask(1, 2), C.mask(1, 2, 3)]])
    with pytest.raises(ValueError):
        wpm.seed_flags(4, 2, [[C.mask(1, 5)]])  # label outside 1..m
    with pytest.raises(ValueError):
        wpm.seed_flags(4, 2, [[C.mask(1, 2), C.mask(1, 2)]])  # duplicate facet
    with pytest.raises(ValueError):
        wpm.seed_flags(17, 2, [[C.mask(1, 2)]])  # beyond the device label range


def test_line13_needs_a_run(wpm):
    with wpm.Plan.orbits(3) as p:
        with pytest.raises(ValueError):
            p.line13()
        p.run()
        with pytest.raises(ValueError):
            p.fetch_complexes(13)  # before line13()
        p.line13()
        with pytest.raises(ValueError):
            p.fetch_complexes(8)


def test_pipeline_line13_one_shot(wpm, golden):
    res = wpm.pipeline_line13(5)
    want = golden["line13"]["5"]
    assert (res.line7, res.line13, len(res)) == (want["line7"], want["line13"], want["line13"])
    assert hashlib.sha256(res.cplx_bytes()).hexdigest() == want["sha256"]
    assert res.d2h_bytes > 0


def test_line13_rerun_is_deterministic(wpm):
    with wpm.Plan.orbits(6) as p:
        p.run()
        a = p.line13()
        da = hashlib.sha256(p.fetch_complexes(13).cplx_bytes()).hexdigest()
        p.run()
        b = p.line13()
        db = hashlib.sha256(p.fetch_complexes(13).cplx_bytes()).hexdigest()
    assert a == b and da == db
