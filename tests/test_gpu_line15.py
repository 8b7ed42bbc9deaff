"""GPU parity of Algorithm 2 line 15 (k7_line15.cu) through the C-ABI.

* line-15 count, the SHA-256 of the representatives' .cplx (first-appearance
  order) and the SHA-256 of every survivor's canonical form (survivor order)
  against golden.json["line15"] -- the reference's own canonical_form and
  dedupe (pipeline.hpp:91-103) run on the golden line-13 survivors -- and the
  paper's line-15 counts (n <= 10);
* wpm_canonical_forms / refine classes against the literal oracle
  restatement (oracle/line15_port.c) on catalog complexes with large
  automorphism groups and on random pure complexes;
* isomorphism invariance: random relabelings share one canonical form;
* PureComplex validation errors (complex.hpp:37-55).
"""
import hashlib
import random

import pytest

import catalog as C

pytestmark = pytest.mark.gpu


def _ns(golden):
    return sorted(int(k) for k in golden.get("line15", {}))


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 8, 9, 10, 11])
def test_line15_counts_and_digests(wpm, golden, n):
    want = golden["line15"][str(n)]
    with wpm.Plan.orbits(n) as p:
        p.run()
        _, l13 = p.line13()
        assert l13 == want["line13"]
        l15 = p.line15()
        if "line15" in want:
            assert l15 == want["line15"]
        if "paper_line15" in want:
            assert l15 == want["paper_line15"]
        reps = p.fetch_complexes(15)
        assert len(reps) == l15 and reps.line15 == l15
        canon = p.fetch_complexes(14)
        assert len(canon) == l13
        if "sha256" in want:  # the reference's own canonical forms (n <= 7)
            assert hashlib.sha256(reps.cplx_bytes()).hexdigest() == want["sha256"]
            assert hashlib.sha256(canon.cplx_bytes()).hexdigest() == want["canon_sha256"]
        # the representatives are the first appearances of the distinct canonical forms
        firsts, seen = [], set()
        for i in range(len(canon)):
            key = canon.bits[i].tobytes()
            if key not in seen:
                seen.add(key)
                firsts.append(canon.complex(i))
        assert [reps.complex(i) for i in range(len(reps))] == firsts
        st = p.line15_stats()
        assert st["labelings"] >= l13 and st["ms_canon"] > 0


@pytest.mark.parametrize("n", [8, 9, 10, 11])
def test_line15_sampled_vs_oracle(wpm, oracle, n):
    """n >= 8: the reference's canonical_form does not finish on the most
    symmetric survivors, so the device's canonical forms are checked against
    the literal oracle restatement on every sampled survivor whose class
    structure keeps the oracle's search small (<= 40320 labelings)."""
    from math import factorial, prod
    from collections import Counter

    m = n + 4
    with wpm.Plan.orbits(n) as p:
        p.run()
        p.line13()
        p.line15()
        surv = p.fetch_complexes(13)
        canon = p.fetch_complexes(14)
    rng = random.Random(n)
    idx = rng.sample(range(len(surv)), 400)
    checked = 0
    for i in idx:
        fs = surv.complex(i)
        cls = oracle.refine_classes(m, fs)
        if prod(factorial(c) for c in Counter(cls).values()) > 40320:
            continue
        want, _ = oracle.canonical_form(m, fs)
        assert canon.complex(i) == want, (n, i)
        checked += 1
    assert checked >= 100


def _relabel(facets, perm):
    out = []
    for f in facets:
        g = 0
        for v in range(1, len(perm)):
            if f >> v & 1:
                g |= 1 << perm[v]
        out.append(g)
    return sorted(out)


def _random_complex(rng, m, n, k):
    import itertools

    all_sub = [sum(1 << v for v in c) for c in itertools.combinations(range(1, m + 1), n)]
    return sorted(rng.sample(all_sub, min(k, len(all_sub))))


def _catalog():
    """complexes with large automorphism groups whose literal (class-boundary
    pruned) oracle search still finishes: <= 8! labelings per class"""
    return [C.s0(), C.square(), C.pentagon(), C.hexagon(), C.cycle_complex(8), C.octahedron(),
            C.cross_polytope_boundary(4), C.simplex_boundary(6), C.suspension(C.octahedron()),
            C.join(C.pentagon(), C.square()), C.wedge(C.square(), 1), C.wedge(C.pentagon(), 2),
            C.suspension(C.pentagon())]


def test_canonical_forms_catalog_vs_oracle(wpm, oracle):
    cases = [(m, n, fs) for (m, n, fs) in _catalog() if m <= 15 and n <= 11]
    assert cases
    for m, n, fs in cases:
        got, cls = wpm.canonical_forms(m, n, [fs], with_classes=True)
        want, _ = oracle.canonical_form(m, fs)
        assert got[0] == want, (m, n, fs)
        assert cls[0] == oracle.refine_classes(m, fs)


@pytest.mark.parametrize("seed", range(6))
def test_canonical_forms_random_vs_oracle(wpm, oracle, seed):
    rng = random.Random(seed)
    by_shape = {}
    for _ in range(120):
        m = rng.randint(4, 11)
        n = rng.randint(1, min(m - 1, 6))
        from math import comb

        k = rng.randint(1, min(comb(m, n), 40))
        by_shape.setdefault((m, n), []).append(_random_complex(rng, m, n, k))
    for (m, n), batch in by_shape.items():
        got, cls = wpm.canonical_forms(m, n, batch, with_classes=True)
        for fs, g, c in zip(batch, got, cls):
            want, _ = oracle.canonical_form(m, fs)
            assert g == want, (m, n, fs)
            assert c == oracle.refine_classes(m, fs), (m, n, fs)


@pytest.mark.parametrize("seed", range(3))
def test_canonical_form_is_an_isomorphism_invariant(wpm, seed):
    rng = random.Random(100 + seed)
    shapes = [(9, 5, _random_complex(rng, 9, 5, 30)), (12, 8, _random_complex(rng, 12, 8, 80)),
              (15, 11, _random_complex(rng, 15, 11, 120)),
              # one refined class of 15 / 12 vertices: the reference's search would visit 15! labelings
              C.cycle_complex(15), C.cross_polytope_boundary(6), C.join(C.cycle_complex(7), C.cycle_complex(8))]
    for m, n, fs in shapes:
        batch = [fs]
        for _ in range(7):
            perm = list(range(m + 1))
            tail = perm[1:]
            rng.shuffle(tail)
            batch.append(_relabel(fs, [0] + tail))
        forms = wpm.canonical_forms(m, n, batch)
        assert all(f == forms[0] for f in forms), (m, n)


def test_canonical_forms_validation(wpm):
    with pytest.raises(wpm.PurityError):
        wpm.canonical_forms(6, 3, [[0b1110, 0b110]])  # facet of size 2
    with pytest.raises(ValueError):
        wpm.canonical_forms(4, 2, [[1 << 5 | 1 << 1]])  # label 5 > m
    with pytest.raises(ValueError):
        wpm.canonical_forms(16, 3, [[0b1110]])  # m > 15 on the device
