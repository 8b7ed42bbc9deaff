"""GPU parity of Algorithm 1 on the device (k6_odometer.cu + kbasis.cpp): the
reference's own search (kernel basis -> combination-space odometer ->
wpm_counts_ok, search.hpp:141-258) with every leaf on the B200.

* per-map WPM counts, combination-space sizes (size_saturated) and kernel
  dimensions, and the byte-exact .cplx digests, against the reference's own
  outputs in golden.json["ubt"] (n = 2..7) -- so the basis built by
  kbasis.cpp is the reference's basis and the leaves are its leaves;
* the leaf count equals the sum of the combination spaces;
* Algorithm 1 and the ridge-driven DFS (kernel 3) give identical resident
  results; link pins (apply_link_constraints) and candidate_cap errors.
"""
import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _digest(wpm, p, res, n):
    h = hashlib.sha256()
    for i in range(res.num_maps):
        h.update(wpm.write_cplx_bytes(res, i, n + 4, n, p.universe(i)))
    return h.hexdigest()


@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7])
def test_alg1_matches_reference(wpm, golden, n):
    ref = golden["ubt"][str(n)]
    with wpm.Plan.orbits(n) as p:
        total = p.run_kernel_basis()
        st = p.kernel_basis_stats()
        res = p.fetch()
        assert total == ref["sum"]
        assert res.counts == [m["wpms"] for m in ref["maps"]]
        spaces = [p.combination_space(i) for i in range(res.num_maps)]
        assert [c["space"] for c in spaces] == [m["space"] for m in ref["maps"]]
        assert [c["s"] for c in spaces] == [m["s"] for m in ref["maps"]]
        assert st["leaves"] == sum(m["space"] for m in ref["maps"])
        assert res.duplicates == 0
        assert _digest(wpm, p, res, n) == ref["sha256"]


@pytest.mark.parametrize("n", [4, 6])
def test_alg1_equals_dfs(wpm, n):
    with wpm.Plan.orbits(n) as p:
        p.run()
        a = p.fetch()
        bits_a = a.bits.copy()
        p.run_kernel_basis()
        b = p.fetch()
        assert a.counts == b.counts
        assert np.array_equal(bits_a, b.bits)


def test_alg1_link_pins_match_dfs(wpm, oracle):
    # the octahedron link pinning of test_search.cpp:178-220 on the full
    # universe of 3-subsets of [6]
    uni = oracle.all_subsets_universe(6, 3)
    oct_f = sorted(((1 << a) | (1 << b) | (1 << c)) for a in (1, 4) for b in (2, 5) for c in (3, 6))
    req = [j for j, f in enumerate(uni) if f >> 1 & 1 and f in oct_f]
    forb = [j for j, f in enumerate(uni) if f >> 1 & 1 and f not in oct_f]
    with wpm.Plan.universes(6, 3, [uni], required=req, forbidden=forb) as p:
        p.run()
        a = p.fetch()
        bits_a = a.bits.copy()
        p.run_kernel_basis()
        b = p.fetch()
        assert a.total == b.total and np.array_equal(bits_a, b.bits)
        assert p.kernel_basis_stats()["leaves"] == p.combination_space(0)["space"]


def test_alg1_random_pins_vs_reference_port(wpm, oracle):
    import random
    rng = random.Random(20240809)
    uni_all = oracle.all_subsets_universe(6, 3)
    done = 0
    while done < 12:
        uni = [f for f in uni_all if rng.random() < 0.6]
        if len(uni) < 10:
            continue
        req = [j for j in range(len(uni)) if rng.random() < 0.1]
        forb = [j for j in range(len(uni)) if rng.random() < 0.1 and j not in req]
        rc, ref = oracle.enumerate_ref(6, 3, uni, -1, req, forb)
        if rc != 0:
            continue
        with wpm.Plan.universes(6, 3, [uni], required=req, forbidden=forb) as p:
            p.run_kernel_basis()
            r = p.fetch()
            assert r.total == ref["count"]
            assert p.combination_space(0)["space"] == ref["space"]
            if r.total:
                assert np.array_equal(r.bits, ref["bits"])
        done += 1


def test_alg1_candidate_cap(wpm):
    with wpm.Plan.orbits(5) as p:
        with pytest.raises(wpm.CapExceededError):
            p.run_kernel_basis(candidate_cap=1000)
