"""CPU tests: pin the oracle against the reference's golden vectors and
known-answer tests, check the two CPU restatements against each other and
against brute force, and check the library's host-side functions.  No GPU."""
import hashlib
import os
import random
import subprocess

import numpy as np
import pytest

from conftest import ROOT

REF_BIN = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")


# ------------------------------------------------------------ orbit / maps

def test_orbit_counts(oracle):
    """acceptance.cpp criterion 1 / test_charmap.cpp:154-159."""
    assert [len(oracle.idcm_orbits(n)) for n in range(2, 12)] == [7, 16, 28, 35, 35, 28, 16, 7, 3, 1]


def test_orbits_match_golden(oracle, golden):
    for n in range(2, 12):
        assert oracle.idcm_orbits(n) == golden["orbits"][str(n)]


def test_map_representatives_app_c(oracle):
    """SURVEY App. C known answers (rows and lambda columns)."""
    o2 = oracle.idcm_orbits(2)
    assert [r[:2] for r in o2] == [[3, 5], [3, 7], [3, 12], [3, 13], [3, 15], [7, 11], [7, 15]]
    assert oracle.charmap_of_dcm(o2[0]) == [1, 2, 3, 1, 2, 0]
    assert oracle.charmap_of_dcm(o2[1]) == [1, 2, 3, 3, 2, 0]
    assert oracle.charmap_of_dcm(o2[5]) == [1, 2, 3, 3, 1, 2]
    o10 = oracle.idcm_orbits(10)
    assert [r[:10] for r in o10] == [[3, 5, 6, 7, 9, 10, 11, 12, 13, 14], [3, 5, 6, 7, 9, 10, 11, 12, 13, 15],
                                     [3, 5, 6, 7, 9, 10, 11, 13, 14, 15]]
    assert oracle.charmap_of_dcm(o10[0])[10:] == [347, 621, 910, 1008]
    o11 = oracle.idcm_orbits(11)
    assert o11[0] == [3, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 1, 2, 4, 8]
    assert oracle.charmap_of_dcm(o11[0])[11:] == [1371, 1645, 1934, 2032]
    # n=2 map0: column 6 is zero (a loop); universe {12,13,23,24,34,15,35,45}
    u = oracle.matroid_universe(o2[0])
    as_pairs = [tuple(v for v in range(1, 16) if (f >> v) & 1) for f in u]
    assert as_pairs == [(1, 2), (1, 3), (2, 3), (2, 4), (3, 4), (1, 5), (3, 5), (4, 5)]


def test_binary_matroid_known_answers(oracle):
    """test_charmap.cpp:49-77."""
    assert oracle.binary_matroid(2, [1, 2, 3]) == [0b0110, 0b1010, 0b1100]
    assert oracle.binary_matroid(2, [1, 2, 1]) == [0b0110, 0b1100]
    with pytest.raises(ValueError):
        oracle.binary_matroid(2, [1, 1, 1])
    rows = oracle.idcm_orbits(11)[0]
    indep = 0
    import itertools

    def rank(vs):
        basis = {}
        r = 0
        for v in vs:
            x = v
            while x:
                b = x.bit_length() - 1
                if b in basis:
                    x ^= basis[b]
                else:
                    basis[b] = x
                    r += 1
                    break
        return r

    for q in itertools.combinations(rows, 4):
        indep += rank(q) == 4
    u = oracle.matroid_universe(rows)
    assert len(u) == indep and indep < 1365


def test_universe_sizes_and_digests(oracle, golden):
    """Kernel-1 golden: universe sizes per map (from the reference run)."""
    for n in range(2, 8):
        Ms = [len(oracle.matroid_universe(r)) for r in golden["orbits"][str(n)]]
        assert Ms == [m["M"] for m in golden["ubt"][str(n)]["maps"]]
    # whole-n universe digests, SURVEY App. C
    exp = {2: "c32f2f8255201fb672248da54866c5043672a59703636fd740ebf378741a101e",
           5: "5ae4dbb465a2789aa05694b69f44717a977076a24252f658d50e8b99a4bf3ad7"}
    for n, d in exp.items():
        h = hashlib.sha256()
        for r in golden["orbits"][str(n)]:
            u = oracle.matroid_universe(r)
            bits = np.zeros((1, (len(u) + 63) // 64), dtype=np.uint64)
            for j in range(len(u)):
                bits[0, j >> 6] |= np.uint64(1) << np.uint64(j & 63)
            h.update(oracle.write_cplx(n + 4, n, u, bits))
        assert h.hexdigest() == d


# ------------------------------------------------------------ UBT cap

def _gale_even(s, n, N):
    """catalog.hpp:76-90 restated."""
    if bin(s).count("1") != n:
        return False
    for i in range(1, N + 1):
        if (s >> i) & 1:
            continue
        for j in range(i + 1, N + 1):
            if (s >> j) & 1:
                continue
            if sum((s >> k) & 1 for k in range(i + 1, j)) & 1:
                return False
    return True


def test_ubt_bound(oracle, wpm):
    """test_search.cpp:54-68 (closed form == Gale evenness count)."""
    assert [oracle.cyclic_facet_bound(n) for n in (2, 3, 4)] == [6, 10, 20]
    for n in range(2, 12):
        N = n + 4
        cnt = sum(1 for s in range(1 << (N + 1)) if not s & 1 and _gale_even(s, n, N))
        assert oracle.cyclic_facet_bound(n) == cnt == wpm.cyclic_facet_bound(n)
    g = wpm.ubt_property(2, 15)
    assert g.constant == 7 and g.is_count_cap()


# ------------------------------------------------------------ enumeration oracles

@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_port_matches_reference_golden(oracle, golden, n):
    """The C restatement of the reference algorithm reproduces the reference's
    per-map counts and .cplx digests (UBT cap)."""
    h = hashlib.sha256()
    per = []
    for i, rows in enumerate(golden["orbits"][str(n)]):
        u = oracle.matroid_universe(rows)
        rc, r = oracle.enumerate_ref(n + 4, n, u, oracle.cyclic_facet_bound(n))
        assert rc == 0
        g = golden["ubt"][str(n)]["maps"][i]
        assert (r["count"], r["space"], r["s"]) == (g["wpms"], g["space"], g["s"])
        b = oracle.write_cplx(n + 4, n, u, r["bits"])
        per.append(hashlib.sha256(b).hexdigest())
        h.update(b)
    assert per == golden["ubt"][str(n)]["map_sha256"]
    assert h.hexdigest() == golden["ubt"][str(n)]["sha256"]


@pytest.mark.parametrize("n", [2, 3, 4])
def test_dfs_port_matches_reference_port(oracle, golden, n):
    """The device search restated (dfs_port) == the reference restated, bit-exact."""
    for i, rows in enumerate(golden["orbits"][str(n)]):
        u = oracle.matroid_universe(rows)
        cap = oracle.cyclic_facet_bound(n)
        rc, r = oracle.enumerate_ref(n + 4, n, u, cap)
        cnt, nodes, bits = oracle.dfs(n, u, cap)
        assert np.array_equal(bits, r["bits"]) and nodes == golden["dfs"][str(n)]["maps"][i]["nodes"]


def test_dfs_port_counts_n5_nocap(oracle, golden):
    for i, rows in enumerate(golden["orbits"]["4"]):
        u = oracle.matroid_universe(rows)
        cnt, _, _ = oracle.dfs(4, u, -1, want_bits=False)
        assert cnt == golden["nocap"]["4"]["counts"][i]


def test_small_examples(oracle):
    """test_search.cpp:104-121, :269-274."""
    u = oracle.all_subsets_universe(4, 2)
    rc, r = oracle.enumerate_ref(4, 2, u)
    assert r["count"] == 7
    cnt, _, bits = oracle.dfs(2, u)
    assert cnt == 7 and np.array_equal(bits, r["bits"])
    s3 = oracle.all_subsets_universe(4, 3)
    cnt, _, bits = oracle.dfs(3, s3)
    assert cnt == 1 and int(bits[0, 0]) == 0b1111
    assert oracle.dfs(2, [0b00110, 0b11000])[0] == 0
    assert oracle.enumerate_ref(4, 2, [0b00110, 0b11000])[1]["count"] == 0


def test_cap_exceeded(oracle):
    """test_search.cpp:263-267: the reference throws past candidate_cap."""
    rc, _ = oracle.enumerate_ref(6, 2, oracle.all_subsets_universe(6, 2), candidate_cap=16)
    assert rc == 5


def test_acceptance_criterion5(oracle):
    """acceptance.cpp:243-320: full-subset and random universes + constrained
    variants against the Gray-code brute force, for both restatements."""
    for m, n in [(4, 2), (5, 2), (6, 2), (7, 2), (4, 3), (5, 3), (6, 3), (6, 4), (5, 4), (6, 5), (7, 5), (7, 6)]:
        u = oracle.all_subsets_universe(m, n)
        brute = oracle.brute_force_count(u)
        rc, r = oracle.enumerate_ref(m, n, u)
        cnt, _, bits = oracle.dfs(n, u)
        assert r["count"] == brute == cnt and np.array_equal(bits, r["bits"])
    rng = random.Random(20240809)
    made = 0
    while made < 10:
        m, n = 6 + rng.randrange(3), 2 + rng.randrange(3)
        if n >= m:
            continue
        u = [f for f in oracle.all_subsets_universe(m, n) if rng.randrange(3) == 0]
        if not 8 <= len(u) <= 24:
            continue
        made += 1
        brute = oracle.brute_force_count(u)
        rc, r = oracle.enumerate_ref(m, n, u)
        cnt, _, bits = oracle.dfs(n, u)
        assert r["count"] == brute == cnt and np.array_equal(bits, r["bits"])
    made = 0
    while made < 8:
        u = [f for f in oracle.all_subsets_universe(6, 3) if rng.randrange(2) == 0]
        if not 10 <= len(u) <= 18:
            continue
        req, forb = [], []
        for j in range(len(u)):
            roll = rng.randrange(10)
            if roll == 0:
                req.append(j)
            elif roll == 1:
                forb.append(j)
        made += 1
        brute = oracle.brute_force_count(u, req, forb)
        cnt, _, bits = oracle.dfs(3, u, -1, req, forb)
        assert cnt == brute
        rc, r = oracle.enumerate_ref(6, 3, u, -1, req, forb)
        if rc == 3:  # apply_link_constraints -> nullopt
            assert brute == 0
        else:
            assert r["count"] == brute and np.array_equal(bits, r["bits"])


def test_direct_recount(oracle):
    """test_search.cpp:222-243: every output passes is_weak_pseudomanifold_direct."""
    rows = oracle.idcm_orbits(4)[3]
    u = oracle.matroid_universe(rows)
    cnt, _, bits = oracle.dfs(4, u, oracle.cyclic_facet_bound(4))
    for row in bits[:500]:
        fs = [u[j] for j in range(len(u)) if (int(row[j >> 6]) >> (j & 63)) & 1]
        assert oracle.is_wpm_direct(fs)


def test_canonical_compare(oracle):
    """po_bits_cmp == lexicographic order of ascending index lists (prefix first)."""
    rng = random.Random(5)
    for _ in range(2000):
        W = rng.choice([1, 2, 3])
        a = [j for j in range(64 * W) if rng.random() < 0.05]
        b = list(a) if rng.random() < 0.3 else [j for j in range(64 * W) if rng.random() < 0.05]
        if rng.random() < 0.3 and a:
            b = a[: rng.randrange(len(a) + 1)]
        A = np.zeros(W, dtype=np.uint64)
        B = np.zeros(W, dtype=np.uint64)
        for j in a:
            A[j >> 6] |= np.uint64(1) << np.uint64(j & 63)
        for j in b:
            B[j >> 6] |= np.uint64(1) << np.uint64(j & 63)
        exp = (tuple(a) > tuple(b)) - (tuple(a) < tuple(b))
        got = oracle.bits_cmp(A, B)
        assert (got > 0) - (got < 0) == exp


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="reference driver not built")
def test_reference_driver_orbits(oracle):
    """oracle/_ref (the unmodified reference) agrees with the restatement."""
    for n in (2, 5, 11):
        out = subprocess.run([REF_BIN, "orbits", str(n)], check=True, capture_output=True, text=True).stdout
        rows = [[int(x) for x in ln.split()] for ln in out.splitlines()]
        assert rows == oracle.idcm_orbits(n)


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="reference driver not built")
def test_reference_driver_n4_digest(golden):
    out = subprocess.run([REF_BIN, "enumerate", "4", "--out", "/dev/stdout"], check=True, capture_output=True).stdout
    # stdout mixes the summary lines after the bytes; recompute via a file instead
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "o.cplx")
        subprocess.run([REF_BIN, "enumerate", "4", "--out", p], check=True, capture_output=True)
        assert hashlib.sha256(open(p, "rb").read()).hexdigest() == golden["ubt"]["4"]["sha256"]
    assert out


def test_golden_consistency(golden):
    """Reference counts (n <= 7, and n = 8 maps run so far) == DFS-restatement counts."""
    for n in range(2, 8):
        assert [m["wpms"] for m in golden["ubt"][str(n)]["maps"]] == [m["wpms"] for m in golden["dfs"][str(n)]["maps"]]
    if "8" in golden["ubt"]:
        ref8 = golden["ubt"]["8"]
        k = len(ref8["maps"])
        assert [m["wpms"] for m in ref8["maps"]] == [m["wpms"] for m in golden["dfs"]["8"]["maps"][:k]]
        assert ref8["map_sha256"] == [m["sha256"] for m in golden["dfs"]["8"]["maps"][:k]]
    exp = {6: "c227c84d679b2697bfa6027301c8d3e250f4a7d5c8ca83cf8d820692f5e2f518",
           7: "51074c71bb01081bd69b00220f69d172fa275f65c233987a931114d42d32a935"}
    for n, d in exp.items():
        assert golden["ubt"][str(n)]["sha256"] == d


# ------------------------------------------------------------ library host side

def test_library_host_functions(wpm, oracle):
    """idcm_orbits / charmap_of_dcm / cyclic_facet_bound in the product's host
    C++ equal the restatement (no GPU needed)."""
    for n in range(2, 12):
        got = wpm.idcm_orbits(n)
        assert [d.rows for d in got] == oracle.idcm_orbits(n)
        for d in got[:3]:
            assert wpm.charmap_of_dcm(d) == oracle.charmap_of_dcm(d.rows)
    # general (non standard form) dual matrix
    d = wpm.DualCharMatrix(6, 4, [1, 2, 4, 8, 3, 5])
    assert wpm.charmap_of_dcm(d) == oracle.charmap_of_dcm(d.rows)
    with pytest.raises(ValueError):
        wpm.idcm_orbits(12)


def test_write_complexes_format(wpm):
    """complex_io.hpp:21-39 byte format."""
    s = wpm.write_complexes(6, 2, [[0b0110, 0b1010, 0b1100], [0b0110]])
    assert s == "6 2\n1 2\n1 3\n2 3\n\n6 2\n1 2\n"


def test_charmap_of_dcm_general_branch(wpm, oracle):
    """charmap_of_dcm's general kernel branch (charmap.hpp:171-203), taken when
    the last p rows are not the identity: the product's host code equals the
    restatement on row-permuted orbit representatives and on random rank-p
    dual matrices; rank-deficient inputs are rejected by both."""
    import random

    rng = random.Random(4)
    checked = 0
    for n in (2, 3, 5, 7):
        for d in wpm.idcm_orbits(n, 4)[:6]:
            rows = list(d.rows)
            rng.shuffle(rows)
            if rows[-4:] == [1, 2, 4, 8]:
                continue
            dd = wpm.DualCharMatrix(d.m, 4, rows)
            assert wpm.charmap_of_dcm(dd) == oracle.charmap_of_dcm(rows), (n, rows)
            checked += 1
    for _ in range(200):
        m = rng.randrange(6, 14)
        rows = [rng.randrange(1, 16) for _ in range(m)]
        dd = wpm.DualCharMatrix(m, 4, rows)
        try:
            want = oracle.charmap_of_dcm(rows)
        except ValueError:
            with pytest.raises(ValueError):
                wpm.charmap_of_dcm(dd)
            continue
        assert wpm.charmap_of_dcm(dd) == want, rows
        checked += 1
    assert checked > 100


def test_alg1_n10_chunks_recorded(golden):
    """The exhaustive Algorithm-1 chunks recorded at n = 10 (tools/alg1_full.py
    on the device): every chunk's accepted set equals the DFS rows sharing its
    prefix, chunks are distinct, and a map whose chunks are all recorded adds
    up to its golden WPM count and to its whole combination space."""
    import json
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tools"))
    from alg1_full import chunks_of

    path = os.path.join(os.path.dirname(__file__), "golden", "alg1_n10_chunks.jsonl")
    recs = [json.loads(ln) for ln in open(path) if ln.strip()]
    assert recs, "no recorded chunks"
    seen = set()
    for r in recs:
        assert r["n"] == 10 and r["equal"] and r["odometer"] == r["dfs"]
        key = (r["map"], tuple(r["prefix"]))
        assert key not in seen
        seen.add(key)
    # the chunking: fix outer blocks until a chunk has <= the leaf budget
    j, pre = chunks_of([4, 4, 3, 1], 100)  # 11 * 11 * 7 * 2 leaves
    assert j == 2 and len(pre) == 121 and pre[0] == (0, 0) and pre[-1] == (10, 10)
    assert chunks_of([2, 1], 100) == (0, [()])
    for m, mrec in enumerate(golden["dfs"]["10"]["maps"]):
        mine = [r for r in recs if r["map"] == m]
        # the widest two blocks have width 4 at n = 10: 11 x 11 chunks cover the map
        if len(mine) == 121:
            assert sum(r["odometer"] for r in mine) == mrec["wpms"]
            assert len({r["leaves"] for r in mine}) == 1
