"""CPU checks of the line-15 oracle (oracle/line15_port.c) -- the literal C
restatement of refine_classes / canonical_form (isomorphism.hpp:162-303) that
the device kernel is compared with.

* the first-appearance representatives and every survivor's canonical form
  for n = 2, 3 equal the reference's (golden.json["line15"], produced by the
  reference itself on the golden line-13 survivors);
* canonical forms decide isomorphism: equal iff brute_force_isomorphic
  (isomorphism.hpp:138-156) on small random complexes and relabelings;
* refine_classes equals the reference's own (oracle/_ref plseeds_ref classes)
  when the compiled reference is present (dev container).
"""
import hashlib
import itertools
import os
import random
import subprocess
import tempfile

import numpy as np
import pytest

import catalog as C
from conftest import ROOT
from oracle_bind import read_cplx

REF = os.path.join(ROOT, "oracle", "_ref", "plseeds_ref")


def _survivor_rows(oracle, golden, n):
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    from make_golden_line13 import global_rows

    m = n + 4
    all_sub = oracle.all_subsets_universe(m, n)
    rows = []
    for r in golden["orbits"][str(n)]:
        uni = oracle.matroid_universe(r)
        _, _, bits = oracle.dfs(n, uni, oracle.cyclic_facet_bound(n))
        rows.append(global_rows(oracle, n, uni, bits, all_sub))
    _, _, surv = oracle.line13(m, n, np.concatenate(rows))
    return all_sub, surv


@pytest.mark.parametrize("n", [2, 3])
def test_oracle_line15_matches_reference_goldens(oracle, golden, n):
    want = golden["line15"][str(n)]
    m = n + 4
    all_sub, surv = _survivor_rows(oracle, golden, n)
    assert surv.shape[0] == want["line13"]
    canon, reps = oracle.line15(m, n, surv)
    assert len(reps) == want["line15"] == want["paper_line15"]
    assert hashlib.sha256(oracle.write_cplx(m, n, all_sub, canon)).hexdigest() == want["canon_sha256"]
    assert hashlib.sha256(oracle.write_cplx(m, n, all_sub, canon[reps])).hexdigest() == want["sha256"]


def _brute_iso(m, A, B):
    if len(A) != len(B):
        return False
    sb = sorted(B)
    for perm in itertools.permutations(range(1, m + 1)):
        img = sorted(sum(1 << perm[v - 1] for v in range(1, m + 1) if f >> v & 1) for f in A)
        if img == sb:
            return True
    return False


def test_canonical_form_decides_isomorphism(oracle):
    rng = random.Random(7)
    for _ in range(60):
        m = rng.randint(4, 6)
        n = rng.randint(2, m - 1)
        allf = [C.mask(*c) for c in itertools.combinations(range(1, m + 1), n)]
        k = rng.randint(1, len(allf))
        A = sorted(rng.sample(allf, k))
        if rng.random() < 0.5:
            tail = list(range(1, m + 1))
            rng.shuffle(tail)
            B = C.relabel((m, n, A), [0] + tail)[2]
        else:
            B = sorted(rng.sample(allf, k))
        ca, _ = oracle.canonical_form(m, A)
        cb, _ = oracle.canonical_form(m, B)
        assert (ca == cb) == _brute_iso(m, A, B), (m, n, A, B)
        assert ca == oracle.canonical_form(m, ca)[0]  # idempotent


@pytest.mark.skipif(not os.path.exists(REF), reason="compiled reference (oracle/_ref) not present")
def test_refine_classes_matches_reference(oracle):
    rng = random.Random(11)
    cases = [C.octahedron(), C.pentagon(), C.suspension(C.pentagon()), C.join(C.square(), C.pentagon()),
             C.wedge(C.hexagon(), 3), C.cross_polytope_boundary(4)]
    for _ in range(40):
        m = rng.randint(5, 10)
        n = rng.randint(2, min(5, m - 1))
        cases.append(C.random_pure(rng, m, n, rng.choice([0.2, 0.5, 0.8])))
    cases = [K for K in cases if K[2]]
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "k.cplx")
        with open(path, "w") as f:
            f.write("\n".join(f"{m} {n}\n" + "".join(" ".join(str(v) for v in range(1, m + 1) if x >> v & 1) + "\n"
                                                     for x in fs) for m, n, fs in cases))
        back = read_cplx(open(path, "rb").read())
        assert [b[2] for b in back] == [K[2] for K in cases]
        out = subprocess.run([REF, "classes", path], capture_output=True, text=True, check=True).stdout.split("\n")
    for (m, n, fs), line in zip(cases, out):
        assert oracle.refine_classes(m, fs) == [int(x) for x in line.split()], (m, n, fs)
