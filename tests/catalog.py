"""Small named complexes and constructions for the seedness tests -- TEST
INFRASTRUCTURE ONLY.  Restates catalog.hpp:11-47 and complex.hpp:122-170
(link / join / suspension / wedge) on facet masks (bit v = vertex v)."""
from __future__ import annotations

import random
from itertools import combinations
from typing import List, Tuple

Complex = Tuple[int, int, List[int]]  # (m, n, facet masks ascending)


def mask(*vs: int) -> int:
    x = 0
    for v in vs:
        x |= 1 << v
    return x


def full(m: int) -> int:
    return ((1 << m) - 1) << 1


def simplex_boundary(k: int) -> Complex:  # catalog.hpp:11-16
    f = full(k + 1)
    return k + 1, k, sorted(f & ~(1 << v) for v in range(1, k + 2))


def cycle_complex(m: int) -> Complex:  # catalog.hpp:19-24
    out = [mask(i, i + 1) for i in range(1, m)] + [mask(m, 1)]
    return m, 2, sorted(out)


def s0() -> Complex:
    return 2, 1, [mask(1), mask(2)]


def square() -> Complex:
    return cycle_complex(4)


def pentagon() -> Complex:
    return cycle_complex(5)


def hexagon() -> Complex:
    return cycle_complex(6)


def cross_polytope_boundary(d: int) -> Complex:  # catalog.hpp:38-45
    out = []
    for choice in range(1 << d):
        f = 0
        for i in range(d):
            f |= 1 << ((i + 1 + d) if (choice >> i) & 1 else (i + 1))
        out.append(f)
    return 2 * d, d, sorted(out)


def octahedron() -> Complex:
    return cross_polytope_boundary(3)


def join(K: Complex, L: Complex) -> Complex:  # complex.hpp:131-139
    mk, nk, fk = K
    ml, nl, fl = L
    return mk + ml, nk + nl, sorted(f | (g << mk) for f in fk for g in fl)


def suspension(K: Complex) -> Complex:  # complex.hpp:142-145
    return join(K, s0())


def wedge(K: Complex, v: int) -> Complex:  # complex.hpp:153-168
    m, n, fs = K
    w = m + 1
    out = []
    for f in fs:
        if f >> v & 1:
            out.append(f | (1 << w))
        else:
            out.append(f | (1 << v))
            out.append(f | (1 << w))
    return m + 1, n + 1, sorted(set(out))


def random_pure(rng: random.Random, m: int, n: int, density: float) -> Complex:
    allf = [mask(*c) for c in combinations(range(1, m + 1), n)]
    fs = [f for f in allf if rng.random() < density]
    return m, n, sorted(fs)


def relabel(K: Complex, perm: List[int]) -> Complex:
    m, n, fs = K
    out = []
    for f in fs:
        g = 0
        for v in range(1, m + 1):
            if f >> v & 1:
                g |= 1 << perm[v]
        out.append(g)
    return m, n, sorted(out)


# ---- BASELINE configs[4]: synthetic candidate-facet sets
M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def synthetic_universe(seed: int, density: float, m: int = 15, n: int = 11) -> List[int]:
    """Facet j of the all-subsets universe of (m, n) (ascending masks,
    catalog.hpp:112-120) is kept iff splitmix64(seed ^ j) * 2^-64 < density."""
    thr = int(density * (1 << 64))
    allf = [mask(*c) for c in combinations(range(1, m + 1), n)]
    allf.sort()
    return [f for j, f in enumerate(allf) if splitmix64(seed ^ j) < thr]
