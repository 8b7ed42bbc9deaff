"""the parity protocol where the reference cannot run to
completion (n >= 10) -- TEST INFRASTRUCTURE.

(2) reachability: every emitted WPM has coordinates in the reference's
    convenient basis (kernel_basis.hpp:84-235) with at most two generators per
    induced block, i.e. it lies in combination_space(kb) (search.hpp:81-104)
    and enumerate_wpm would emit it.  Checked on the device for every row
    (Plan.verify(reach=True), kernel 8), which also returns the coordinates.
(3) prefix-sampled two-sided completeness: for sampled emitted WPMs, fix the
    reference candidates of the outermost (widest) blocks to that WPM's
    coordinates and run the reference's inner odometer over the remaining
    blocks (search.hpp:204-243, every leaf, on the device:
    Plan.run_kernel_basis_prefix).  The accepted set must EQUAL the set of
    DFS-emitted WPMs whose coordinates share the prefix.

Used by tests/test_gpu_reach.py and tests/golden/make_golden_reach.py.
"""
from __future__ import annotations

import numpy as np


def ncand(w: int) -> int:
    """candidates of a block of w generators: none, singles, pairs (search.hpp:88-93)."""
    return 1 + w + w * (w - 1) // 2


def block_candidates(coords: np.ndarray, widths, nblocks: int) -> np.ndarray:
    """Reference candidate index of the first `nblocks` blocks for every
    coordinate vector (uint64, bit g = usable generator g in block order).
    Rows using > 2 generators of a block get -1."""
    coords = np.asarray(coords, dtype=np.uint64)
    out = np.zeros((coords.shape[0], nblocks), dtype=np.int64)
    lo = 0
    for b in range(nblocks):
        w = widths[b]
        bits = [((coords >> np.uint64(lo + i)) & np.uint64(1)).astype(np.int64) for i in range(w)]
        cnt = sum(bits)
        cand = np.full(coords.shape[0], -1, dtype=np.int64)
        cand[cnt == 0] = 0
        for i in range(w):
            cand[(cnt == 1) & (bits[i] == 1)] = 1 + i
            for j in range(i + 1, w):
                cand[(cnt == 2) & (bits[i] == 1) & (bits[j] == 1)] = 1 + w + i * (2 * w - i - 1) // 2 + (j - i - 1)
        out[:, b] = cand
        lo += w
    return out


def prefix_length(widths, max_leaves: int) -> int:
    """Smallest number of fixed outer blocks whose remaining inner space has
    at most max_leaves leaves."""
    sizes = [ncand(w) for w in widths]
    for j in range(len(sizes) + 1):
        rest = 1
        for c in sizes[j:]:
            rest *= c
        if rest <= max_leaves:
            return j
    return len(sizes)


def run_protocol(wpm, n: int, samples: int, max_leaves: int, seed: int = 2301, log=None):
    """Runs (2) and (3) for every map of idcm_orbits(n, 4).  Returns a dict
    with the row count, the unsound / unreachable counts and one record per
    sampled prefix: map, prefix candidates, leaves of the inner space, the
    odometer's accepted count and the DFS count sharing the prefix, and
    whether the two sets are equal."""
    out = {"n": n, "samples": []}
    with wpm.Plan.orbits(n) as p:
        total = p.run()
        res = p.fetch()
        unsound, unreach, coords = p.verify(reach=True, coords=True)
        out.update({"rows": total, "unsound": unsound, "unreachable": unreach})
        rng = np.random.default_rng(seed + n)
        picks = np.sort(rng.choice(total, size=min(samples, total), replace=False))
        for row in picks:
            i = int(np.searchsorted(res.offsets, row, side="right") - 1)
            widths = p.space_blocks(i)
            j = prefix_length(widths, max_leaves)
            lo, hi = res.offsets[i], res.offsets[i + 1]
            cands = block_candidates(coords[lo:hi], widths, j)
            want = cands[row - lo]
            share = np.all(cands == want[None, :], axis=1)
            dfs_rows = res.map_bits(i)[share]
            got_total = p.run_kernel_basis_prefix(i, [int(c) for c in want])
            leaves = p.kernel_basis_stats()["leaves"]
            got = p.fetch().map_bits(i)
            equal = got.shape == dfs_rows.shape and np.array_equal(got, dfs_rows)
            rec = {"map": i, "row": int(row), "nfixed": j, "prefix": [int(c) for c in want], "leaves": int(leaves),
                   "odometer": int(got_total), "dfs": int(dfs_rows.shape[0]), "equal": bool(equal)}
            out["samples"].append(rec)
            if log:
                log(rec)
    return out
