"""SURVEY 8(c)(1)-(3) on the device for every n, and the pinned n = 10 / 11
records: the parity protocol where the reference cannot finish.

(1) soundness of EVERY emitted row (kernel 8: direct WPM recount, cap, inside
    the universe), n = 2..11;
(2) reachability of every row in the reference's convenient basis (<= 2
    generators per induced block, kernel_basis.hpp:84-235, search.hpp:81-104);
(3) two-sided completeness on sampled outer prefixes: the reference's inner
    odometer (search.hpp:204-243, every leaf on the device) accepts exactly
    the DFS rows whose coordinates share the prefix.  The sampled prefixes and
    both sides' counts are recorded in golden.json["reach"]
    (tests/golden/make_golden_reach.py) and re-checked here."""
import numpy as np
import pytest

from reach_protocol import block_candidates, run_protocol

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", list(range(2, 12)))
def test_every_row_sound_and_reachable(wpm, golden, n):
    with wpm.Plan.orbits(n) as p:
        total = p.run()
        unsound, unreach, coords = p.verify(reach=True, coords=True)
    assert total == golden["dfs"][str(n)]["sum"]
    assert unsound == 0 and unreach == 0, (unsound, unreach)
    assert coords.shape[0] == total and np.count_nonzero(coords) == total  # every WPM is a nonzero cycle


def test_prefix_candidates_roundtrip(wpm):
    """Coordinates -> reference candidate indices: the odometer run on a row's
    full candidate list (no inner blocks) returns exactly that row."""
    with wpm.Plan.orbits(4) as p:
        p.run()
        res = p.fetch()
        _, _, coords = p.verify(reach=True, coords=True)
        for i in range(p.num_maps):
            widths = p.space_blocks(i)
            lo, hi = res.offsets[i], res.offsets[i + 1]
            cands = block_candidates(coords[lo:hi], widths, len(widths))
            assert (cands >= 0).all()
            for r in range(0, hi - lo, max(1, (hi - lo) // 5)):
                assert p.run_kernel_basis_prefix(i, [int(c) for c in cands[r]]) == 1
                assert np.array_equal(p.fetch().map_bits(i), res.map_bits(i)[r:r + 1])


@pytest.mark.parametrize("n,samples,leaves", [(6, 12, 1 << 26), (8, 16, 1 << 31)])
def test_prefix_completeness_small_n(wpm, n, samples, leaves):
    """The protocol where the reference ran in full (n <= 8): a cross-check of
    the protocol itself."""
    r = run_protocol(wpm, n, samples, leaves)
    assert r["unsound"] == 0 and r["unreachable"] == 0
    assert all(s["equal"] and s["odometer"] == s["dfs"] >= 1 for s in r["samples"]), r["samples"]


@pytest.mark.parametrize("n", [10, 11])
def test_prefix_completeness_pinned(wpm, golden, n):
    """n = 10 / 11: the recorded sampled prefixes, two-sided, with the recorded
    counts (golden.json["reach"], >= 200 prefixes per n)."""
    rec = golden.get("reach", {}).get(str(n))
    if rec is None:
        pytest.skip("golden.json has no reach record (tests/golden/make_golden_reach.py)")
    r = run_protocol(wpm, n, rec["samples_requested"], rec["max_leaves"], seed=rec["seed"])
    assert r["rows"] == rec["rows"] and r["unsound"] == 0 and r["unreachable"] == 0
    assert len(r["samples"]) == len(rec["samples"]) >= 200
    for got, want in zip(r["samples"], rec["samples"]):
        assert got["equal"], got
        assert (got["map"], got["prefix"], got["odometer"], got["dfs"]) == \
            (want["map"], want["prefix"], want["odometer"], want["dfs"])
