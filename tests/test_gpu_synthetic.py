"""BASELINE.json configs[4]: synthetic candidate-facet sets at (m, n) =
(15, 11), density sweep, on the device through the
C-ABI.

* d <= 0.73, seeds 1..8: count and the .cplx SHA-256 of every universe
  equal the reference's own enumerate_wpm output (golden.json["synthetic"],
  tests/golden/make_golden_synthetic.py);
* d = 0.75 / 0.78: count, node count and digest equal the CPU restatement of
  the device search (the reference's search does not finish there);
* above the checkable band (d = 0.82 .. 1.0) a node-budgeted stress run:
  the run stops at the budget, and every WPM it emitted is a sound WPM of
  the universe (direct recount, complex.hpp:224-233) within the cap, with no
  duplicates -- a throughput / divergence stress, no completeness claim.
"""
import hashlib

import numpy as np
import pytest

import catalog as C

pytestmark = pytest.mark.gpu


def _cases(golden, pred):
    return [c for c in golden["synthetic"]["cases"] if pred(c)]


def _digest(wpm, oracle, u, res):
    if res.total == 0:
        return hashlib.sha256(b"").hexdigest()
    return hashlib.sha256(oracle.write_cplx(15, 11, u, res.map_bits(0))).hexdigest()


@pytest.mark.parametrize("d", [0.60, 0.65, 0.70, 0.72, 0.73, 0.75, 0.78])
def test_synthetic_density_parity(wpm, oracle, golden, d):
    cases = _cases(golden, lambda c: abs(c["d"] - d) < 1e-9)
    assert cases
    for c in cases:
        u = C.synthetic_universe(c["seed"], d)
        assert len(u) == c["M"]
        with wpm.Plan.universes(15, 11, [u], facet_cap=golden["synthetic"]["cap"]) as p:
            total = p.run()
            st = p.stats()
            res = p.fetch()
        assert total == c["wpms"] and res.duplicates == 0, (d, c["seed"])
        assert st["nodes"] == c["nodes"], (d, c["seed"])
        assert _digest(wpm, oracle, u, res) == c["sha256"], (d, c["seed"])


@pytest.mark.parametrize("d", [0.82, 0.9, 1.0])
def test_synthetic_budgeted_stress(wpm, oracle, d):
    u = C.synthetic_universe(1, d)
    budget = 200_000_000
    with wpm.Plan.universes(15, 11, [u], facet_cap=252) as p:
        p.set_node_budget(budget)
        p.run()
        st = p.stats()
        res = p.fetch()
        truncated = p.truncated()
    assert st["nodes"] >= (budget if truncated else 0)
    assert res.duplicates == 0
    rng = np.random.default_rng(int(d * 100))
    rows = res.map_bits(0)
    for i in rng.choice(len(rows), size=min(len(rows), 300), replace=False) if len(rows) else []:
        facets = wpm.bits_to_facets(rows[i], u)
        assert 11 + 1 <= len(facets) <= 252
        assert oracle.is_wpm_direct(facets)


def test_node_budget_truncates_and_resets(wpm, golden):
    """n = 8 orbit maps: a small budget stops the run early (truncated), a
    zero budget enumerates everything again."""
    with wpm.Plan.orbits(8) as p:
        p.set_node_budget(1_000_000)
        p.run()
        assert p.truncated() and p.stats()["nodes"] >= 1_000_000
        p.set_node_budget(0)
        assert p.run() == golden["dfs"]["8"]["sum"] and not p.truncated()
        assert p.stats()["nodes"] == golden["dfs"]["8"]["nodes"]
