"""CPU checks of the synthetic configs (BASELINE.json configs[4]): the
portable generator (splitmix64) and the oracle
restatements against the reference-produced goldens at low density."""
import pytest

import catalog as C


def test_splitmix64_known_answers():
    # the reference splitmix64 sequence from state 0 (Vigna): first outputs
    assert C.splitmix64(0) == 0xE220A8397B1DCDAF
    assert C.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_synthetic_universe_sizes(golden):
    for c in golden["synthetic"]["cases"]:
        u = C.synthetic_universe(c["seed"], c["d"])
        assert len(u) == c["M"] and u == sorted(u)
        assert all(bin(f).count("1") == 11 and f >> 16 == 0 and f & 1 == 0 for f in u)


@pytest.mark.parametrize("d", [0.60, 0.65, 0.70, 0.72])
def test_dfs_port_matches_reference_goldens(oracle, golden, d):
    import hashlib

    for c in golden["synthetic"]["cases"]:
        if abs(c["d"] - d) > 1e-9:
            continue
        assert c["source"].startswith("oracle/_ref")
        u = C.synthetic_universe(c["seed"], d)
        cnt, nodes, bits = oracle.dfs(11, u, 252)
        assert (cnt, nodes) == (c["wpms"], c["nodes"])
        data = oracle.write_cplx(15, 11, u, bits) if cnt else b""
        assert hashlib.sha256(data).hexdigest() == c["sha256"]
