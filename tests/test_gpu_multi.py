"""The split below the root, the shared-frontier claims (the multi-GPU
protocol) and the boundary features the reference's SearchJob
has (progress, any universe order), through the C-ABI on the device.

Only one GPU is available here, so the multi-GPU job runs its "GPUs" as
plans on the same device: every plan's kernel pulls frontier records from
one shared claim counter and no kernel ever waits for another, so the
protocol is exercised exactly (B200_PROFILING: no cross-rank waiting)."""
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.counts == b.counts and a.total == b.total
    assert np.array_equal(a.bits, b.bits)


@pytest.mark.parametrize("n,depth", [(4, 2), (5, 3), (7, 4), (8, 5), (11, 6)])
def test_split_then_search(wpm, golden, n, depth):
    """Split at a branch depth, then search the frontier: the same tree --
    identical node count, rows and per-map counts."""
    with wpm.Plan.orbits(n) as p:
        p.set_split(depth)
        assert p.run() == golden["dfs"][str(n)]["sum"]
        res = p.fetch()
    assert res.nodes == golden["dfs"][str(n)]["nodes"] and res.duplicates == 0
    assert res.counts == [m["wpms"] for m in golden["dfs"][str(n)]["maps"]]


@pytest.mark.parametrize("n,ndev", [(5, 2), (8, 3), (11, 2), (9, 4)])
def test_multi_device_job_same_gpu(wpm, golden, n, ndev):
    """wpm_plan_create_orbits_multi with every 'GPU' = device 0: split on the
    leader, frontier copied to each plan, shared claim counter, rows gathered
    into the leader and sorted once.  Bit-exact with the 1-GPU run; node
    counts add up over the devices."""
    with wpm.Plan.orbits(n) as p:
        p.run()
        want = p.fetch()
    with wpm.Plan.orbits(n, devices=[0] * ndev) as p:
        assert p.run() == want.total
        got = p.fetch()
        per = p.device_stats()
    _same(got, want)
    assert got.nodes == want.nodes == golden["dfs"][str(n)]["nodes"] and got.duplicates == 0
    assert len(per) == ndev and sum(x[1] for x in per) <= got.nodes


def test_claim_protocol_single_rank(wpm, golden):
    """The cross-process protocol with one rank: split, the IPC-capable claim
    counter, run_claim -- the same rows and nodes."""
    n = 8
    with wpm.Plan.orbits(n) as p:
        p.run()
        want = p.fetch()
        f = p.split(3, 2048)
        assert f >= 1024  # within 2x of the target
        ctr, handle = wpm.claim_counter_create(0)
        assert len(handle) == 64
        try:
            assert p.run_claim(ctr) == want.total
            got = p.fetch()
        finally:
            wpm.claim_counter_close(0, ctr, False)
    _same(got, want)
    assert got.nodes == want.nodes


def test_claim_two_plans_sequential(wpm):
    """Two plans share one frontier and one counter, run one after the other
    (no concurrency needed): the first takes every record, the second finds
    the counter exhausted; the union is the full result."""
    n = 6
    with wpm.Plan.orbits(n) as a, wpm.Plan.orbits(n) as b:
        a.run()
        want = a.fetch()
        f = a.split(3, 1024)
        ptr, cnt, recw = a.frontier()
        b.load_frontier(ptr, cnt)
        ctr, _ = wpm.claim_counter_create(0)
        try:
            ta = a.run_claim(ctr)
            tb = b.run_claim(ctr)
        finally:
            wpm.claim_counter_close(0, ctr, False)
        assert tb == 0 and ta == want.total and f == cnt
        _same(a.fetch(), want)


def test_claim_loaded_plan_claims_first(wpm):
    """A plan that did not split (wpm_plan_load_frontier + run_claim) claims
    the shared frontier itself: run first it takes every record, the
    splitting plan keeps only the rows found above the frontier; together
    they are the full result."""
    import numpy as np

    n = 6
    with wpm.Plan.orbits(n) as a, wpm.Plan.orbits(n) as b:
        a.run()
        want = a.fetch()
        a.split(3, 1024)
        ptr, cnt, recw = a.frontier()
        b.load_frontier(ptr, cnt)
        ctr, _ = wpm.claim_counter_create(0)
        try:
            tb = b.run_claim(ctr)
            ta = a.run_claim(ctr)
        finally:
            wpm.claim_counter_close(0, ctr, False)
        assert tb > 0 and ta + tb == want.total
        ra, rb = a.fetch(), b.fetch()
        for i in range(want.num_maps):
            got = np.concatenate([ra.map_bits(i), rb.map_bits(i)])
            rows = sorted(map(bytes, got))
            assert rows == sorted(map(bytes, want.map_bits(i))), i


@pytest.mark.parametrize("n", [5, 9])
def test_progress_callback(wpm, golden, n):
    """SearchJob::progress (search.hpp:54, :244): called while the search
    runs, monotone, the last call done == total."""
    calls = []
    with wpm.Plan.orbits(n) as p:
        p.set_progress(lambda d, t: calls.append((d, t)))
        p.run()
        assert p.fetch().total == golden["dfs"][str(n)]["sum"]
    assert calls and calls[-1][0] == calls[-1][1] > 0
    assert all(a[0] <= b[0] and a[1] == b[1] for a, b in zip(calls, calls[1:]))


def test_progress_through_job(wpm, oracle):
    calls = []
    u = oracle.all_subsets_universe(6, 3)
    out = wpm.enumerate_wpm(wpm.SearchJob(6, 3, u, progress=lambda d, t: calls.append((d, t))))
    assert out and calls[-1][0] == calls[-1][1]


def test_unsorted_universe_and_pins(wpm, oracle):
    """The reference accepts a universe in any order (incidence.hpp:34-55,
    search.hpp:247-257): the same canonical output, pins follow the caller's
    indices."""
    rng = random.Random(7)
    for n in (3, 4, 5):
        rows = oracle.idcm_orbits(n)[1]
        uni = oracle.matroid_universe(rows)
        shuf = uni[:]
        rng.shuffle(shuf)
        cap = oracle.cyclic_facet_bound(n)
        a = wpm.enumerate_wpm(wpm.SearchJob(n + 4, n, uni, properties=[wpm.ubt_property(n, len(uni))]))
        b = wpm.enumerate_wpm(wpm.SearchJob(n + 4, n, shuf, properties=[wpm.ubt_property(n, len(uni))]))
        assert a == b and len(a) == oracle.dfs(n, uni, cap)[0]
    u = oracle.all_subsets_universe(6, 3)
    octa = sorted(sum(1 << (i + 1 + (3 if (c >> i) & 1 else 0)) for i in range(3)) for c in range(8))
    perm = list(range(len(u)))
    rng.shuffle(perm)
    us = [u[i] for i in perm]
    req = [j for j, f in enumerate(us) if f & 2 and f in octa]
    forb = [j for j, f in enumerate(us) if f & 2 and f not in octa]
    pinned = wpm.enumerate_wpm(wpm.SearchJob(6, 3, us, required=req, forbidden=forb))
    full = wpm.enumerate_wpm(wpm.SearchJob(6, 3, u))
    filt = [K for K in full if all(us[j] in K for j in req) and not any(us[j] in K for j in forb)]
    assert pinned == filt and len(pinned) > 0


def test_job_devices_field(wpm, oracle):
    """wpm_job_t.devices: one job over several (here: the same) GPUs."""
    u = oracle.all_subsets_universe(7, 3)
    a = wpm.enumerate_wpm(wpm.SearchJob(7, 3, u, properties=[wpm.AffineProperty([-1] * len(u), 9)]))
    b = wpm.enumerate_wpm(wpm.SearchJob(7, 3, u, properties=[wpm.AffineProperty([-1] * len(u), 9)], devices=[0, 0]))
    assert a == b and len(a) > 0
