"""Parity of the CUDA path (through the C-ABI) against the oracle and the
reference's golden vectors.  Bit-exact: the same canonical WPM lists, the same
per-map counts, the same `.cplx` bytes; node counts equal to the CPU
restatement of the device search."""
import hashlib
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _digest_plan(wpm, plan, res, n):
    h = hashlib.sha256()
    per = []
    for i in range(plan.num_maps):
        b = wpm.write_cplx_bytes(res, i, n + 4, n, plan.universe(i))
        per.append(hashlib.sha256(b).hexdigest())
        h.update(b)
    return h.hexdigest(), per


@pytest.mark.parametrize("n", list(range(2, 12)))
def test_kernel1_universes(wpm, oracle, golden, n):
    """binary_matroid (charmap.hpp:117-141) on the GPU == the restatement, every map."""
    rows = golden["orbits"][str(n)]
    with wpm.Plan.orbits(n) as p:
        assert p.num_maps == len(rows)
        for i, r in enumerate(rows):
            assert p.universe(i) == oracle.matroid_universe(r), (n, i)


@pytest.mark.parametrize("n", list(range(2, 12)))
def test_kernel2_incidence(wpm, oracle, golden, n):
    """incidence_matrix (incidence.hpp:34-55): ridges, cols and parents, every map."""
    rows = golden["orbits"][str(n)]
    with wpm.Plan.orbits(n) as p:
        for i in range(len(rows)):
            uni = p.universe(i)
            assert p.incidence(i) == oracle.incidence(uni), (n, i)


@pytest.mark.parametrize("n", list(range(2, 12)))
def test_orbit_counts_and_nodes(wpm, golden, n):
    """Per-map WPM counts == the reference (n <= 7: oracle/_ref; n = 8: the
    maps the reference finished) and == the CPU restatement (every n); DFS
    nodes == the CPU restatement, map by map."""
    with wpm.Plan.orbits(n) as p:
        p.run()
        res = p.fetch()
    assert res.duplicates == 0
    dfs = golden["dfs"][str(n)]
    assert res.counts == [m["wpms"] for m in dfs["maps"]]
    if str(n) in golden["ubt"]:
        ref = [m["wpms"] for m in golden["ubt"][str(n)]["maps"]]
        assert res.counts[: len(ref)] == ref
    assert res.nodes == dfs["nodes"]
    # per-map node counts: one map at a time through the same plan path
    if n in (5, 9):
        with wpm.Plan.orbits(n) as p:
            for i in range(p.num_maps):
                u = p.universe(i)
                r = wpm.enumerate_wpm_bits(wpm.SearchJob(n + 4, n, u, properties=[wpm.ubt_property(n, len(u))]))
                assert r.nodes == dfs["maps"][i]["nodes"]


@pytest.mark.parametrize("n", list(range(2, 12)))
def test_orbit_digests(wpm, golden, n):
    """Byte-exact .cplx per map and per n (SURVEY App. C protocol): against
    the reference for n <= 7 (and the n = 8 maps it finished), against the
    CPU restatement's bytes for n = 8..11."""
    with wpm.Plan.orbits(n) as p:
        p.run()
        res = p.fetch()
        whole, per = _digest_plan(wpm, p, res, n)
    if n <= 7:
        assert per == golden["ubt"][str(n)]["map_sha256"]
        assert whole == golden["ubt"][str(n)]["sha256"]
    else:
        assert per == [m["sha256"] for m in golden["dfs"][str(n)]["maps"]]
        assert whole == golden["dfs"][str(n)]["sha256"]
        if str(n) in golden["ubt"]:
            ref = golden["ubt"][str(n)]["map_sha256"]
            assert per[: len(ref)] == ref


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_nocap_counts(wpm, golden, n):
    """No property: every WPM (classify_full_universe semantics)."""
    with wpm.Plan.orbits(n, facet_cap=wpm.WPM_CAP_NONE) as p:
        p.run()
        res = p.fetch()
        whole, _ = _digest_plan(wpm, p, res, n)
    assert res.counts == golden["nocap"][str(n)]["counts"]
    assert whole == golden["nocap"][str(n)]["sha256"]


def test_small_examples(wpm, oracle):
    """test_search.cpp:104-121 and :269-274."""
    u = oracle.all_subsets_universe(4, 2)
    out = wpm.enumerate_wpm(wpm.SearchJob(4, 2, u))
    assert len(out) == 7
    assert sorted(len(k) for k in out) == [3, 3, 3, 3, 4, 4, 4]
    s3 = oracle.all_subsets_universe(4, 3)
    out = wpm.enumerate_wpm(wpm.SearchJob(4, 3, s3))
    assert out == [s3]
    # two disjoint edges: empty output is valid
    assert wpm.enumerate_wpm(wpm.SearchJob(4, 2, [0b00110, 0b11000])) == []


def _random_universes(seed, count, mlo, mhi, nlo, nhi, Mlo, Mhi, oracle, keep=3):
    rng = random.Random(seed)
    out = []
    while len(out) < count:
        m = rng.randint(mlo, mhi)
        n = rng.randint(nlo, nhi)
        if n >= m:
            continue
        u = [f for f in oracle.all_subsets_universe(m, n) if rng.randrange(keep) == 0]
        if Mlo <= len(u) <= Mhi:
            out.append((m, n, u))
    return out


def test_full_subset_universes_vs_oracles(wpm, oracle):
    """acceptance.cpp:259-262 shapes: all n-subsets of [m] vs brute force and
    the restated reference, bit-exact lists."""
    for m, n in [(4, 2), (5, 2), (6, 2), (7, 2), (4, 3), (5, 3), (6, 3), (6, 4), (5, 4), (6, 5), (7, 5), (7, 6)]:
        u = oracle.all_subsets_universe(m, n)
        res = wpm.enumerate_wpm_bits(wpm.SearchJob(m, n, u))
        assert res.duplicates == 0
        if len(u) <= 24:
            assert res.total == oracle.brute_force_count(u), (m, n)
        rc, ref = oracle.enumerate_ref(m, n, u)
        assert rc == 0
        assert np.array_equal(res.map_bits(0), ref["bits"]), (m, n)
        cnt, nodes, _ = oracle.dfs(n, u, -1, want_bits=False)
        assert res.nodes == nodes


def test_random_universes_vs_bruteforce(wpm, oracle):
    """acceptance.cpp:264-279: random universes, M in [8, 24]."""
    for m, n, u in _random_universes(20240809, 12, 6, 8, 2, 4, 8, 24, oracle):
        for cap in (-1, 4, 7):
            job = wpm.SearchJob(m, n, u, properties=[wpm.AffineProperty([-1] * len(u), cap + 1)] if cap >= 0 else [])
            res = wpm.enumerate_wpm_bits(job)
            assert res.total == oracle.brute_force_count(u, cap=cap), (m, n, cap)
            cnt, nodes, bits = oracle.dfs(n, u, cap)
            assert np.array_equal(res.map_bits(0), bits)
            assert res.nodes == nodes


def test_constrained_vs_bruteforce(wpm, oracle):
    """acceptance.cpp:281-315: required/forbidden pins vs brute force."""
    rng = random.Random(20240809)
    made = 0
    while made < 10:
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
        if set(req) & set(forb):
            continue
        res = wpm.enumerate_wpm_bits(wpm.SearchJob(6, 3, u, required=req, forbidden=forb))
        assert res.total == oracle.brute_force_count(u, req, forb), (u, req, forb)
        cnt, nodes, bits = oracle.dfs(3, u, -1, req, forb)
        assert np.array_equal(res.map_bits(0), bits)
        assert res.nodes == nodes


def test_octahedron_link_pinning(wpm, oracle):
    """test_search.cpp:178-220: pinned link of vertex 1 == filtered unconstrained."""
    u = oracle.all_subsets_universe(6, 3)
    octa = sorted(sum(1 << (i + 1 + (3 if (c >> i) & 1 else 0)) for i in range(3)) for c in range(8))
    req = [j for j, f in enumerate(u) if f & 2 and f in octa]
    forb = [j for j, f in enumerate(u) if f & 2 and f not in octa]
    pinned = wpm.enumerate_wpm(wpm.SearchJob(6, 3, u, required=req, forbidden=forb))
    full = wpm.enumerate_wpm(wpm.SearchJob(6, 3, u))
    filt = [K for K in full if all(u[j] in K for j in req) and not any(u[j] in K for j in forb)]
    assert pinned == filt and len(pinned) > 0


@pytest.mark.parametrize("n", [5, 6])
def test_shards_partition(wpm, golden, n):
    """Root-task sharding (the multi-GPU split): shards are disjoint, their
    union is the full canonical list, node counts add up."""
    with wpm.Plan.orbits(n) as p:
        p.run()
        full = p.fetch()
        parts = []
        nodes = 0
        for s in range(3):
            p.run(s, 3)
            r = p.fetch()
            parts.append(r)
            nodes += r.nodes
    assert nodes == full.nodes
    for i in range(full.num_maps):
        rows = np.concatenate([r.map_bits(i) for r in parts])
        assert rows.shape[0] == full.counts[i]
        got = {tuple(x) for x in rows.tolist()}
        assert got == {tuple(x) for x in full.map_bits(i).tolist()}


def test_deterministic_repeat(wpm):
    """test_search.cpp:147-157 analogue: identical bytes across runs."""
    with wpm.Plan.orbits(5) as p:
        p.run()
        a = p.fetch()
        p.run()
        b = p.fetch()
    assert np.array_equal(a.bits, b.bits) and a.nodes == b.nodes


def test_soundness_n11(wpm, oracle):
    """every emitted K at n = 11 is a WPM (direct recount,
    complex.hpp:224-233) inside the universe and within the UBT cap."""
    with wpm.Plan.orbits(11) as p:
        p.run()
        res = p.fetch()
        u = p.universe(0)
    cap = oracle.cyclic_facet_bound(11)
    rows = res.map_bits(0)
    step = max(1, rows.shape[0] // 3000)
    for row in rows[::step]:
        fs = [u[j] for j in range(len(u)) if (int(row[j >> 6]) >> (j & 63)) & 1]
        assert 0 < len(fs) <= cap
        assert oracle.is_wpm_direct(fs)


def test_cpp_dropin_on_gpu(wpm, golden, tmp_path):
    """include/plseeds_b200.hpp end to end: enumerate_wpm over the n = 5 map 0
    universe, write_complexes bytes == the reference's digest."""
    import os
    import shutil
    import subprocess

    from conftest import ROOT

    if shutil.which("g++") is None:
        pytest.skip("no g++")
    src = tmp_path / "t.cpp"
    src.write_text(r'''
#include "plseeds_b200.hpp"
#include <iostream>
#include <sstream>
int main() {
    using namespace plseeds_b200;
    auto orbits = idcm_orbits(5, 4);
    SearchJob job;
    job.m = 9; job.n = 5;
    job.facets = matroid_universe(orbits.at(0));
    job.properties = {ubt_property(5, (int)job.facets.size())};
    write_complexes(std::cout, enumerate_wpm(job));
    return 0;
}
''')
    lib = os.path.join(ROOT, "paper_2301_00806_b200", "libwpm_b200.so")
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe), lib,
                    f"-Wl,-rpath,{os.path.dirname(lib)}"], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True).stdout
    assert hashlib.sha256(out).hexdigest() == golden["ubt"]["5"]["map_sha256"][0]


def test_nccl_gather_world1(wpm, golden):
    """The multi-GPU result path (dist.gather_to_rank0_device) on a 1-rank NCCL
    group: resident rows -> all_gather -> device canonical sort."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2301_00806_b200 import dist as wdist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]))
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        with wpm.Plan.orbits(5) as p:
            p.run(0, 1)
            total, dups = wdist.gather_to_rank0_device(dist, p, 0, 0)
        assert total == golden["ubt"]["5"]["sum"] and dups == 0
    finally:
        dist.destroy_process_group()


def test_cpp_adapter_vs_reference():
    """plseeds::b200::enumerate_wpm(const plseeds::SearchJob&) against the
    reference's own enumerate_wpm in one binary (tests/cpp/adapter_check.cpp,
    reference headers compiled in): orbit maps n = 2..5, full-subset
    universes, link-pinned bases (apply_link_constraints), candidate_cap."""
    import os
    import subprocess

    from conftest import ROOT

    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_check")
    if not os.path.exists(exe):
        pytest.skip("adapter_check not built (needs the reference headers at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout


def test_output_overflow_reruns_exactly(wpm, golden, monkeypatch):
    """The row buffer starts at 2^21 rows; a result larger than the buffer
    reruns once with the exact count (forced here with a 1000-row buffer)."""
    monkeypatch.setenv("WPM_OUT_CAP", "1000")
    with wpm.Plan.orbits(4) as p:
        assert p.run() == golden["dfs"]["4"]["sum"]
        res = p.fetch()
    assert res.duplicates == 0 and res.total == golden["dfs"]["4"]["sum"]


@pytest.mark.parametrize("n", [4, 8, 11])
def test_canonical_sort_device_shuffled(wpm, n):
    """wpm_canonical_sort_device (kernel 4 on rows that already live on the
    device, e.g. gathered from several GPUs): a random permutation of a run's
    canonical rows (map ids kept with them) sorts back to the same bytes, with
    no duplicates; with every row twice, exactly `count` duplicates."""
    import torch

    from paper_2301_00806_b200.dist import _wrap_device

    with wpm.Plan.orbits(n) as p:
        total = p.run()
        bits_ptr, map_ptr, count, w32 = p.device_result()
        dev = torch.device("cuda", 0)
        rows = _wrap_device(bits_ptr, count * w32, torch.int32, dev).view(count, w32).clone()
        maps = _wrap_device(map_ptr, count, torch.int16, dev).clone()
    g = torch.Generator(device="cpu").manual_seed(n)
    perm = torch.randperm(count, generator=g).to(dev)
    for k in (1, 2):
        src_r = rows[perm].repeat(k, 1).contiguous()
        src_m = maps[perm].repeat(k).contiguous()
        out_r = torch.empty_like(src_r)
        out_m = torch.empty_like(src_m)
        torch.cuda.synchronize()
        dups = wpm.canonical_sort_device(0, src_r.data_ptr(), src_m.data_ptr(), k * count, w32, out_r.data_ptr(),
                                         out_m.data_ptr())
        assert dups == (k - 1) * count
        if k == 1:
            assert torch.equal(out_r, rows) and torch.equal(out_m, maps) and count == total
        else:
            assert torch.equal(out_r[0::2], rows) and torch.equal(out_r[1::2], rows)


@pytest.mark.parametrize("n", [3, 5, 8, 11])
def test_bucketed_sort_variant(wpm, golden, n, monkeypatch):
    """The bucketed kernel-4 variant (WPM_SORT=bucket, opt-in: measured
    slower) gives the same rows as the merge sort."""
    import numpy as np

    with wpm.Plan.orbits(n) as p:
        p.run()
        want = np.array(p.fetch().bits)
    monkeypatch.setenv("WPM_SORT", "bucket")
    with wpm.Plan.orbits(n) as p:
        for _ in range(2):  # the second run reuses the zeroed count block
            p.run()
            res = p.fetch()
            assert res.duplicates == 0 and res.counts == [m["wpms"] for m in golden["dfs"][str(n)]["maps"]]
            assert np.array_equal(np.array(res.bits), want)
