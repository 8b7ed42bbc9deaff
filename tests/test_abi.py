"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/wpm_b200.h declares, the C++ drop-in header compiles and
links against it, and compute entry points fail loudly without a GPU (no
CPU fallback)."""
import ctypes
import os
import re
import shutil
import subprocess
import tempfile

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "wpm_b200.h")
LIB = os.path.join(ROOT, "paper_2301_00806_b200", "libwpm_b200.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(wpm_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("wpm_enumerate", "wpm_result_free", "wpm_device_count", "wpm_last_error", "wpm_plan_run",
                 "wpm_idcm_orbits", "wpm_write_cplx"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for n in declared_functions():
        assert re.search(rf"\bT {n}$", nm, flags=re.M), n


def test_python_mirror_binds_every_symbol(wpm):
    assert set(wpm.EXPORTED_SYMBOLS) == set(declared_functions())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cpp_dropin_compiles_and_links():
    """include/plseeds_b200.hpp: the reference-named C++ API over the C-ABI."""
    src = r'''
#include "plseeds_b200.hpp"
#include <sstream>
int main() {
    using namespace plseeds_b200;
    auto orbits = idcm_orbits(5, 4);
    SearchJob job;
    job.m = 9; job.n = 5;
    job.facets = matroid_universe(orbits.at(0));
    job.properties = {ubt_property(5, (int)job.facets.size())};
    std::ostringstream os;
    if (std::getenv("WPM_RUN")) write_complexes(os, enumerate_wpm(job));
    return orbits.size() == 35 ? 0 : 1;
}
'''
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "t.cpp")
        open(p, "w").write(src)
        exe = os.path.join(td, "t")
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), p, "-o", exe,
                            LIB, f"-Wl,-rpath,{os.path.dirname(LIB)}"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        # host-only path runs without a GPU (idcm_orbits is host C++); matroid_universe needs the device
        env = dict(os.environ)
        r = subprocess.run([exe], capture_output=True, text=True, env=env)
        if not _has_gpu():
            assert r.returncode != 0 and "no CUDA device" in (r.stderr + r.stdout)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include") or shutil.which("g++") is None,
                    reason="reference headers not present (dev container only)")
def test_cpp_adapter_compiles_with_reference_headers():
    """plseeds::b200::enumerate_wpm(const plseeds::SearchJob&) type-checks
    against the unmodified reference headers."""
    src = r'''
#include "plseeds/pipeline.hpp"
#include "plseeds_b200.hpp"
int main() {
    using namespace plseeds;
    SearchJob job;
    job.m = 6; job.n = 2;
    job.facets = matroid_universe(idcm_orbits(2, 4)[0]);
    const auto A = incidence_matrix(job.facets);
    job.basis = convenient_basis(kernel_basis(A), A);
    job.properties = {ubt_property(2, (int)job.facets.size())};
    auto out = std::getenv("WPM_RUN") ? b200::enumerate_wpm(job) : std::vector<PureComplex>{};
    return (int)out.size() * 0;
}
'''
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.cpp")
        open(p, "w").write(src)
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I/root/reference/proj/include", "-I",
                            os.path.join(ROOT, "include"), p], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def _has_gpu():
    import paper_2301_00806_b200 as w

    return w.device_count() > 0


def test_no_cpu_fallback(wpm, oracle):
    """Without a B200 every compute call raises instead of computing on the CPU."""
    if _has_gpu():
        pytest.skip("GPU present")
    u = oracle.all_subsets_universe(4, 2)
    with pytest.raises(wpm.WpmError, match="no CPU fallback"):
        wpm.enumerate_wpm(wpm.SearchJob(4, 2, u))
    with pytest.raises(wpm.WpmError):
        wpm.enumerate_orbits(2)
    with pytest.raises(wpm.WpmError):
        wpm.Plan.orbits(2)


def test_job_validation_errors(wpm):
    """PureComplex::validate / incidence_matrix error behaviour (complex.hpp:37-55,
    incidence.hpp:35) is checked on the host before any device work."""
    with pytest.raises(wpm.PurityError):
        wpm.enumerate_wpm(wpm.SearchJob(4, 2, []))
    with pytest.raises(ValueError, match="duplicate"):
        wpm.enumerate_wpm(wpm.SearchJob(4, 2, [0b1100, 0b0110, 0b1100]))  # PureComplex::validate, complex.hpp:50-51
    with pytest.raises(ValueError):
        wpm.enumerate_wpm(wpm.SearchJob(4, 2, [0b0110], properties=[wpm.AffineProperty([2], 3)]))


def test_idcm_orbits_host_matches_goldens(wpm, oracle, golden):
    """wpm_idcm_orbits (host C++, table-driven) = the reference's orbit
    representatives (charmap.hpp:212-281), every Picard-4 n, and the oracle
    for Picard 3 and 5."""
    for n in range(2, 12):
        got = [d.rows for d in wpm.idcm_orbits(n, 4)]
        assert got == golden["orbits"][str(n)], n
    for n, p in ((2, 3), (3, 3), (4, 3), (2, 5), (3, 5)):  # the oracle returns <= 64 orbits
        assert [d.rows for d in wpm.idcm_orbits(n, p)] == oracle.idcm_orbits(n, p), (n, p)


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_cpp_host_pool_visits_every_item_once():
    """detail::HostPool (the drop-in's PureComplex builder): every index of
    every parallel region exactly once, regions back to back, small and empty
    regions -- host C++ only, no device."""
    src = r'''
#include "plseeds_b200.hpp"
#include <atomic>
#include <cstdio>
#include <vector>
int main() {
    auto& pool = plseeds_b200::detail::HostPool::get();
    for (std::size_t items : {0, 1, 2, 7, 1000, 100000}) {
        for (int rep = 0; rep < 3; ++rep) {
            std::vector<std::atomic<int>> hit(items);
            for (auto& h : hit) h.store(0);
            pool.run(items, [&](std::size_t i) { hit[i].fetch_add(1); });
            for (std::size_t i = 0; i < items; ++i)
                if (hit[i].load() != 1) { std::printf("item %zu of %zu hit %d\n", i, items, hit[i].load()); return 1; }
        }
    }
    std::printf("ok\n");
    return 0;
}
'''
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "t.cpp")
        open(p, "w").write(src)
        exe = os.path.join(td, "t")
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-pthread", "-Wall", "-I", os.path.join(ROOT, "include"), p,
                            "-o", exe, LIB, f"-Wl,-rpath,{os.path.dirname(LIB)}"], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
