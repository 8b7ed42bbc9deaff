// tests/cpp/adapter_check.cpp -- TEST INFRASTRUCTURE.
//
// Runs the UNMODIFIED reference enumerate_wpm (compiled in from
// /root/reference/proj/include at build time) and the drop-in
// plseeds::b200::enumerate_wpm (include/plseeds_b200.hpp -> libwpm_b200.so)
// on the same reference SearchJob and compares the outputs complex by
// complex: every orbit map for n = 2..5 (UBT cap), full-subset universes, the
// test_search.cpp:178-220 link-pinned octahedron basis, random pinned bases
// from apply_link_constraints, universes in shuffled order, hand-made bases
// (a block whose WPMs need three generators, the raw kernel basis, a block
// list with a gap), SearchJob::progress, and the candidate_cap error.  Built by
// oracle/Makefile (target `ref`) into oracle/_ref/; run by tests/test_gpu_parity.py.
#include <algorithm>
#include <cstdio>
#include <random>
#include <set>

#include "plseeds/catalog.hpp"
#include "plseeds/classify.hpp"
#include "plseeds/pipeline.hpp"
#include "plseeds/search.hpp"
#include "plseeds/isomorphism.hpp"
#include "plseeds_b200.hpp"

using namespace plseeds;

static int failures = 0;

static void check(const SearchJob& job, const char* what) {
    const auto ref = enumerate_wpm(job);
    const auto got = b200::enumerate_wpm(job);
    if (!(ref == got)) {
        std::printf("MISMATCH %s: reference %zu, b200 %zu\n", what, ref.size(), got.size());
        ++failures;
    }
}

static SearchJob make_job(const std::vector<VertexSet>& u, int m, int n) {
    SearchJob job;
    job.m = m;
    job.n = n;
    job.facets = u;
    const auto A = incidence_matrix(u);
    job.basis = convenient_basis(kernel_basis(A), A);
    job.candidate_cap = ~0ull;
    return job;
}

int main() {
    int jobs = 0;
    for (int n = 2; n <= 5; ++n)
        for (const auto& d : idcm_orbits(n, 4)) {
            auto job = make_job(matroid_universe(d), n + 4, n);
            job.properties = {ubt_property(n, static_cast<int>(job.facets.size()))};
            check(job, "orbit map");
            ++jobs;
        }
    for (auto [m, n] : {std::pair{5, 2}, {6, 2}, {6, 3}, {7, 3}, {6, 4}})
        check(make_job(all_subsets_universe(m, n), m, n), "full subsets"), ++jobs;
    {  // octahedron link pinning, test_search.cpp:178-220
        const auto u = all_subsets_universe(6, 3);
        auto job = make_job(u, 6, 3);
        const auto oct = octahedron();
        std::vector<int> req, forb;
        for (std::size_t j = 0; j < u.size(); ++j) {
            if (!u[j].contains(1)) continue;
            (std::binary_search(oct.facets.begin(), oct.facets.end(), u[j]) ? req : forb).push_back((int)j);
        }
        job.basis = *apply_link_constraints(job.basis, req, forb);
        check(job, "octahedron pin");
        ++jobs;
    }
    std::mt19937 rng(20240809);
    int made = 0;
    while (made < 20) {
        std::vector<VertexSet> u;
        for (VertexSet f : all_subsets_universe(6, 3))
            if (rng() % 2 == 0) u.push_back(f);
        if (u.size() < 10 || u.size() > 18) continue;
        std::vector<int> req, forb;
        for (std::size_t j = 0; j < u.size(); ++j) {
            const auto roll = rng() % 10;
            if (roll == 0) req.push_back((int)j);
            else if (roll == 1) forb.push_back((int)j);
        }
        auto job = make_job(u, 6, 3);
        const auto pinned = apply_link_constraints(job.basis, req, forb);
        ++made;
        if (!pinned) continue;
        job.basis = *pinned;
        check(job, "random pin");
        ++jobs;
    }
    {  // a universe in any order (incidence_matrix indexes by hash, incidence.hpp:34-55)
        std::mt19937 sh(11);
        for (int n = 3; n <= 5; ++n) {
            auto u = matroid_universe(idcm_orbits(n, 4)[1]);
            std::shuffle(u.begin(), u.end(), sh);
            auto job = make_job(u, n + 4, n);
            job.properties = {ubt_property(n, static_cast<int>(u.size()))};
            check(job, "unsorted universe");
            ++jobs;
        }
    }
    {  // hand-made bases: the adapter must return exactly what the reference reaches
        auto u = matroid_universe(idcm_orbits(5, 4)[2]);
        auto job = make_job(u, 9, 5);
        job.properties = {ubt_property(5, static_cast<int>(u.size()))};
        int b3 = -1;
        for (std::size_t b = 0; b < job.basis.blocks.size() && b3 < 0; ++b)
            if (job.basis.blocks[b].width >= 3) b3 = static_cast<int>(b);
        if (b3 >= 0) {  // g2 += g0 + g1 inside one block: a WPM g2 now needs 3 block generators
            const int off = job.basis.blocks[static_cast<std::size_t>(b3)].offset;
            job.basis.gens[static_cast<std::size_t>(off + 2)] ^= job.basis.gens[static_cast<std::size_t>(off)];
            job.basis.gens[static_cast<std::size_t>(off + 2)] ^= job.basis.gens[static_cast<std::size_t>(off + 1)];
            check(job, "block-mixed basis");
            ++jobs;
        } else {
            std::printf("MISMATCH no block of width >= 3 for the mixed-basis case\n");
            ++failures;
        }
        auto raw = job;  // the raw kernel basis: every generator a free singleton, the full span
        raw.basis = KernelBasis{};
        raw.basis.M = static_cast<int>(u.size());
        raw.basis.gens = kernel_basis(incidence_matrix(u));
        check(raw, "raw kernel basis");
        ++jobs;
        auto sub = job;  // a truncated block list: the skipped generators are never used
        if (sub.basis.blocks.size() > 1) {
            sub.basis.blocks.erase(sub.basis.blocks.begin());
            check(sub, "block list without its first block");
            ++jobs;
        }
    }
    {  // SearchJob::progress (search.hpp:54): called, monotone, ends at done == total
        auto u = matroid_universe(idcm_orbits(6, 4)[0]);
        auto job = make_job(u, 10, 6);
        job.properties = {ubt_property(6, static_cast<int>(u.size()))};
        std::vector<std::pair<long long, long long>> calls;
        job.progress = [&](long long d, long long t) { calls.emplace_back(d, t); };
        const auto got = b200::enumerate_wpm(job);
        bool ok = !calls.empty() && calls.back().first == calls.back().second && !got.empty();
        for (std::size_t i = 1; i < calls.size(); ++i) ok &= calls[i - 1].first <= calls[i].first;
        if (!ok) {
            std::printf("MISMATCH progress: %zu calls\n", calls.size());
            ++failures;
        }
        ++jobs;
    }
    {  // candidate_cap: same exception type
        auto job = make_job(all_subsets_universe(6, 2), 6, 2);
        job.candidate_cap = 16;
        bool threw = false;
        try {
            b200::enumerate_wpm(job);
        } catch (const cap_exceeded_error&) {
            threw = true;
        }
        if (!threw) {
            std::printf("MISMATCH cap_exceeded_error not thrown\n");
            ++failures;
        }
    }
    // Algorithm 2 lines 7 and 13 (pipeline.hpp:58-89) vs the reference's own
    // union + support + is_seed, n = 2..4
    for (int n = 2; n <= 4; ++n) {
        const int m = n + 4;
        std::set<std::vector<VertexSet>> labeled;
        for (const auto& d : idcm_orbits(n, 4)) {
            auto job = make_job(matroid_universe(d), m, n);
            job.properties = {ubt_property(n, static_cast<int>(job.facets.size()))};
            for (const auto& K : enumerate_wpm(job)) labeled.insert(K.facets);
        }
        std::vector<PureComplex> survivors;
        for (const auto& fs : labeled) {
            PureComplex K(m, n, fs, true);
            if (K.support() == VertexSet::full(m) && is_seed(K)) survivors.emplace_back(m, n, fs);
        }
        const auto got = b200::pipeline_line13(n);
        if (got.line7 != (long long)labeled.size() || got.line13 != (long long)survivors.size() ||
            !(got.survivors == survivors)) {
            std::printf("MISMATCH line13 n=%d: reference %zu/%zu, b200 %lld/%lld\n", n, labeled.size(),
                        survivors.size(), got.line7, got.line13);
            ++failures;
        }
        ++jobs;
    }
    {  // batch is_seed on catalog complexes (test_classify.cpp:24-31)
        const std::vector<PureComplex> cat = {s0(), simplex_boundary(2), square(), wedge(square(), 1), hexagon(),
                                              octahedron(), pentagon(), suspension(pentagon())};
        const auto got = b200::is_seed(cat);
        for (std::size_t i = 0; i < cat.size(); ++i)
            if ((got[i] != 0) != is_seed(cat[i])) {
                std::printf("MISMATCH is_seed catalog %zu\n", i);
                ++failures;
            }
        ++jobs;
    }
    // Algorithm 2 line 15 (pipeline.hpp:91-103): the reference's canonical
    // forms and first-appearance representatives, n = 2..4
    for (int n = 2; n <= 4; ++n) {
        const auto l13 = b200::pipeline_line13(n);
        std::vector<PureComplex> reps;
        std::set<std::vector<VertexSet>> seen;
        for (const auto& K : l13.survivors) {
            auto c = canonical_form(K);
            if (seen.insert(c.facets).second) reps.push_back(std::move(c));
        }
        const auto got = b200::pipeline_line15(n);
        if (got.line15 != (long long)reps.size() || !(got.reps == reps)) {
            std::printf("MISMATCH line15 n=%d: reference %zu, b200 %lld\n", n, reps.size(), got.line15);
            ++failures;
        }
        const auto canon = b200::canonical_form(l13.survivors);
        for (std::size_t i = 0; i < canon.size(); ++i)
            if (!(canon[i] == canonical_form(l13.survivors[i]))) {
                std::printf("MISMATCH canonical_form n=%d survivor %zu\n", n, i);
                ++failures;
                break;
            }
        ++jobs;
    }
    {  // canonical_form on catalog complexes with large automorphism groups
        const std::vector<PureComplex> cat = {s0(), square(), hexagon(), octahedron(), pentagon(),
                                              suspension(pentagon()), suspension(octahedron()), wedge(square(), 1)};
        const auto got = b200::canonical_form(cat);
        for (std::size_t i = 0; i < cat.size(); ++i)
            if (!(got[i] == canonical_form(cat[i]))) {
                std::printf("MISMATCH canonical_form catalog %zu\n", i);
                ++failures;
            }
        ++jobs;
    }
    std::printf("adapter_check: %d jobs, %d mismatches\n", jobs, failures);
    return failures ? 1 : 0;
}
