// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin driver around the UNMODIFIED reference library, compiled by
// oracle/Makefile straight from the headers where they lie
// (/root/reference/proj/include); the binary goes to oracle/_ref/ (git-ignored,
// shipped to the GPU box by gpurun).  It is the golden generator and the
// `--impl reference` CPU baseline.  It runs the reference path exactly as
// pipeline.hpp:58-72 does per orbit: matroid_universe -> incidence_matrix ->
// convenient_basis(kernel_basis) -> ubt_property -> enumerate_wpm.
//
// usage:
//   plseeds_ref orbits N
//   plseeds_ref enumerate N [--nocap] [--threads T] [--out FILE] [--maps a:b]
//        per map prints "map i M N s space wpms seconds"; --out writes the
//        concatenated .cplx bytes (SURVEY App. C protocol) and per-map offsets
//   plseeds_ref universe N --out FILE
//   plseeds_ref job FILE [--threads T] [--out FILE]
//        FILE: "m n M cap nreq nforb" then M facet masks, then req, forb
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "plseeds/catalog.hpp"
#include "plseeds/classify.hpp"
#include "plseeds/charmap.hpp"
#include "plseeds/complex_io.hpp"
#include "plseeds/incidence.hpp"
#include "plseeds/isomorphism.hpp"
#include "plseeds/kernel_basis.hpp"
#include "plseeds/pipeline.hpp"
#include "plseeds/search.hpp"

using namespace plseeds;
using Clock = std::chrono::steady_clock;

static double since(Clock::time_point t) {
    return std::chrono::duration<double>(Clock::now() - t).count();
}

static int arg_int(int argc, char** argv, const char* key, int def) {
    for (int i = 0; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], key)) return std::atoi(argv[i + 1]);
    return def;
}
static const char* arg_str(int argc, char** argv, const char* key) {
    for (int i = 0; i + 1 < argc; ++i)
        if (!std::strcmp(argv[i], key)) return argv[i + 1];
    return nullptr;
}
static bool has_flag(int argc, char** argv, const char* key) {
    for (int i = 0; i < argc; ++i)
        if (!std::strcmp(argv[i], key)) return true;
    return false;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: plseeds_ref orbits|enumerate|universe|job ...\n");
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "orbits") {
            const int n = std::atoi(argv[2]);
            for (const auto& d : idcm_orbits(n, 4)) {
                for (std::size_t i = 0; i < d.rows.size(); ++i)
                    std::printf("%s%u", i ? " " : "", d.rows[i]);
                std::printf("\n");
            }
            return 0;
        }
        if (cmd == "universe") {
            const int n = std::atoi(argv[2]);
            const char* out = arg_str(argc, argv, "--out");
            std::ofstream os(out ? out : "/dev/null", std::ios::binary);
            for (const auto& d : idcm_orbits(n, 4))
                write_complex(os, PureComplex(n + 4, n, matroid_universe(d), true));
            return 0;
        }
        if (cmd == "enumerate") {
            const int n = std::atoi(argv[2]);
            const bool nocap = has_flag(argc, argv, "--nocap");
            const int threads = arg_int(argc, argv, "--threads", 1);
            const char* out = arg_str(argc, argv, "--out");
            const auto orbits = idcm_orbits(n, 4);
            int a = 0, b = static_cast<int>(orbits.size());
            if (const char* r = arg_str(argc, argv, "--maps")) std::sscanf(r, "%d:%d", &a, &b);
            std::ofstream os;
            if (out) os.open(out, std::ios::binary);
            double total_enum = 0, total_prep = 0;
            long long total_wpm = 0;
            unsigned long long total_space = 0;
            for (int i = a; i < b && i < static_cast<int>(orbits.size()); ++i) {
                const auto t0 = Clock::now();
                SearchJob job;
                job.m = n + 4;
                job.n = n;
                job.facets = matroid_universe(orbits[static_cast<std::size_t>(i)]);
                const IncidenceMatrix A = incidence_matrix(job.facets);
                job.basis = convenient_basis(kernel_basis(A), A);
                if (!nocap) job.properties = {ubt_property(n, static_cast<int>(job.facets.size()))};
                job.threads = threads;
                job.candidate_cap = ~0ull;
                const double prep = since(t0);
                const auto t1 = Clock::now();
                const auto found = enumerate_wpm(job);
                const double dt = since(t1);
                const unsigned long long space = combination_space(job.basis).size_saturated();
                std::printf("map %d M %d N %d s %d space %llu wpms %zu prep %.6f seconds %.6f\n", i, A.M, A.N,
                            job.basis.s(), space, found.size(), prep, dt);
                std::fflush(stdout);
                total_enum += dt;
                total_prep += prep;
                total_wpm += static_cast<long long>(found.size());
                total_space += space;
                if (out) {
                    std::ostringstream ss;
                    write_complexes(ss, found);
                    const std::string s = ss.str();
                    os.write(s.data(), static_cast<std::streamsize>(s.size()));
                }
            }
            std::printf("total wpms %lld space %llu prep %.6f seconds %.6f threads %d\n", total_wpm, total_space,
                        total_prep, total_enum, threads);
            return 0;
        }
        if (cmd == "job") {
            std::ifstream in(argv[2]);
            int m, n, M, nreq, nforb;
            long long cap;
            in >> m >> n >> M >> cap >> nreq >> nforb;
            std::vector<VertexSet> u(static_cast<std::size_t>(M));
            for (auto& f : u) {
                unsigned long long x;
                in >> x;
                f = VertexSet(x);
            }
            std::vector<int> req(static_cast<std::size_t>(nreq)), forb(static_cast<std::size_t>(nforb));
            for (auto& x : req) in >> x;
            for (auto& x : forb) in >> x;
            SearchJob job;
            job.m = m;
            job.n = n;
            job.facets = u;
            const IncidenceMatrix A = incidence_matrix(u);
            auto kb = convenient_basis(kernel_basis(A), A);
            auto pinned = apply_link_constraints(kb, req, forb);
            if (!pinned) {
                std::printf("infeasible\n");
                return 3;
            }
            job.basis = *pinned;
            if (cap >= 0) {
                AffineProperty g;
                g.weights.assign(static_cast<std::size_t>(M), -1);
                g.constant = cap + 1;
                job.properties = {g};
            }
            job.threads = arg_int(argc, argv, "--threads", 1);
            job.candidate_cap = ~0ull;
            const auto t1 = Clock::now();
            const auto found = enumerate_wpm(job);
            std::printf("wpms %zu seconds %.6f\n", found.size(), since(t1));
            if (const char* out = arg_str(argc, argv, "--out")) {
                std::ofstream os(out, std::ios::binary);
                write_complexes(os, found);
            }
            return 0;
        }
        if (cmd == "seed") {
            // per complex of a .cplx file: "<full support> <is_seed>" (classify.hpp:51)
            std::ifstream in(argv[2]);
            for (const PureComplex& K : read_complexes(in, /*embedded=*/true))
                std::printf("%d %d\n", K.support() == VertexSet::full(K.m) ? 1 : 0, is_seed(K) ? 1 : 0);
            return 0;
        }
        if (cmd == "line13") {
            // Algorithm 2 lines 1-13 as pipeline.hpp:58-89 runs them (union of
            // the per-orbit lists, then the Picard and seedness filters);
            // --out writes the line-13 survivors in order as .cplx
            const int n = std::atoi(argv[2]);
            const int threads = arg_int(argc, argv, "--threads", 1);
            const int m = n + 4;
            const auto t0 = Clock::now();
            std::set<std::vector<VertexSet>> labeled;
            for (const auto& d : idcm_orbits(n, 4)) {
                SearchJob job;
                job.m = m;
                job.n = n;
                job.facets = matroid_universe(d);
                const IncidenceMatrix A = incidence_matrix(job.facets);
                job.basis = convenient_basis(kernel_basis(A), A);
                job.properties = {ubt_property(n, static_cast<int>(job.facets.size()))};
                job.threads = threads;
                job.candidate_cap = ~0ull;
                for (const PureComplex& K : enumerate_wpm(job)) labeled.insert(K.facets);
            }
            const double t_enum = since(t0);
            const auto t1 = Clock::now();
            std::vector<std::vector<VertexSet>> all(labeled.begin(), labeled.end());
            std::vector<char> keep(all.size(), 0);
            parallel_for_index(static_cast<long long>(all.size()), threads, [&](long long i) {
                PureComplex K(m, n, all[static_cast<std::size_t>(i)], true);
                if (K.support() != VertexSet::full(m)) return;
                if (!is_seed(K)) return;
                keep[static_cast<std::size_t>(i)] = 1;
            });
            std::vector<PureComplex> survivors;
            for (std::size_t i = 0; i < all.size(); ++i)
                if (keep[i]) survivors.emplace_back(m, n, all[i]);
            std::printf("line7 %zu line13 %zu enum_seconds %.6f filter_seconds %.6f threads %d\n", all.size(),
                        survivors.size(), t_enum, since(t1), threads);
            if (const char* out = arg_str(argc, argv, "--out")) {
                std::ofstream os(out, std::ios::binary);
                write_complexes(os, survivors);
            }
            return 0;
        }
        if (cmd == "line15") {
            // Algorithm 2 line 15 as pipeline.hpp:91-103 runs it on a .cplx of
            // line-13 survivors: canonical_form per complex (isomorphism.hpp:228-303)
            // and the first-appearance representatives.  --canon writes every
            // canonical form in input order, --out the representatives in order.
            const int threads = arg_int(argc, argv, "--threads", 1);
            std::ifstream in(argv[2]);
            std::vector<PureComplex> survivors = read_complexes(in, /*embedded=*/true);
            const auto t0 = Clock::now();
            std::vector<PureComplex> canon(survivors.size());
            parallel_for_index(static_cast<long long>(survivors.size()), threads, [&](long long i) {
                canon[static_cast<std::size_t>(i)] = canonical_form(survivors[static_cast<std::size_t>(i)]);
            });
            std::vector<PureComplex> reps;
            std::set<std::vector<VertexSet>> seen;
            for (auto& c : canon)
                if (seen.insert(c.facets).second) reps.push_back(c);
            std::printf("line13 %zu line15 %zu canon_seconds %.6f threads %d\n", survivors.size(), reps.size(),
                        since(t0), threads);
            if (const char* out = arg_str(argc, argv, "--canon")) {
                std::ofstream os(out, std::ios::binary);
                write_complexes(os, canon);
            }
            if (const char* out = arg_str(argc, argv, "--out")) {
                std::ofstream os(out, std::ios::binary);
                write_complexes(os, reps);
            }
            return 0;
        }
        if (cmd == "classes") {
            // per complex: refine_classes (isomorphism.hpp:162-218) "v:class ..." for vertices 1..m
            std::ifstream in(argv[2]);
            for (const PureComplex& K : read_complexes(in, /*embedded=*/true)) {
                const auto cls = detail::refine_classes(K, minimal_nonfaces(K));
                for (int v = 1; v <= K.m; ++v) std::printf("%d%c", cls[static_cast<std::size_t>(v)], v == K.m ? '\n' : ' ');
            }
            return 0;
        }
    } catch (const cap_exceeded_error& e) {
        std::fprintf(stderr, "cap exceeded: %s\n", e.what());
        return 5;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 2;
}
