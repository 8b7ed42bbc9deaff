// plseeds_b200.hpp -- header-only C++ drop-in for the reference's enumeration
// path, over the C-ABI of libwpm_b200.so (include/wpm_b200.h).
//
// Two ways to use it:
//
// 1. Standalone, namespace plseeds_b200: the same names, argument meaning and
//    error types as the reference (/root/reference/proj/include/plseeds):
//      VertexSet            vertex_set.hpp:20-68
//      PureComplex          complex.hpp:23-104
//      DualCharMatrix       charmap.hpp:64-87      CharMatrixZ2  charmap.hpp:20-26
//      idcm_orbits          charmap.hpp:212-281    charmap_of_dcm charmap.hpp:155-204
//      binary_matroid       charmap.hpp:117-141 (kernel 1 on the GPU)
//      matroid_universe     pipeline.hpp:33-35
//      AffineProperty, ubt_property, cyclic_facet_bound   affine_property.hpp:16-54
//      SearchJob            search.hpp:46-55 (+ required/forbidden pins, device)
//      enumerate_wpm        search.hpp:141-258 (kernels 2-3 + canonical sort)
//      enumerate_orbits     the per-orbit loop of pipeline.hpp:58-72, one launch
//      write_complex(es)    complex_io.hpp:21-39
//      pipeline_line13      pipeline.hpp:52-89 lines 1-13 (union, support, is_seed on the GPU)
//      is_seed              classify.hpp:51-53 (batch, on the GPU)
//      canonical_form       isomorphism.hpp:228-303 (batch, on the GPU)
//      pipeline_line15      pipeline.hpp:52-103 lines 1-15 (+ canonical forms, class dedupe)
//      purity_error, cap_exceeded_error, format_error   errors.hpp:10-32
//
// 2. Inside a program that already includes the reference headers
//    (plseeds/search.hpp first): plseeds::b200::enumerate_wpm(const
//    plseeds::SearchJob&) takes the reference's own job type -- universe,
//    properties, the (possibly link-pinned) KernelBasis and candidate_cap --
//    and returns the reference's std::vector<plseeds::PureComplex>, identical
//    to plseeds::enumerate_wpm(job).
#ifndef PLSEEDS_B200_HPP
#define PLSEEDS_B200_HPP

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <atomic>
#include <condition_variable>
#include <initializer_list>
#include <mutex>
#include <ostream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "wpm_b200.h"

namespace plseeds_b200 {

struct purity_error : std::runtime_error {
    explicit purity_error(const std::string& w) : std::runtime_error(w) {}
};
struct format_error : std::runtime_error {
    explicit format_error(const std::string& w) : std::runtime_error(w) {}
};
struct cap_exceeded_error : std::runtime_error {
    explicit cap_exceeded_error(const std::string& w) : std::runtime_error(w) {}
};
// status 1: CUDA / no device (there is no CPU fallback)
struct device_error : std::runtime_error {
    explicit device_error(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
    if (rc == WPM_OK) return;
    const std::string msg = wpm_last_error();
    if (rc == WPM_ECAP) throw cap_exceeded_error(msg);
    if (rc == WPM_EINVAL) {
        if (msg.find("purity") != std::string::npos || msg.find("empty facet set") != std::string::npos)
            throw purity_error(msg);
        throw std::invalid_argument(msg);
    }
    if (rc == WPM_EINFEASIBLE) throw std::invalid_argument(msg);
    throw device_error(msg);
}

struct VertexSet {
    std::uint64_t bits = 0;
    constexpr VertexSet() = default;
    constexpr explicit VertexSet(std::uint64_t raw) : bits(raw) {}
    VertexSet(std::initializer_list<int> labels) {
        for (int v : labels) bits |= std::uint64_t{1} << v;
    }
    constexpr bool contains(int v) const { return (bits >> v) & 1u; }
    int count() const { return __builtin_popcountll(bits); }
    bool operator==(const VertexSet& o) const { return bits == o.bits; }
    bool operator!=(const VertexSet& o) const { return bits != o.bits; }
    bool operator<(const VertexSet& o) const { return bits < o.bits; }  // canonical order
};

struct PureComplex {
    int m = 0;
    int n = 0;
    std::vector<VertexSet> facets;  // canonical (ascending) order
    bool embedded = false;
    bool operator==(const PureComplex& o) const { return m == o.m && n == o.n && facets == o.facets; }
    int facet_count() const { return static_cast<int>(facets.size()); }
};

struct DualCharMatrix {
    int m = 0;
    int p = 0;
    std::vector<std::uint32_t> rows;
};

struct CharMatrixZ2 {
    int n = 0;
    int m = 0;
    std::vector<std::uint32_t> cols;
};

struct AffineProperty {
    std::vector<std::int64_t> weights;
    std::int64_t constant = 0;
    bool is_count_cap() const {
        for (auto w : weights)
            if (w != -1) return false;
        return true;
    }
};

inline std::int64_t cyclic_facet_bound(int n) { return wpm_cyclic_facet_bound(n); }

inline AffineProperty ubt_property(int n, int universe_size) {
    AffineProperty g;
    g.weights.assign(static_cast<std::size_t>(universe_size), -1);
    g.constant = cyclic_facet_bound(n) + 1;
    return g;
}

struct SearchJob {
    int m = 0;
    int n = 0;
    std::vector<VertexSet> facets;  // the universe, canonical order
    std::vector<AffineProperty> properties;
    std::vector<int> required;      // link pins (apply_link_constraints semantics)
    std::vector<int> forbidden;
    int threads = 1;                // accepted; the device search has its own parallelism
    std::uint64_t candidate_cap = std::uint64_t{1} << 48;  // no combination space on the device
    std::function<void(long long, long long)> progress;
    int device = 0;
    std::vector<std::int32_t> devices;  // several GPUs for one job (threads -> GPUs); empty = `device`
};

inline std::vector<DualCharMatrix> idcm_orbits(int n, int p) {
    const int m = n + p;
    std::vector<std::uint32_t> rows(static_cast<std::size_t>(4096) * m);
    const int k = wpm_idcm_orbits(n, p, rows.data(), 4096);
    if (k < 0) check(-k);
    std::vector<DualCharMatrix> out(static_cast<std::size_t>(k));
    for (int i = 0; i < k; ++i) {
        out[i].m = m;
        out[i].p = p;
        out[i].rows.assign(rows.begin() + static_cast<long>(i) * m, rows.begin() + static_cast<long>(i + 1) * m);
    }
    return out;
}

inline CharMatrixZ2 charmap_of_dcm(const DualCharMatrix& d) {
    CharMatrixZ2 lam;
    lam.m = d.m;
    lam.cols.assign(static_cast<std::size_t>(d.m), 0);
    const int n = wpm_charmap_of_dcm(d.m, d.p, d.rows.data(), lam.cols.data());
    if (n < 0) check(-n);
    lam.n = n;
    return lam;
}

namespace detail {
struct Plan {
    wpm_plan_t* p = nullptr;
    ~Plan() { wpm_plan_destroy(p); }
};
struct Result {
    wpm_result_t* r = nullptr;
    ~Result() { wpm_result_free(r); }
};

inline std::vector<VertexSet> universe_of(wpm_plan_t* p, int map) {
    std::vector<std::uint64_t> f(WPM_MAX_FACETS);
    const int M = wpm_plan_universe(p, map, f.data(), WPM_MAX_FACETS);
    if (M < 0) check(-M);
    std::vector<VertexSet> out;
    out.reserve(static_cast<std::size_t>(M));
    for (int j = 0; j < M; ++j) out.emplace_back(f[static_cast<std::size_t>(j)]);
    return out;
}

// A persistent host worker pool for building the reference's return objects
// (one std::vector<VertexSet> per WPM: 242,043 heap vectors at n = 5).
// Spawning threads per call cost ~20 us each; these wait on a condition
// variable between calls.  run(items, fn) calls fn(i) for every i < items,
// dynamically scheduled over the workers and the calling thread.
class HostPool {
public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    void run(std::size_t items, const std::function<void(std::size_t)>& fn) {
        if (items == 0) return;
        if (workers_.empty() || items == 1) {
            for (std::size_t i = 0; i < items; ++i) fn(i);
            return;
        }
        std::lock_guard<std::mutex> call(call_mu_);  // one parallel region at a time
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            items_ = items;
            next_.store(0);
            busy_ = workers_.size();
            ++gen_;
        }
        cv_.notify_all();
        drain();
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return busy_ == 0; });
        fn_ = nullptr;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

private:
    HostPool() {
        const unsigned hc = std::thread::hardware_concurrency();
        const unsigned n = hc > 1 ? hc - 1 : 0;
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    void drain() {
        for (std::size_t i; (i = next_.fetch_add(1)) < items_;) (*fn_)(i);
    }
    void loop() {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
            }
            drain();
            std::lock_guard<std::mutex> lk(mu_);
            if (--busy_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(std::size_t)>* fn_ = nullptr;
    std::size_t items_ = 0, busy_ = 0;
    std::atomic<std::size_t> next_{0};
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

// rows [lo, hi) of map `map` -> the PureComplex objects out[lo..hi)
// (search.hpp:247-253): facets in ascending order, each vector sized once
inline void fill_complexes(const wpm_result_t* r, int map, int m, int n, const std::vector<VertexSet>& u,
                           std::vector<PureComplex>& out, std::size_t lo, std::size_t hi) {
    const int W = r->words;
    const std::uint64_t* row = r->bits + (static_cast<std::size_t>(r->offsets[map]) + lo) * W;
    for (std::size_t j = lo; j < hi; ++j) {
        PureComplex& K = out[j];
        K.m = m;
        K.n = n;
        K.embedded = true;
        int k = 0;
        for (int w = 0; w < W; ++w) k += __builtin_popcountll(row[w]);
        K.facets.resize(static_cast<std::size_t>(k));
        VertexSet* f = K.facets.data();
        for (int w = 0; w < W; ++w)
            for (std::uint64_t x = row[w]; x; x &= x - 1) *f++ = u[static_cast<std::size_t>(w * 64 + __builtin_ctzll(x))];
        row += W;
    }
}

// rows of map `map` -> PureComplex (search.hpp:247-253): facets in
// ascending order, each vector sized once
inline std::vector<PureComplex> complexes_of(const wpm_result_t* r, int map, int m, int n,
                                             const std::vector<VertexSet>& u) {
    std::vector<PureComplex> out(static_cast<std::size_t>(r->counts[map]));
    const int W = r->words;
    const std::uint64_t* row = r->bits + static_cast<std::size_t>(r->offsets[map]) * W;
    for (auto& K : out) {
        K.m = m;
        K.n = n;
        K.embedded = true;
        int k = 0;
        for (int w = 0; w < W; ++w) k += __builtin_popcountll(row[w]);
        K.facets.resize(static_cast<std::size_t>(k));
        VertexSet* f = K.facets.data();
        for (int w = 0; w < W; ++w)
            for (std::uint64_t x = row[w]; x; x &= x - 1) *f++ = u[static_cast<std::size_t>(w * 64 + __builtin_ctzll(x))];
        row += W;
    }
    return out;
}

inline std::int64_t facet_cap_of(const std::vector<AffineProperty>& props) {
    std::int64_t cap = WPM_CAP_NONE;
    for (const auto& g : props) {
        if (!g.is_count_cap())
            throw std::invalid_argument("general affine properties are not supported by the B200 path (count caps only)");
        const std::int64_t c = g.constant - 1;
        cap = cap < 0 ? c : std::min(cap, c);
    }
    return cap;
}
}  // namespace detail

// binary_matroid (charmap.hpp:117-141): kernel 1 on device 0
inline PureComplex binary_matroid(const CharMatrixZ2& lam, int device = 0) {
    detail::Plan P;
    check(wpm_plan_create_charmaps(lam.n, lam.m, 1, lam.cols.data(), WPM_CAP_UBT, device, &P.p));
    PureComplex K;
    K.m = lam.m;
    K.n = lam.n;
    K.embedded = true;
    K.facets = detail::universe_of(P.p, 0);
    return K;
}

inline std::vector<VertexSet> matroid_universe(const DualCharMatrix& d, int device = 0) {
    return binary_matroid(charmap_of_dcm(d), device).facets;
}

// enumerate_wpm (search.hpp:141-258)
inline std::vector<PureComplex> enumerate_wpm(const SearchJob& job) {
    if (job.facets.empty()) throw purity_error("incidence of an empty facet set");
    std::vector<std::uint64_t> f;
    f.reserve(job.facets.size());
    for (const auto& v : job.facets) f.push_back(v.bits);
    wpm_job_t j{};
    j.m = job.m;
    j.n = job.n;
    j.num_facets = static_cast<std::int32_t>(f.size());
    j.facets = f.data();
    j.facet_cap = detail::facet_cap_of(job.properties);
    j.required = job.required.data();
    j.num_required = static_cast<std::int32_t>(job.required.size());
    j.forbidden = job.forbidden.data();
    j.num_forbidden = static_cast<std::int32_t>(job.forbidden.size());
    j.device = job.device;
    // SearchJob::progress (search.hpp:54): forwarded from the C-ABI's calls
    auto relay = [](std::int64_t done, std::int64_t total, void* user) {
        (*static_cast<const std::function<void(long long, long long)>*>(user))(done, total);
    };
    if (job.progress) {
        j.progress = relay;
        j.progress_user = const_cast<std::function<void(long long, long long)>*>(&job.progress);
    }
    j.devices = job.devices.empty() ? nullptr : job.devices.data();
    j.num_devices = static_cast<std::int32_t>(job.devices.size());
    detail::Result R;
    check(wpm_enumerate(&j, &R.r));
    // result bits index the universe in canonical (ascending) order
    std::vector<VertexSet> sorted = job.facets;
    std::sort(sorted.begin(), sorted.end());
    return detail::complexes_of(R.r, 0, job.m, job.n, sorted);
}

// the Algorithm-2 per-orbit loop (pipeline.hpp:58-72) for one n in one launch:
// element i = enumerate_wpm over matroid_universe(idcm_orbits(n, p)[i]) with the UBT cap
inline std::vector<std::vector<PureComplex>> enumerate_orbits(int n, int p = 4, int device = 0,
                                                              std::int64_t facet_cap = WPM_CAP_UBT) {
    detail::Plan P;
    check(wpm_plan_create_orbits(n, p, facet_cap, device, &P.p));
    std::int64_t total = 0;
    check(wpm_plan_run(P.p, 0, 1, &total));
    detail::Result R;
    check(wpm_plan_fetch(P.p, &R.r));
    const int K = R.r->num_maps;
    std::vector<std::vector<VertexSet>> uni(static_cast<std::size_t>(K));
    for (int i = 0; i < K; ++i) uni[static_cast<std::size_t>(i)] = detail::universe_of(P.p, i);
    // the reference's return objects, built on the persistent host pool:
    // every map's vector sized (one item per map), then filled in chunks of
    // 2048 rows (the maps hold 2,043-17,606 WPMs at n = 5)
    std::vector<std::vector<PureComplex>> out(static_cast<std::size_t>(K));
    detail::HostPool& pool = detail::HostPool::get();
    pool.run(static_cast<std::size_t>(K), [&](std::size_t i) { out[i].resize(static_cast<std::size_t>(R.r->counts[i])); });
    constexpr std::size_t kChunk = 2048;
    std::vector<std::pair<int, std::size_t>> chunks;  // (map, first row)
    for (int i = 0; i < K; ++i)
        for (std::size_t lo = 0; lo < static_cast<std::size_t>(R.r->counts[i]); lo += kChunk) chunks.emplace_back(i, lo);
    pool.run(chunks.size(), [&](std::size_t c) {
        const int i = chunks[c].first;
        const std::size_t lo = chunks[c].second, cnt = static_cast<std::size_t>(R.r->counts[i]);
        detail::fill_complexes(R.r, i, n + p, n, uni[static_cast<std::size_t>(i)], out[static_cast<std::size_t>(i)], lo,
                               std::min(cnt, lo + kChunk));
    });
    return out;
}

// complex_io.hpp:21-39
inline void write_complex(std::ostream& os, const PureComplex& K) {
    os << K.m << ' ' << K.n << '\n';
    for (const VertexSet& f : K.facets) {
        bool first = true;
        for (std::uint64_t b = f.bits; b; b &= b - 1) {
            if (!first) os << ' ';
            os << __builtin_ctzll(b);
            first = false;
        }
        os << '\n';
    }
}

inline void write_complexes(std::ostream& os, const std::vector<PureComplex>& list) {
    for (std::size_t i = 0; i < list.size(); ++i) {
        if (i > 0) os << '\n';
        write_complex(os, list[i]);
    }
}

// ---- Algorithm 2 lines 7 and 13 (pipeline.hpp:58-89) on the device

// PipelineResult's line7 / line13 (pipeline.hpp:23-30) and the line-13
// survivors in the labeled set's order (the `survivors` of pipeline.hpp:74-89)
struct Line13Result {
    long long line7 = 0;
    long long line13 = 0;
    std::vector<PureComplex> survivors;
    double ms_union = 0, ms_filter = 0;
};

namespace detail {
struct Complexes {
    wpm_complexes_t* c = nullptr;
    ~Complexes() { wpm_complexes_free(c); }
};
inline std::vector<PureComplex> complexes_of(const wpm_complexes_t* c) {
    std::vector<PureComplex> out;
    out.reserve(static_cast<std::size_t>(c->count));
    for (std::int64_t i = 0; i < c->count; ++i) {
        PureComplex K;
        K.m = c->m;
        K.n = c->n;
        for (std::int64_t j = c->offsets[i]; j < c->offsets[i + 1]; ++j) K.facets.emplace_back(c->facets[j]);
        out.push_back(std::move(K));
    }
    return out;
}
}  // namespace detail

// lines 1-13 of pipeline(n, db) (pipeline.hpp:52-89): every orbit map, UBT cap
inline Line13Result pipeline_line13(int n, int p = 4, int device = 0, std::int64_t facet_cap = WPM_CAP_UBT) {
    detail::Complexes C;
    check(wpm_pipeline_line13(n, p, facet_cap, device, &C.c));
    Line13Result r;
    r.line7 = C.c->line7;
    r.line13 = C.c->line13;
    r.ms_union = C.c->ms_union;
    r.ms_filter = C.c->ms_filter;
    r.survivors = detail::complexes_of(C.c);
    return r;
}

// is_seed (classify.hpp:51-53) over a batch, on the device
inline std::vector<char> is_seed(const std::vector<PureComplex>& list, int device = 0) {
    std::vector<char> out(list.size(), 0);
    std::size_t i = 0;
    while (i < list.size()) {  // one call per run of equal (m, n)
        std::size_t j = i;
        std::vector<std::int64_t> off{0};
        std::vector<std::uint64_t> fac;
        while (j < list.size() && list[j].m == list[i].m && list[j].n == list[i].n) {
            for (const auto& f : list[j].facets) fac.push_back(f.bits);
            off.push_back(static_cast<std::int64_t>(fac.size()));
            ++j;
        }
        std::vector<std::uint8_t> flags(j - i);
        check(wpm_seed_flags(list[i].m, list[i].n, static_cast<std::int64_t>(j - i), off.data(), fac.data(), device,
                             flags.data()));
        for (std::size_t k = i; k < j; ++k) out[k] = static_cast<char>(flags[k - i] & 1);
        i = j;
    }
    return out;
}
inline bool is_seed(const PureComplex& K, int device = 0) { return is_seed(std::vector<PureComplex>{K}, device)[0]; }

// ---- Algorithm 2 line 15 (pipeline.hpp:91-103) on the device

// canonical_form (isomorphism.hpp:228-303) over a batch; m <= 15, n <= 11
inline std::vector<PureComplex> canonical_form(const std::vector<PureComplex>& list, int device = 0) {
    std::vector<PureComplex> out(list.size());
    std::size_t i = 0;
    while (i < list.size()) {  // one call per run of equal (m, n)
        std::size_t j = i;
        std::vector<std::int64_t> off{0};
        std::vector<std::uint64_t> fac;
        while (j < list.size() && list[j].m == list[i].m && list[j].n == list[i].n) {
            for (const auto& f : list[j].facets) fac.push_back(f.bits);
            off.push_back(static_cast<std::int64_t>(fac.size()));
            ++j;
        }
        std::vector<std::uint64_t> canon(fac.size() + 1);
        check(wpm_canonical_forms(list[i].m, list[i].n, static_cast<std::int64_t>(j - i), off.data(), fac.data(),
                                  device, canon.data(), nullptr));
        for (std::size_t k = i; k < j; ++k) {
            PureComplex K;
            K.m = list[k].m;
            K.n = list[k].n;
            for (std::int64_t q = off[k - i]; q < off[k - i + 1]; ++q) K.facets.emplace_back(canon[q]);
            out[k] = std::move(K);
        }
        i = j;
    }
    return out;
}
inline PureComplex canonical_form(const PureComplex& K, int device = 0) {
    return canonical_form(std::vector<PureComplex>{K}, device)[0];
}

// PipelineResult's line7 / line13 / line15 (pipeline.hpp:23-30) and the
// line-15 representatives (canonical forms, order of first appearance:
// the `reps` of pipeline.hpp:91-101)
struct Line15Result {
    long long line7 = 0, line13 = 0, line15 = 0;
    std::vector<PureComplex> reps;
    double ms_canon = 0, ms_dedupe = 0;
};

// lines 1-15 of pipeline(n, db) (pipeline.hpp:52-103): every orbit map, UBT cap
inline Line15Result pipeline_line15(int n, int p = 4, int device = 0, std::int64_t facet_cap = WPM_CAP_UBT) {
    detail::Complexes C;
    check(wpm_pipeline_line15(n, p, facet_cap, device, &C.c));
    Line15Result r;
    r.line7 = C.c->line7;
    r.line13 = C.c->line13;
    r.line15 = C.c->line15;
    r.ms_canon = C.c->ms_canon;
    r.ms_dedupe = C.c->ms_dedupe;
    r.reps = detail::complexes_of(C.c);
    return r;
}

}  // namespace plseeds_b200

// ---------------------------------------------------------------------------
// Adapter for programs that include the reference headers first.
#ifdef PLSEEDS_SEARCH_HPP
namespace plseeds {
namespace b200 {

// Drop-in for plseeds::enumerate_wpm(job).  Honours job.basis exactly: the
// reference enumerates base + one candidate per block of
// combination_space(kb) (search.hpp:81-104, :152-153) -- at most two
// generators of each induced block, any subset of the free singletons
// (g >= covered), nothing else.  A facet on which every usable generator
// vanishes is fixed to its base bit; those pins go to the device search.
// Every device WPM K is then written in coordinates, K xor base = sum of
// x_g gens[g] (the generators are independent, so x is unique), and kept iff
// x exists and obeys the combination-space rules -- for bases produced by
// convenient_basis / apply_link_constraints this keeps every WPM; for a
// hand-made basis it drops exactly the K the reference cannot reach.  The
// candidate cap throws cap_exceeded_error like the reference (search.hpp:147-150).
inline std::vector<PureComplex> enumerate_wpm(const SearchJob& job) {
    const KernelBasis& kb = job.basis;
    const std::uint64_t space = combination_space(kb).size_saturated();
    if (space > job.candidate_cap)
        throw cap_exceeded_error("combination space of " + std::to_string(space) + " candidates exceeds cap " +
                                 std::to_string(job.candidate_cap));
    const int M = static_cast<int>(job.facets.size());
    const int s = kb.s();
    const int first_free = kb.pinned_ones + kb.pinned_zeros;
    // usable generators and their block (search.hpp:85-103): block id, or -1
    // for a free singleton; unusable ones (pinned, or skipped by `covered`) -2
    std::vector<int> block_of(static_cast<std::size_t>(s), -2);
    int covered = first_free;
    for (std::size_t b = 0; b < kb.blocks.size(); ++b) {
        for (int i = 0; i < kb.blocks[b].width; ++i) block_of[static_cast<std::size_t>(kb.blocks[b].offset + i)] = static_cast<int>(b);
        covered = std::max(covered, kb.blocks[b].offset + kb.blocks[b].width);
    }
    for (int g = covered; g < s; ++g) block_of[static_cast<std::size_t>(g)] = -1;
    BitVec base(M);
    for (int g = 0; g < kb.pinned_ones; ++g) base ^= kb.gens[static_cast<std::size_t>(g)];
    std::vector<int> req, forb;
    {
        BitVec any_free(M);
        for (int g = 0; g < s; ++g)
            if (block_of[static_cast<std::size_t>(g)] >= -1)
                for (std::size_t w = 0; w < any_free.words.size(); ++w)
                    any_free.words[w] |= kb.gens[static_cast<std::size_t>(g)].words[w];
        for (int j = 0; j < M; ++j)
            if (!any_free.test(j)) (base.test(j) ? req : forb).push_back(j);
    }
    plseeds_b200::SearchJob j;
    j.m = job.m;
    j.n = job.n;
    for (const auto& f : job.facets) j.facets.emplace_back(f.bits);
    for (const auto& g : job.properties) j.properties.push_back({g.weights, g.constant});
    j.required = req;
    j.forbidden = forb;
    j.progress = job.progress;
    // reduced echelon of the usable generators, each row remembering which
    // generators it sums (coordinate bookkeeping)
    const std::size_t sw = (static_cast<std::size_t>(s) + 63) / 64;
    std::vector<BitVec> ech;
    std::vector<std::vector<std::uint64_t>> comb;
    std::vector<int> lead;
    for (int g = 0; g < s; ++g) {
        if (block_of[static_cast<std::size_t>(g)] < -1) continue;
        BitVec v = kb.gens[static_cast<std::size_t>(g)];
        std::vector<std::uint64_t> c(sw, 0);
        c[static_cast<std::size_t>(g) / 64] |= std::uint64_t{1} << (g % 64);
        for (std::size_t i = 0; i < ech.size(); ++i)
            if (v.test(lead[i])) {
                v ^= ech[i];
                for (std::size_t w = 0; w < sw; ++w) c[w] ^= comb[i][w];
            }
        int l = -1;
        for (int b = 0; b < M && l < 0; ++b)
            if (v.test(b)) l = b;
        if (l < 0) continue;  // dependent generator: not a basis; its span is still covered
        for (std::size_t i = 0; i < ech.size(); ++i)
            if (ech[i].test(l)) {
                ech[i] ^= v;
                for (std::size_t w = 0; w < sw; ++w) comb[i][w] ^= c[w];
            }
        ech.push_back(std::move(v));
        comb.push_back(std::move(c));
        lead.push_back(l);
    }
    // facet mask -> index in job.facets (the universe may be in any order)
    std::vector<std::pair<std::uint64_t, int>> index;
    index.reserve(job.facets.size());
    for (int i = 0; i < M; ++i) index.emplace_back(job.facets[static_cast<std::size_t>(i)].bits, i);
    std::sort(index.begin(), index.end());
    std::vector<PureComplex> out;
    std::vector<int> per_block(kb.blocks.size());
    for (auto& K : plseeds_b200::enumerate_wpm(j)) {
        BitVec x = base;
        for (const auto& f : K.facets) {
            const auto it = std::lower_bound(index.begin(), index.end(), std::make_pair(f.bits, -1));
            x.flip(it->second);
        }
        std::vector<std::uint64_t> coords(sw, 0);
        for (std::size_t i = 0; i < ech.size(); ++i)
            if (x.test(lead[i])) {
                x ^= ech[i];
                for (std::size_t w = 0; w < sw; ++w) coords[w] ^= comb[i][w];
            }
        if (x.any()) continue;  // not in base + span
        std::fill(per_block.begin(), per_block.end(), 0);
        bool ok = true;
        for (int g = 0; g < s && ok; ++g) {
            if (!((coords[static_cast<std::size_t>(g) / 64] >> (g % 64)) & 1u)) continue;
            const int b = block_of[static_cast<std::size_t>(g)];
            if (b >= 0) ok = ++per_block[static_cast<std::size_t>(b)] <= 2;  // {0, singles, pairs}
        }
        if (!ok) continue;
        std::vector<VertexSet> fs;
        for (const auto& f : K.facets) fs.emplace_back(f.bits);
        out.emplace_back(job.m, job.n, std::move(fs), /*embedded=*/true);
    }
    return out;
}

}  // namespace b200
}  // namespace plseeds
#endif

// Line-13 adapter for programs that include plseeds/classify.hpp (or
// pipeline.hpp) first: the reference's own PureComplex type in and out.
#ifdef PLSEEDS_CLASSIFY_HPP
namespace plseeds {
namespace b200 {

// is_seed(K) (classify.hpp:51-53) for a batch, on the device
inline std::vector<char> is_seed(const std::vector<PureComplex>& list, int device = 0) {
    std::vector<plseeds_b200::PureComplex> in;
    in.reserve(list.size());
    for (const auto& K : list) {
        plseeds_b200::PureComplex k;
        k.m = K.m;
        k.n = K.n;
        for (const auto& f : K.facets) k.facets.emplace_back(f.bits);
        in.push_back(std::move(k));
    }
    return plseeds_b200::is_seed(in, device);
}

struct Line13Result {
    long long line7 = 0, line13 = 0;
    std::vector<PureComplex> survivors;  // pipeline.hpp:74-89, in order
};

namespace detail {
inline std::vector<PureComplex> to_ref(const std::vector<plseeds_b200::PureComplex>& in, bool embedded) {
    std::vector<PureComplex> out;
    out.reserve(in.size());
    for (const auto& K : in) {
        std::vector<VertexSet> fs;
        fs.reserve(K.facets.size());
        for (const auto& f : K.facets) fs.emplace_back(f.bits);
        out.emplace_back(K.m, K.n, std::move(fs), embedded);
    }
    return out;
}
}  // namespace detail

// canonical_form(K) (isomorphism.hpp:228-303) for a batch, on the device
inline std::vector<PureComplex> canonical_form(const std::vector<PureComplex>& list, int device = 0) {
    std::vector<plseeds_b200::PureComplex> in;
    in.reserve(list.size());
    for (const auto& K : list) {
        plseeds_b200::PureComplex k;
        k.m = K.m;
        k.n = K.n;
        for (const auto& f : K.facets) k.facets.emplace_back(f.bits);
        in.push_back(std::move(k));
    }
    const auto canon = plseeds_b200::canonical_form(in, device);
    std::vector<PureComplex> out;
    out.reserve(canon.size());
    for (std::size_t i = 0; i < canon.size(); ++i) {
        std::vector<VertexSet> fs;
        fs.reserve(canon[i].facets.size());
        for (const auto& f : canon[i].facets) fs.emplace_back(f.bits);
        out.emplace_back(list[i].m, list[i].n, std::move(fs), list[i].embedded);  // isomorphism.hpp:302
    }
    return out;
}

struct Line15Result {
    long long line7 = 0, line13 = 0, line15 = 0;
    std::vector<PureComplex> reps;  // pipeline.hpp:91-101, first-appearance order
};

// lines 1-15 of pipeline(n, db) (pipeline.hpp:52-103) with the reference's types
inline Line15Result pipeline_line15(int n, int device = 0) {
    const auto r = plseeds_b200::pipeline_line15(n, 4, device);
    Line15Result out;
    out.line7 = r.line7;
    out.line13 = r.line13;
    out.line15 = r.line15;
    out.reps = detail::to_ref(r.reps, false);
    return out;
}

// lines 1-13 of pipeline(n, db) (pipeline.hpp:52-89) with the reference's types
inline Line13Result pipeline_line13(int n, int device = 0) {
    const auto r = plseeds_b200::pipeline_line13(n, 4, device);
    Line13Result out;
    out.line7 = r.line7;
    out.line13 = r.line13;
    out.survivors.reserve(r.survivors.size());
    for (const auto& K : r.survivors) {
        std::vector<VertexSet> fs;
        fs.reserve(K.facets.size());
        for (const auto& f : K.facets) fs.emplace_back(f.bits);
        out.survivors.emplace_back(K.m, K.n, std::move(fs));
    }
    return out;
}

}  // namespace b200
}  // namespace plseeds
#endif

#endif
