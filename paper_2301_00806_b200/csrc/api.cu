// api.cu -- the C-ABI (include/wpm_b200.h) and the host orchestration.
//
// Host side of the path: IDCM orbits (charmap.hpp:212-281) and
// charmap_of_dcm (charmap.hpp:155-204) in C++, then everything
// data-parallel on the device: kernel 1 (universes), kernel 2 (incidence),
// kernel 3 (search), the canonical sort.  The per-orbit sequential loop of
// pipeline.hpp:58-72 becomes ONE persistent launch over every map's search
// tree; job.threads / parallel_for_index (parallel.hpp:27-54) becomes the
// device work queue.  There is no CPU fallback: no device, no result.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <unordered_map>
#include <chrono>
#include <cmath>
#include <functional>
#include <cstdlib>
#include <climits>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/wpm_b200.h"
#include "kbasis.h"
#include "wpm_dev.cuh"
#include "wpm_internal.h"

using namespace wpm;

namespace {

thread_local std::string g_err;

// WPM_TRACE=1: report a pending (non-sticky) CUDA error at a checkpoint
void trace_pending(const char* where) {
    static const bool on = std::getenv("WPM_TRACE") != nullptr;
    if (!on) return;
    const cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) std::fprintf(stderr, "[wpm] pending CUDA error at %s: %s\n", where, cudaGetErrorString(e));
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// WPM_TRACE=2: every CUDA runtime call made through CU() that takes >= 2 us
// of host time is reported with its source line (e2e engineering)
const bool g_trace_calls = [] {
    const char* e = std::getenv("WPM_TRACE");
    return e && std::atoi(e) >= 2;
}();
struct CallTimer {
    const char* what;
    int line;
    std::chrono::steady_clock::time_point t0;
    CallTimer(const char* w, int l) : what(w), line(l) {
        if (g_trace_calls) t0 = std::chrono::steady_clock::now();
    }
    ~CallTimer() {
        if (!g_trace_calls) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        if (us >= 2.0) std::fprintf(stderr, "[wpm]   call %8.1f us  api.cu:%d  %.60s\n", us, line, what);
    }
};

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_;                                                                           \
        {                                                                                         \
            CallTimer ct_(#call, __LINE__);                                                       \
            e_ = (call);                                                                          \
        }                                                                                         \
        if (e_ != cudaSuccess)                                                                    \
            return fail(WPM_EINTERNAL, std::string(#call) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// Device buffers come from the stream-ordered caching allocator (the
// device's default memory pool with an unbounded release threshold), so
// repeated plans / one-shot calls reuse memory instead of paying
// cudaMalloc / cudaFree each time.
thread_local cudaStream_t g_alloc_stream = nullptr;

void init_pool(int device) {
    static bool done[64] = {false};
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

// Buffers of a destroyed plan (its stream synchronised first) are kept per
// device and handed to the next plan's DevBuf::ensure: a one-shot call
// allocates ~20 buffers, and each cudaMallocAsync / cudaFreeAsync pair cost
// ~2.5 us of host time (WPM_TRACE=2).  Local DevBufs of API functions free
// through the stream as before (g_recycle is only set inside
// wpm_plan_destroy).
thread_local bool g_recycle = false;
struct BlockCache {
    std::mutex mu;
    std::vector<std::pair<void*, size_t>> blocks[64];
    size_t bytes[64] = {};
    static constexpr size_t kMaxBytes = size_t(8) << 30;
    void* take(int dev, size_t want, size_t* got) {
        if (dev < 0 || dev >= 64) return nullptr;
        std::lock_guard<std::mutex> lk(mu);
        auto& v = blocks[dev];
        size_t best = SIZE_MAX;
        for (size_t i = 0; i < v.size(); ++i)  // best fit, at most 2x (+64 KB) the request
            if (v[i].second >= want && v[i].second <= 2 * want + (64 << 10) &&
                (best == SIZE_MAX || v[i].second < v[best].second))
                best = i;
        if (best == SIZE_MAX) return nullptr;
        void* p = v[best].first;
        *got = v[best].second;
        bytes[dev] -= v[best].second;
        v[best] = v.back();
        v.pop_back();
        return p;
    }
    bool put(int dev, void* p, size_t sz) {
        if (dev < 0 || dev >= 64) return false;
        std::lock_guard<std::mutex> lk(mu);
        if (bytes[dev] + sz > kMaxBytes) return false;
        blocks[dev].emplace_back(p, sz);
        bytes[dev] += sz;
        return true;
    }
};
BlockCache g_blocks;

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    int dev = -1;
    int ensure(size_t count) {
        if (count <= n && p) return 0;
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
        s = g_alloc_stream;
        const size_t c = std::max<size_t>(count, 1);
        if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
        size_t got = 0;
        if (void* q = g_blocks.take(dev, c * sizeof(T), &got)) {
            p = static_cast<T*>(q);
            n = got / sizeof(T);
            return 0;
        }
        cudaError_t e;
        {
            CallTimer ct("cudaMallocAsync (DevBuf::ensure)", __LINE__);
            e = cudaMallocAsync(reinterpret_cast<void**>(&p), c * sizeof(T), s);
        }
        if (e != cudaSuccess) {
            p = nullptr;
            return 1;
        }
        n = c;
        return 0;
    }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;  // owning: a copy would free twice
    DevBuf& operator=(const DevBuf&) = delete;
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
        std::swap(s, o.s);
        std::swap(dev, o.dev);
    }
    ~DevBuf() {
        if (!p) return;
        if (g_recycle && g_blocks.put(dev, p, n * sizeof(T))) return;
        cudaFreeAsync(p, s);
    }
};

// Result rows live in page-locked host memory from a grow-only cache, so the
// D2H of the canonical list runs at full PCIe/C2C speed without paying the
// pinning cost on every call; wpm_result_free returns the block.
struct PinnedCache {
    std::mutex mu;
    std::vector<std::pair<void*, size_t>> free_blocks;
    void* get(size_t bytes, size_t* got) {
        {
            std::lock_guard<std::mutex> lk(mu);
            size_t best = (size_t)-1;
            for (size_t i = 0; i < free_blocks.size(); ++i)
                if (free_blocks[i].second >= bytes && (best == (size_t)-1 || free_blocks[i].second < free_blocks[best].second))
                    best = i;
            if (best != (size_t)-1) {
                auto b = free_blocks[best];
                free_blocks.erase(free_blocks.begin() + (long)best);
                *got = b.second;
                return b.first;
            }
        }
        void* p = nullptr;
        const size_t sz = std::max<size_t>(bytes, 1 << 20);
        if (cudaHostAlloc(&p, sz, cudaHostAllocPortable) != cudaSuccess) return nullptr;
        *got = sz;
        return p;
    }
    void put(void* p, size_t bytes) {
        std::lock_guard<std::mutex> lk(mu);
        free_blocks.emplace_back(p, bytes);
    }
};
PinnedCache g_pinned;
// rows of the last run of each workload (plan signature): sizes the sort grid
std::mutex g_rows_mu;
std::map<std::string, long long> g_rows_seen;
std::mutex g_block_mu;
std::unordered_map<void*, size_t> g_block_size;

// WPM_TRACE=1: host-side phase timings on stderr
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point t0;
    Trace() : on(std::getenv("WPM_TRACE") != nullptr), t0(std::chrono::steady_clock::now()) {}
    void mark(const char* what) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[wpm] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

int64_t cyclic_bound(int n) {  // affine_property.hpp:35-45
    auto binom = [](int64_t top, int64_t k) -> int64_t {
        if (top < k) return 0;
        int64_t r = 1;
        for (int64_t i = 1; i <= k; ++i) r = r * (top - k + i) / i;
        return r;
    };
    return binom(n + 4 - (n + 1) / 2, 4) + binom(n + 3 - n / 2, 4);
}

}  // namespace

struct wpm_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 0;
    int n = 0, m = 0, num_maps = 0;
    int64_t facet_cap = WPM_CAP_UBT;
    std::vector<int32_t> M, N, cap;
    std::vector<MapDesc> desc;
    int maxM = 0, maxN = 0, maxDepth = 0, w32 = 0, mw = 0, rw = 0;
    // device tables
    DevBuf<MapDesc> d_maps;
    DevBuf<uint32_t> d_facets, d_ridges;
    DevBuf<uint16_t> d_fr, d_rp;
    DevBuf<uint8_t> d_npar;
    DevBuf<int32_t> d_tmpi;
    // pins (map-major mw words), optional
    std::vector<uint32_t> pin_in, pin_out;
    bool has_pins = false;
    DevBuf<uint32_t> d_pin_in, d_pin_out;
    // work queue
    DevBuf<uint32_t> d_qrec;
    DevBuf<unsigned long long> d_qready, d_qctl;
    int qcap = 0, recw = 0;
    DevBuf<int32_t> d_task_map, d_task_f, d_task_kind;
    DevBuf<int32_t> d_map_first;  // root tasks per map, prefix (the per-map queues)
    std::vector<int32_t> h_map_first;
    // outputs
    DevBuf<uint32_t> d_out_keys, d_sorted_bits;  // key rows from kernel 3; canonical rows
    DevBuf<uint32_t> d_bucket;  // bucketed-sort scratch (its count block stays zero between sorts)
    long long bucket_cap = -1, bucket_facets = -1;  // the layout the zeroed count block belongs to
    DevBuf<uint16_t> d_sorted_map;
    DevBuf<unsigned long long> d_out_ctl, d_per_map;
    DevBuf<uint8_t> d_temp;
    unsigned long long out_cap = 0;
    // last run
    long long total = 0, nodes = 0, tasks = 0, dups = 0, reruns = 0;
    unsigned long long node_budget = 0;  // 0 = enumerate everything
    bool truncated = false;              // the last run stopped at the node budget
    std::vector<unsigned long long> per_map;
    float ms_search = 0, ms_sort = 0, ms_total = 0;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    int warps = 0;
    long long h2d = 0, d2h = 0;  // bytes moved by create + run + fetch
    bool ran = false;
    // Algorithm 2 lines 7 / 13 of the last run (k5_line13.cu)
    DevBuf<uint16_t> d_gidx, d_unrank, d_l13_map;
    DevBuf<uint32_t> d_l13_keys, d_l13_rows, d_l13_iota, d_l13_uidx, d_l13_sidx;
    DevBuf<uint8_t> d_l13_flags, d_l13_temp;
    DevBuf<int> d_l13_num;
    DevBuf<unsigned long long> d_l13_dups;
    std::vector<uint16_t> unrank;  // all n-subsets of [m], ascending, 0-based masks
    long long line7 = -1, line13 = -1;
    int gw = 0;
    float ms_union = 0, ms_filter = 0;
    // Algorithm 2 line 15 of the last line-13 result (k7_line15.cu)
    DevBuf<uint32_t> d_l15_rows, d_l15_sidx, d_l15_iota, d_l15_rep;
    DevBuf<uint8_t> d_l15_first, d_l15_temp;
    DevBuf<int> d_l15_num;
    DevBuf<unsigned long long> d_l15_ctl, d_l15_cost, d_l15_ckey;
    DevBuf<uint16_t> d_l15_cdata;
    long long l15_hits = 0;
    long long line15 = -1, l15_leaves = 0, l15_steps = 0;
    int l15_kmax = 0, l15_mnfcap = 0, l15_launches = 0;
    float ms_canon = 0, ms_dedupe = 0;
    // Algorithm 1 (k6_odometer.cu): the reference's combination space per map
    std::vector<CombinationSpaceHost> spaces;
    DevBuf<OdoMap> d_odo_maps;
    DevBuf<int> d_odo_blk;
    DevBuf<uint32_t> d_odo_words;
    DevBuf<unsigned long long> d_odo_ctl;
    long long leaves = 0, checked = 0;
    double ms_prep = 0, ms_basis = 0;
    bool spaces_ok = false;
    // frontier (split below the root) and shared-frontier claims
    DevBuf<uint32_t> d_front;
    DevBuf<unsigned long long> d_front_ctl, d_acc;
    unsigned long long front_cap = 0;
    long long frontier = 0;       // records of the last split
    int split_depth = 0;          // > 0: split at this branch depth, then search the frontier
    long long claim_count = 0;
    unsigned long long* claim_ctr = nullptr;
    int claim_devices = 1;        // GPUs claiming from the shared frontier (fair-share claim cap)
    // progress callback (search.hpp:54): root tasks finished / root tasks
    void (*progress_fn)(int64_t, int64_t, void*) = nullptr;
    void* progress_user = nullptr;
    unsigned long long* progress_host = nullptr;  // host-mapped
    unsigned long long* progress_dev = nullptr;
    DevBuf<unsigned int> d_root_pend;
    // multi-GPU: plans of the same maps on the other devices of the job
    std::vector<wpm_plan*> peers;
    std::vector<double> dev_ms;   // per device: kernel-3 ms of the last run
    std::vector<long long> dev_nodes;
    void* claim_raw = nullptr;  // the shared claim counter of a multi-GPU job (the leader's)
    std::function<int(int, wpm_plan_t**)> recreate;  // the same plan on another device
    DevBuf<uint32_t> d_front2, d_gather, d_front_all;
    bool split_kept = false;  // wpm_plan_split ran: the claim run appends to its rows
    bool root_stats = false;  // count search nodes per root task / frontier record
    std::vector<uint32_t> h_facets;  // host copy of every universe (wpm_plan_universe)
    std::string signature;           // the workload: (m, n, cap, every universe's facet count)
    unsigned long long h_dups = 0;   // sort results, read back with the run's synchronisation
    std::vector<long long> h_first;
    // Pinned staging for the small copies of create / run: a pageable
    // cudaMemcpyAsync stages through the driver, and a pageable D2H blocks the
    // host until the stream drains -- one round trip per small read.  H2D
    // sources are bump-allocated (reset only after a synchronisation of the
    // stream); D2H results land in the mailbox at the end of the block.
    uint8_t* stage = nullptr;
    size_t stage_cap = 0, stage_used = 0;
    ~wpm_plan();
    DevBuf<unsigned long long> d_root_nodes;
    long long root_count = 0;
    int ntasks = 0, frame_cap = 64;
    int fr_words = 0, rp_words = 0;  // uint16 entries of the fr / rp tables over every map
    bool full_depth = false;
};

namespace {
constexpr size_t kStageBytes = 1 << 20;
constexpr size_t kMailBytes = 64 << 10;  // >= 128 + 8 (K + 1) for K <= 4096 maps
// mailbox slots (D2H): out_ctl[0..3], qctl[0..7], duplicates, then per map
constexpr size_t kMailOctl = 0, kMailQc = 32, kMailDups = 96, kMailMaps = 128;

int stage_init(wpm_plan* P) {
    size_t got = 0;
    P->stage = static_cast<uint8_t*>(g_pinned.get(kStageBytes, &got));
    if (!P->stage) return fail(WPM_EINTERNAL, "pinned host allocation failed (staging)");
    P->stage_cap = got;
    P->stage_used = 0;
    return WPM_OK;
}
uint8_t* mail(wpm_plan* P, size_t off) { return P->stage + P->stage_cap - kMailBytes + off; }
// H2D of a small host array through the pinned staging block (pageable when
// the block is full: correct, just slower)
cudaError_t h2d_async(wpm_plan* P, void* dst, const void* src, size_t bytes) {
    if (!bytes) return cudaSuccess;
    const size_t off = (P->stage_used + 15) & ~size_t(15);
    if (P->stage && off + bytes <= P->stage_cap - kMailBytes) {
        std::memcpy(P->stage + off, src, bytes);
        P->stage_used = off + bytes;
        src = P->stage + off;
    }
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, P->stream);
}
// the stream is idle: staged sources may be reused
void stage_reset(wpm_plan* P) { P->stage_used = 0; }
}  // namespace

wpm_plan::~wpm_plan() {
    if (stage) g_pinned.put(stage, stage_cap);
}

// ------------------------------------------------------------------ host

extern "C" const char* wpm_last_error(void) { return g_err.c_str(); }

extern "C" int wpm_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

extern "C" int64_t wpm_cyclic_facet_bound(int32_t n) { return cyclic_bound(n); }

// idcm_orbits (charmap.hpp:212-281): one representative per S_n x GL-free
// (column permutation) orbit of injective [M; I_p]; representative = the
// lexicographically least sorted row list over the p! bit shuffles; the
// representatives sorted; identity rows appended.
// idcm_orbits (charmap.hpp:212-281): one representative per S_n x S_p orbit
// of injective dual matrices [M; I_p] -- the lex-min sorted row list over the
// p! column permutations (:237-249), representatives in sorted order
// (:268), identity rows appended (:277).  A row set is a bitmask over the
// 2^p vectors; for sets of equal size the sorted-list order is "the set
// holding the lowest element of the symmetric difference is smaller", and a
// column permutation acts on a mask through per-byte lookup tables built
// once per p (0.35 ms -> ~0.03 ms per call at n = 5).
namespace {
struct OrbitTables {
    int p = 0, words = 0;                       // mask words of 64 bits over 2^p vectors
    std::vector<std::vector<uint32_t>> img;     // per permutation: image of every vector
    std::vector<uint64_t> byte_img;             // [perm][chunk][byte][word] -> image mask words
};
inline bool set_less(const uint64_t* a, const uint64_t* b, int words) {
    for (int w = 0; w < words; ++w) {
        const uint64_t x = a[w] ^ b[w];
        if (x) return (a[w] & (x & (0 - x))) != 0;
    }
    return false;
}
const OrbitTables& orbit_tables(int p) {
    static std::mutex mu;
    static std::map<int, OrbitTables> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(p);
    if (it != cache.end()) return it->second;
    OrbitTables T;
    T.p = p;
    const int nv = 1 << p;
    T.words = (nv + 63) / 64;
    std::vector<int> perm(p);
    std::iota(perm.begin(), perm.end(), 0);
    do {
        std::vector<uint32_t> im(nv, 0);
        for (int v = 0; v < nv; ++v)
            for (int b = 0; b < p; ++b)
                if ((v >> b) & 1) im[v] |= 1u << perm[b];
        T.img.push_back(std::move(im));
    } while (std::next_permutation(perm.begin(), perm.end()));
    const int chunks = (nv + 7) / 8;
    if (p > 5) return cache.emplace(p, std::move(T)).first->second;  // tables would be too big: direct images
    T.byte_img.assign(T.img.size() * chunks * 256 * T.words, 0);
    for (size_t q = 0; q < T.img.size(); ++q)
        for (int c = 0; c < chunks; ++c)
            for (int x = 0; x < 256; ++x) {
                uint64_t* dst = &T.byte_img[(((q * chunks) + c) * 256 + x) * T.words];
                for (int bit = 0; bit < 8; ++bit) {
                    const int v = c * 8 + bit;
                    if (v < nv && ((x >> bit) & 1)) dst[T.img[q][v] >> 6] |= 1ull << (T.img[q][v] & 63);
                }
            }
    return cache.emplace(p, std::move(T)).first->second;
}
}  // namespace

extern "C" int32_t wpm_idcm_orbits(int32_t n, int32_t p, uint32_t* rows_out, int32_t cap) {
    if (n < 1 || p < 1 || p > 8) return -fail(WPM_EINVAL, "unsupported (n, p)");
    if (n + p > (1 << p) - 1) return -fail(WPM_EINVAL, "no injective dual matrix: m exceeds 2^p - 1");
    std::vector<uint32_t> pool;  // the non-unit nonzero vectors (rows of M)
    for (uint32_t v = 1; v < (1u << p); ++v)
        if (v & (v - 1)) pool.push_back(v);
    if (n > (int)pool.size()) return -fail(WPM_EINVAL, "no injective dual matrix: m exceeds 2^p - 1");
    const OrbitTables& T = orbit_tables(p);
    const int W = T.words, chunks = ((1 << p) + 7) / 8;
    std::vector<uint64_t> reps;  // W words per representative
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::vector<uint64_t> cur(W), img(W), best(W);
    const int P = (int)pool.size();
    if (W == 1 && !T.byte_img.empty()) {  // p <= 5: one-word masks, straight-line minimum
        const size_t Q = T.img.size();
        const uint64_t* tab = T.byte_img.data();
        // p <= 4: a row set is a 16-bit mask; every image of a processed set
        // is marked, so each orbit's p! images are computed once (35 orbits x
        // 24 images at n = 5 instead of 462 subsets x 24)
        std::vector<uint64_t> seen(p <= 4 ? 1024 : 0, 0ull);
        for (;;) {
            uint64_t c = 0;
            for (int i = 0; i < n; ++i) c |= 1ull << pool[idx[i]];
            if (seen.empty() || !((seen[c >> 6] >> (c & 63)) & 1ull)) {
                uint64_t bm = 0;
                for (size_t q = 0; q < Q; ++q) {
                    uint64_t im = 0;
                    for (int ch = 0; ch < chunks; ++ch) im |= tab[((q * chunks) + ch) * 256 + ((c >> (8 * ch)) & 0xFFu)];
                    if (!seen.empty()) seen[im >> 6] |= 1ull << (im & 63);
                    const uint64_t x = im ^ bm;
                    if (q == 0 || (im & x & (0 - x))) bm = im;
                }
                reps.push_back(bm);
            }
            int pos = n - 1;
            while (pos >= 0 && idx[pos] == P - (n - pos)) --pos;
            if (pos < 0) break;
            ++idx[pos];
            for (int i = pos + 1; i < n; ++i) idx[i] = idx[i - 1] + 1;
        }
    } else
    for (;;) {
        std::fill(cur.begin(), cur.end(), 0ull);
        for (int i = 0; i < n; ++i) cur[pool[idx[i]] >> 6] |= 1ull << (pool[idx[i]] & 63);
        for (size_t q = 0; q < T.img.size(); ++q) {
            std::fill(img.begin(), img.end(), 0ull);
            if (T.byte_img.empty()) {
                for (int i = 0; i < n; ++i) {
                    const uint32_t y = T.img[q][pool[idx[i]]];
                    img[y >> 6] |= 1ull << (y & 63);
                }
            } else {
                for (int c = 0; c < chunks; ++c) {
                    const unsigned x = (unsigned)((cur[(c * 8) >> 6] >> ((c * 8) & 63)) & 0xFFu);
                    if (!x) continue;
                    const uint64_t* src = &T.byte_img[(((q * chunks) + c) * 256 + x) * W];
                    for (int w = 0; w < W; ++w) img[w] |= src[w];
                }
            }
            if (q == 0 || set_less(img.data(), best.data(), W)) best = img;
        }
        reps.insert(reps.end(), best.begin(), best.end());
        int pos = n - 1;
        while (pos >= 0 && idx[pos] == P - (n - pos)) --pos;
        if (pos < 0) break;
        ++idx[pos];
        for (int i = pos + 1; i < n; ++i) idx[i] = idx[i - 1] + 1;
    }
    // sort + unique the representatives (std::set order, :268)
    const size_t R = reps.size() / W;
    std::vector<size_t> order(R);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(),
              [&](size_t a, size_t b) { return set_less(&reps[a * W], &reps[b * W], W); });
    const int m = n + p;
    int k = 0;
    for (size_t r = 0; r < R; ++r) {
        const uint64_t* x = &reps[order[r] * W];
        if (r > 0 && std::equal(x, x + W, &reps[order[r - 1] * W])) continue;
        if (k < cap && rows_out) {
            int i = 0;
            for (int w = 0; w < W; ++w)
                for (uint64_t y = x[w]; y; y &= y - 1) rows_out[(size_t)k * m + i++] = (uint32_t)(w * 64 + __builtin_ctzll(y));
            for (int j = 0; j < p; ++j) rows_out[(size_t)k * m + n + j] = 1u << j;
        }
        ++k;
    }
    return k;
}

// charmap_of_dcm (charmap.hpp:155-204): lambda = [I_n | M^t] in standard
// form, else a kernel basis of D^t by elimination.
extern "C" int32_t wpm_charmap_of_dcm(int32_t m, int32_t p, const uint32_t* rows, uint32_t* cols) {
    const int n = m - p;
    if (n < 1 || m > 31) return -fail(WPM_EINVAL, "unsupported dual matrix shape");
    for (int i = 0; i < m; ++i) cols[i] = 0;
    bool standard = true;
    for (int i = 0; i < p; ++i) standard &= rows[m - p + i] == (1u << i);
    if (standard) {
        for (int i = 0; i < n; ++i) cols[i] = 1u << i;
        for (int j = 0; j < p; ++j)
            for (int i = 0; i < n; ++i)
                if ((rows[i] >> j) & 1u) cols[n + j] |= 1u << i;
        return n;
    }
    std::vector<uint64_t> a(p, 0);
    for (int j = 0; j < p; ++j)
        for (int v = 0; v < m; ++v)
            if ((rows[v] >> j) & 1u) a[j] |= 1ull << v;
    std::vector<int> piv;
    int rank = 0;
    for (int c = 0; c < m && rank < p; ++c) {
        int r0 = -1;
        for (int r = rank; r < p; ++r)
            if ((a[r] >> c) & 1u) { r0 = r; break; }
        if (r0 < 0) continue;
        std::swap(a[rank], a[r0]);
        for (int r = 0; r < p; ++r)
            if (r != rank && ((a[r] >> c) & 1u)) a[r] ^= a[rank];
        piv.push_back(c);
        ++rank;
    }
    if (rank != p) return -fail(WPM_EINVAL, "dual matrix is rank deficient");
    int row = 0;
    for (int fc = 0; fc < m; ++fc) {
        if (std::find(piv.begin(), piv.end(), fc) != piv.end()) continue;
        cols[fc] |= 1u << row;
        for (int r = 0; r < rank; ++r)
            if ((a[r] >> fc) & 1u) cols[piv[r]] |= 1u << row;
        ++row;
    }
    return n;
}

// ------------------------------------------------------------------ plans

// Per-device context, created once: attributes, and a free list of
// (stream, events) bundles that plans borrow and return.
struct DevCtx {
    bool init = false;
    int major = 0, num_sms = 0;
    std::mutex mu;
    struct Bundle {
        cudaStream_t s;
        cudaEvent_t ev[5];
    };
    std::vector<Bundle> free_bundles;
};
DevCtx g_dev[64];
std::mutex g_dev_mu;

static int plan_init(wpm_plan* P, int device) {
    static int count = -1;
    if (count < 0 && cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
    if (count == 0) return fail(WPM_EINTERNAL, "no CUDA device: the B200 path has no CPU fallback");
    if (device < 0 || device >= count || device >= 64) return fail(WPM_EINVAL, "device ordinal out of range");
    P->device = device;
    CU(cudaSetDevice(device));
    // a non-sticky error left by an earlier call must not fail this plan's
    // first launch check (a sticky fault still fails every call)
    const cudaError_t stale = cudaGetLastError();
    if (stale != cudaSuccess && std::getenv("WPM_TRACE"))
        std::fprintf(stderr, "[wpm] cleared a stale CUDA error: %s\n", cudaGetErrorString(stale));
    DevCtx& dc = g_dev[device];
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        if (!dc.init) {
            CU(cudaDeviceGetAttribute(&dc.major, cudaDevAttrComputeCapabilityMajor, device));
            CU(cudaDeviceGetAttribute(&dc.num_sms, cudaDevAttrMultiProcessorCount, device));
            init_pool(device);
            dc.init = true;
        }
    }
    if (dc.major < 10) return fail(WPM_EINTERNAL, "device is not sm_100 (Blackwell); this build targets sm_100a");
    P->num_sms = dc.num_sms;
    {
        std::lock_guard<std::mutex> lk(dc.mu);
        if (!dc.free_bundles.empty()) {
            const auto b = dc.free_bundles.back();
            dc.free_bundles.pop_back();
            P->stream = b.s;
            for (int i = 0; i < 5; ++i) P->ev[i] = b.ev[i];
        }
    }
    if (!P->stream) {
        CU(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking));
        for (auto& e : P->ev) CU(cudaEventCreate(&e));
    }
    g_alloc_stream = P->stream;
    return stage_init(P);
}

static int resolve_cap(int64_t facet_cap, int n, int M) {
    (void)M;
    if (facet_cap == WPM_CAP_UBT) return (int)cyclic_bound(n);
    if (facet_cap < 0) return INT32_MAX;
    return (int)std::min<int64_t>(facet_cap, INT32_MAX);
}

// lay out tables once M is known per map (facets already on device at
// d_facets with per-map offsets `foff`), run kernel 2, finish the plan.
static int plan_build_tables(wpm_plan* P, const std::vector<uint32_t>& foff) {
    const int K = P->num_maps;
    P->desc.assign(K, MapDesc{});
    size_t fr_tot = 0, r_tot = 0;
    P->maxM = 0;
    for (int i = 0; i < K; ++i) {
        const int M = P->M[i];
        if (M <= 0) return fail(WPM_EINVAL, "empty facet universe (incidence of an empty facet set)");
        if (M > WPM_MAX_FACETS) return fail(WPM_EINVAL, "universe larger than WPM_MAX_FACETS");
        MapDesc& d = P->desc[i];
        d.M = M;
        d.n = P->n;
        d.m = P->m;
        d.cap = P->cap[i];
        d.facet_off = foff[i];
        d.fr_stride = P->n;
        d.rp_stride = std::min(WPM_MAX_PARENTS, P->m - P->n + 1);
        d.fr_off = (uint32_t)(fr_tot * P->n);
        const size_t rcap = std::min<size_t>(binom_small(P->m, P->n - 1), (size_t)M * P->n);
        d.ridge_off = (uint32_t)r_tot;
        d.rp_off = (uint32_t)(r_tot * d.rp_stride);
        d.np_off = (uint32_t)r_tot;
        fr_tot += (size_t)M;
        r_tot += rcap;
        P->maxM = std::max(P->maxM, M);
    }
    P->fr_words = (int)(fr_tot * P->n);
    P->rp_words = (int)(r_tot * std::min(WPM_MAX_PARENTS, P->m - P->n + 1));
    // fr / rp padded to 16-byte multiples (TS layouts copy them with 16-byte vectors)
    if (P->d_maps.ensure(K) || P->d_ridges.ensure(r_tot) || P->d_fr.ensure(fr_tot * P->n + 8) ||
        P->d_rp.ensure(r_tot * WPM_MAX_PARENTS + 8) || P->d_npar.ensure(r_tot) || P->d_tmpi.ensure(K + 1))
        return fail(WPM_EINTERNAL, "device allocation failed (tables)");
    CU(h2d_async(P, P->d_maps.p, P->desc.data(), K * sizeof(MapDesc)));
    CU(cudaMemsetAsync(P->d_tmpi.p, 0, (K + 1) * sizeof(int32_t), P->stream));
    if (launch_k2_incidence(K, P->d_maps.p, P->m, P->n, P->d_facets.p, P->d_ridges.p, P->d_fr.p, P->d_rp.p,
                            P->d_npar.p, P->d_tmpi.p, P->d_tmpi.p + K, P->stream))
        return fail(WPM_EINTERNAL, std::string("kernel 2 launch: ") + cudaGetErrorString(cudaGetLastError()));
    P->h2d += 2LL * K * (long long)sizeof(MapDesc);
    CU(cudaMemcpyAsync(mail(P, kMailMaps), P->d_tmpi.p, (K + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, P->stream));
    P->d2h += (long long)(K + 1) * 4;
    CU(cudaStreamSynchronize(P->stream));
    stage_reset(P);
    std::vector<int32_t> hN(K + 1);
    std::memcpy(hN.data(), mail(P, kMailMaps), (K + 1) * sizeof(int32_t));
    if (hN[K]) return fail(WPM_EINVAL, "a ridge has more than WPM_MAX_PARENTS candidate facets");
    P->N.assign(hN.begin(), hN.begin() + K);
    P->maxN = 0;
    P->maxDepth = 0;
    for (int i = 0; i < K; ++i) {
        P->desc[i].N = P->N[i];
        if (P->N[i] > WPM_MAX_RIDGES) return fail(WPM_EINVAL, "more than WPM_MAX_RIDGES ridges");
        P->maxN = std::max(P->maxN, P->N[i]);
        P->maxDepth = std::max(P->maxDepth, std::min(P->cap[i], P->M[i]) + 1);
    }
    CU(h2d_async(P, P->d_maps.p, P->desc.data(), K * sizeof(MapDesc)));
    P->signature = std::to_string(P->m) + "/" + std::to_string(P->n) + "/" + std::to_string(P->facet_cap) + "/" +
                   std::to_string(P->has_pins ? 1 : 0);
    for (int i = 0; i < K; ++i) P->signature += ":" + std::to_string(P->M[i]) + "," + std::to_string(P->N[i]);
    P->mw = (P->maxM + 31) / 32;
    P->w32 = 2 * ((P->maxM + 63) / 64);  // C-ABI rows: whole 64-bit words
    P->rw = rec_words(P->mw);             // emitted records: the mw words the bitsets use + the map id
    P->recw = 4 + 2 * P->mw;
    return WPM_OK;  // the desc upload is staged (pinned); the run orders after it on the stream
}

static int create_from_cols(int32_t n, int32_t m, int32_t K, const uint32_t* cols, int64_t facet_cap,
                            int32_t device, wpm_plan_t** out) {
    *out = nullptr;
    if (n < 1 || m < n || m > WPM_MAX_M) return fail(WPM_EINVAL, "unsupported (m, n): need 1 <= n <= m <= 16");
    if (K < 1) return fail(WPM_EINVAL, "no characteristic maps");
    Trace tr;
    auto* P = new wpm_plan();
    int rc = plan_init(P, device);
    if (rc) { delete P; return rc; }
    tr.mark("plan init (stream, events)");
    P->n = n;
    P->m = m;
    P->num_maps = K;
    P->facet_cap = facet_cap;
    const int stride = (int)binom_small(m, n);
    DevBuf<uint32_t> d_cols;
    if (d_cols.ensure((size_t)K * m) || P->d_facets.ensure((size_t)K * stride) || P->d_tmpi.ensure(K + 1)) {
        delete P;
        return fail(WPM_EINTERNAL, "device allocation failed (universes)");
    }
    if (h2d_async(P, d_cols.p, cols, (size_t)K * m * sizeof(uint32_t)) != cudaSuccess) {
        delete P;
        return fail(WPM_EINTERNAL, "H2D of the characteristic maps failed");
    }
    P->h2d += (long long)K * m * 4;
    int k1rc;
    {
        CallTimer ct_("launch_k1_universe", __LINE__);
        k1rc = launch_k1_universe(n, m, K, d_cols.p, P->d_facets.p, stride, P->d_tmpi.p, P->stream);
    }
    if (k1rc) {
        delete P;
        return fail(WPM_EINTERNAL, "kernel 1 launch failed");
    }
    P->M.assign(K, 0);
    cudaMemcpyAsync(mail(P, kMailMaps), P->d_tmpi.p, K * sizeof(int32_t), cudaMemcpyDeviceToHost, P->stream);
    P->d2h += (long long)K * 4;
    cudaError_t s1;
    {
        CallTimer ct_("sync after kernel 1", __LINE__);
        s1 = cudaStreamSynchronize(P->stream);
    }
    if (s1 != cudaSuccess) {
        delete P;
        return fail(WPM_EINTERNAL, std::string("kernel 1: ") + cudaGetErrorString(cudaGetLastError()));
    }
    stage_reset(P);
    std::memcpy(P->M.data(), mail(P, kMailMaps), K * sizeof(int32_t));
    for (int i = 0; i < K; ++i)
        if (P->M[i] < 0) {
            delete P;
            return fail(WPM_EINVAL, "matrix is rank deficient");
        }
    tr.mark("kernel 1 + sync");
    P->cap.resize(K);
    std::vector<uint32_t> foff(K);
    for (int i = 0; i < K; ++i) {
        P->cap[i] = resolve_cap(facet_cap, n, P->M[i]);
        foff[i] = (uint32_t)((size_t)i * stride);
    }
    rc = plan_build_tables(P, foff);
    tr.mark("kernel 2 + sync");
    if (rc) { delete P; return rc; }
    {
        std::vector<uint32_t> c(cols, cols + (size_t)K * m);
        P->recreate = [n, m, K, c, facet_cap](int dev, wpm_plan_t** o) {
            return create_from_cols(n, m, K, c.data(), facet_cap, dev, o);
        };
    }
    *out = P;
    return WPM_OK;
}

extern "C" int wpm_plan_create_charmaps(int32_t n, int32_t m, int32_t num_maps, const uint32_t* cols,
                                        int64_t facet_cap, int32_t device, wpm_plan_t** out) {
    return create_from_cols(n, m, num_maps, cols, facet_cap, device, out);
}

extern "C" int wpm_plan_create_orbits(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_plan_t** out) {
    *out = nullptr;
    Trace tr;
    const int m = n + p;
    // at most one orbit per n-subset of the 2^p - 1 - p non-unit rows
    const int pool = p >= 1 && p <= 8 ? (1 << p) - 1 - p : 0;
    uint64_t choose = n >= 0 && n <= pool ? 1 : 4096;  // C(pool, n), saturated: C(pool - n + i, i) grows with i
    for (int i = 1; i <= n && n <= pool && choose <= 4096; ++i) choose = choose * (uint64_t)(pool - n + i) / (uint64_t)i;
    const int32_t bound = (int32_t)std::min<uint64_t>(4096, std::max<uint64_t>(choose, 1));
    std::vector<uint32_t> rows((size_t)std::max(bound, 1) * std::max(m, 1));
    const int32_t K = wpm_idcm_orbits(n, p, rows.data(), bound);
    if (K < 0) return -K;
    tr.mark("orbits (host)");
    if (K > bound) return fail(WPM_EINVAL, "too many orbits");
    std::vector<uint32_t> cols((size_t)K * m);
    for (int i = 0; i < K; ++i)
        if (wpm_charmap_of_dcm(m, p, rows.data() + (size_t)i * m, cols.data() + (size_t)i * m) < 0)
            return WPM_EINVAL;
    tr.mark("orbits + charmaps (host)");
    return create_from_cols(n, m, K, cols.data(), facet_cap, device, out);
}

// Explicit universes (SearchJob.facets), in ANY order: incidence_matrix
// indexes ridges by hash (incidence.hpp:34-55) and enumerate_wpm rebuilds and
// sorts its output (search.hpp:247-257), so the reference accepts an
// unsorted universe.  Here each universe is sorted into the canonical order
// (the plan's facet j = the j-th smallest mask; results and wpm_plan_universe
// use that order) and required / forbidden indices (into the caller's order)
// are remapped.  Duplicate facets are rejected like PureComplex::validate
// (complex.hpp:50-51).
extern "C" int wpm_plan_create_universes(int32_t m, int32_t n, int32_t K, const int32_t* counts,
                                         const uint64_t* facets, int64_t facet_cap, const int32_t* required,
                                         int32_t num_required, const int32_t* forbidden, int32_t num_forbidden,
                                         int32_t device, wpm_plan_t** out) {
    *out = nullptr;
    if (n < 1 || m < n || m > WPM_MAX_M) return fail(WPM_EINVAL, "unsupported (m, n): need 1 <= n <= m <= 16");
    if (K < 1) return fail(WPM_EINVAL, "no universes");
    if ((num_required || num_forbidden) && K != 1) return fail(WPM_EINVAL, "pins need a single universe");
    // validate: pure, labels in 1..m (PureComplex::validate, complex.hpp:37-55); sort
    std::vector<uint32_t> h;
    std::vector<uint32_t> foff(K);
    std::vector<int32_t> rank_of;  // caller index -> canonical index (universe 0, for the pins)
    size_t off = 0;
    const uint64_t full = ((1ull << m) - 1ull) << 1;
    for (int i = 0; i < K; ++i) {
        foff[i] = (uint32_t)off;
        if (counts[i] <= 0) return fail(WPM_EINVAL, "incidence of an empty facet set");
        std::vector<std::pair<uint64_t, int32_t>> u((size_t)counts[i]);
        for (int j = 0; j < counts[i]; ++j) {
            const uint64_t f = facets[off + j];
            if (f & ~full) return fail(WPM_EINVAL, "facet uses a label outside 1..m");
            if (__builtin_popcountll(f) != n) return fail(WPM_EINVAL, "facet size differs from n (purity)");
            u[(size_t)j] = {f, j};
        }
        std::sort(u.begin(), u.end());
        for (int j = 1; j < counts[i]; ++j)
            if (u[(size_t)j].first == u[(size_t)j - 1].first) return fail(WPM_EINVAL, "duplicate facet in the universe");
        if (i == 0) {
            rank_of.assign((size_t)counts[0], 0);
            for (int j = 0; j < counts[0]; ++j) rank_of[(size_t)u[(size_t)j].second] = j;
        }
        for (const auto& x : u) h.push_back((uint32_t)x.first);
        off += counts[i];
    }
    auto* P = new wpm_plan();
    int rc = plan_init(P, device);
    if (rc) { delete P; return rc; }
    P->n = n;
    P->m = m;
    P->num_maps = K;
    P->facet_cap = facet_cap;
    P->M.assign(counts, counts + K);
    P->cap.resize(K);
    for (int i = 0; i < K; ++i) P->cap[i] = resolve_cap(facet_cap, n, P->M[i]);
    if (P->d_facets.ensure(h.size())) { delete P; return fail(WPM_EINTERNAL, "device allocation failed"); }
    h2d_async(P, P->d_facets.p, h.data(), h.size() * sizeof(uint32_t));
    P->h2d += (long long)h.size() * 4;
    rc = plan_build_tables(P, foff);
    if (rc) { delete P; return rc; }
    if (num_required || num_forbidden) {
        const int M = P->M[0];
        P->pin_in.assign(P->mw, 0);
        P->pin_out.assign(P->mw, 0);
        for (int i = 0; i < num_required; ++i) {
            if (required[i] < 0 || required[i] >= M) { delete P; return fail(WPM_EINVAL, "required facet index out of range"); }
            const int f = rank_of[(size_t)required[i]];
            P->pin_in[f >> 5] |= 1u << (f & 31);
        }
        for (int i = 0; i < num_forbidden; ++i) {
            if (forbidden[i] < 0 || forbidden[i] >= M) { delete P; return fail(WPM_EINVAL, "forbidden facet index out of range"); }
            const int f = rank_of[(size_t)forbidden[i]];
            P->pin_out[f >> 5] |= 1u << (f & 31);
        }
        P->has_pins = true;
    }
    {
        std::vector<int32_t> c(counts, counts + K);
        std::vector<uint64_t> fa(facets, facets + off);
        std::vector<int32_t> rq(required, required + num_required), fb(forbidden, forbidden + num_forbidden);
        P->recreate = [m, n, K, c, fa, facet_cap, rq, fb](int dev, wpm_plan_t** o) {
            return wpm_plan_create_universes(m, n, K, c.data(), fa.data(), facet_cap, rq.data(), (int32_t)rq.size(),
                                             fb.data(), (int32_t)fb.size(), dev, o);
        };
    }
    *out = P;
    return WPM_OK;
}

extern "C" int wpm_plan_num_maps(const wpm_plan_t* P) { return P ? P->num_maps : 0; }

extern "C" int32_t wpm_plan_universe(wpm_plan_t* P, int32_t map, uint64_t* out, int32_t cap) {
    if (!P || map < 0 || map >= P->num_maps) return -fail(WPM_EINVAL, "bad map index");
    if (P->h_facets.empty()) {  // every map's universe in one copy, kept on the host
        cudaSetDevice(P->device);
        const MapDesc& last = P->desc[P->num_maps - 1];
        P->h_facets.resize((size_t)last.facet_off + (size_t)last.M);
        if (cudaMemcpy(P->h_facets.data(), P->d_facets.p, P->h_facets.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
            P->h_facets.clear();
            return -fail(WPM_EINTERNAL, "copy failed");
        }
        P->d2h += (long long)P->h_facets.size() * 4;
    }
    const int M = P->M[map];
    const uint32_t* h = P->h_facets.data() + P->desc[map].facet_off;
    for (int j = 0; j < M && j < cap; ++j) out[j] = h[j];
    return M;
}

extern "C" int32_t wpm_plan_incidence(wpm_plan_t* P, int32_t map, uint64_t* ridges_out, int32_t ridges_cap,
                                      int32_t* cols_out, int32_t* par_out) {
    if (!P || map < 0 || map >= P->num_maps) return -fail(WPM_EINVAL, "bad map index");
    cudaSetDevice(P->device);
    const MapDesc& d = P->desc[map];
    const int M = d.M, N = d.N, n = d.n;
    if (ridges_cap < N) return N;
    std::vector<uint32_t> r(N);
    const int RS = d.rp_stride;
    std::vector<uint16_t> fr((size_t)M * n), rp((size_t)N * RS);
    if (cudaMemcpy(r.data(), P->d_ridges.p + d.ridge_off, N * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(fr.data(), P->d_fr.p + d.fr_off, fr.size() * 2, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(rp.data(), P->d_rp.p + d.rp_off, rp.size() * 2, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -fail(WPM_EINTERNAL, "copy failed");
    for (int i = 0; i < N; ++i) ridges_out[i] = r[i];
    if (cols_out)
        for (int j = 0; j < M; ++j)
            for (int k = 0; k < n; ++k) cols_out[j * n + k] = fr[(size_t)j * n + k];
    if (par_out)
        for (int i = 0; i < N; ++i)
            for (int q = 0; q < WPM_MAX_PARENTS; ++q) {
                const uint16_t g = q < RS ? rp[(size_t)i * RS + q] : NONE16;
                par_out[i * WPM_MAX_PARENTS + q] = g == NONE16 ? -1 : (int32_t)g;
            }
    return N;
}

static int plan_sort(wpm_plan* P);
static int plan_sort_launch(wpm_plan* P, bool device_count);
static int plan_sort_collect(wpm_plan* P);

// ---- one kernel-3 launch on the plan's stream: seed (root tasks or task
// records), optional frontier output (split mode) or shared-frontier claims
struct K3Launch {
    const int32_t* d_tm = nullptr;  // root tasks (map, f, kind), ntasks of them
    const int32_t* d_tf = nullptr;
    const int32_t* d_tk = nullptr;
    int ntasks = 0;
    const uint32_t* d_recs = nullptr;  // or task records (a frontier)
    long long nrecs = 0;
    int cutoff = 0;                    // split mode: frames at depth >= cutoff go to d_front_out
    uint32_t* d_front_out = nullptr;
    unsigned long long front_cap = 0;
    const uint32_t* claim_recs = nullptr;  // claim mode
    long long claim_count = 0;
    unsigned long long* claim_ctr = nullptr;
    bool full_depth = false;
    bool progress = false;             // root-task progress accounting (the main phase)
};

static int k3_launch(wpm_plan* P, const K3Launch& L, int frame_cap) {
    const long long nseed = L.d_recs ? L.nrecs : L.ntasks;
    const long long nroots = L.claim_recs ? L.claim_count : nseed;
    const bool prog = L.progress && P->progress_fn;
    if (prog && P->d_root_pend.ensure((size_t)std::max<long long>(nroots, 1)))
        return fail(WPM_EINTERNAL, "device allocation failed (progress)");
    SearchParams sp{};
    sp.num_maps = P->num_maps;
    sp.max_M = P->maxM;
    sp.max_N = P->maxN;
    sp.max_n = P->n;
    sp.max_depth = L.full_depth ? P->maxDepth : frame_cap;
    sp.maps = P->d_maps.p;
    sp.fr = P->d_fr.p;
    sp.rp = P->d_rp.p;
    sp.fr_words = P->fr_words;
    sp.rp_words = P->rp_words;
    sp.npar = P->d_npar.p;
    sp.recw = P->recw;
    sp.mw = P->mw;
    sp.out_keys = P->d_out_keys.p;
    sp.out_ctl = P->d_out_ctl.p;
    sp.per_map = P->d_per_map.p;
    sp.out_cap = P->out_cap;
    sp.rw = P->rw;
    sp.node_budget = P->node_budget;
    sp.cutoff = L.cutoff;
    sp.front_out = L.d_front_out;
    sp.front_ctl = P->d_front_ctl.p;
    sp.front_cap = L.front_cap;
    sp.claim_recs = L.claim_recs;
    sp.claim_count = L.claim_count;
    sp.claim_ctr = L.claim_ctr;
    // the queue: one ring, or one per map when the kernel keeps a single map's
    // tables per CTA (k3_map_queues); the root tasks' map-major order gives
    // each map its seed slots
    int ma_tab = 0;
    for (const MapDesc& d : P->desc)
        ma_tab = std::max(ma_tab, ((2 * d.M * d.fr_stride + 15) & ~15) + ((2 * d.N * d.rp_stride + 15) & ~15));
    sp.ma_tab_bytes = ma_tab;
    sp.map_first = P->d_map_first.p;
    sp.map_queues = !L.d_recs && L.ntasks > 0 && !P->has_pins && k3_map_queues(sp);
    const int nq = sp.map_queues ? P->num_maps : 1;
    long long qcap = sp.map_queues ? 1 << 14 : 1 << 16;  // > pending: 2 x warps + seeds
    while (qcap < 2 * (sp.map_queues ? P->maxM : nseed)) qcap <<= 1;
    if (P->d_qrec.ensure((size_t)nq * qcap * P->recw) || P->d_qready.ensure((size_t)nq * qcap) ||
        P->d_qctl.ensure(8 * (size_t)(nq + 1)))
        return fail(WPM_EINTERNAL, "device allocation failed (queue)");
    P->qcap = (int)qcap;
    sp.qrec = P->d_qrec.p;
    sp.qready = P->d_qready.p;
    sp.qctl = P->d_qctl.p;
    sp.qcap = P->qcap;
    {
        unsigned long long ctl[3] = {(unsigned long long)nseed << 32, 0, (unsigned long long)nseed};
        if (sp.map_queues) ctl[0] = ctl[2] = 0;  // plan-wide words only
        CU(h2d_async(P, P->d_qctl.p, ctl, sizeof(ctl)));  // [3], [4] add up
        P->h2d += (long long)sizeof(ctl);
        if (sp.map_queues) {
            const std::vector<int32_t>& first = P->h_map_first;
            std::vector<unsigned long long> qc(8 * (size_t)nq, 0);
            for (int q = 0; q < nq; ++q) {
                const unsigned long long c = (unsigned long long)(first[q + 1] - first[q]);
                qc[8 * q] = c << 32;
                qc[8 * q + 2] = c;
            }
            CU(h2d_async(P, P->d_qctl.p + 8, qc.data(), qc.size() * 8));
            P->h2d += (long long)qc.size() * 8;
        }
        CU(cudaMemsetAsync(P->d_qready.p, 0, (size_t)nq * qcap * 8, P->stream));
    }
    if (prog) {
        sp.root_pend = P->d_root_pend.p;
        sp.roots_done = P->d_acc.p;
        sp.progress_host = P->progress_dev;
        CU(cudaMemsetAsync(P->d_acc.p, 0, 8, P->stream));
        *(volatile unsigned long long*)P->progress_host = 0;
        if (L.claim_recs && launch_fill_u32(sp.root_pend, 1u, nroots, P->stream))
            return fail(WPM_EINTERNAL, "progress init failed");
    }
    if (L.d_recs) {
        if (launch_seed_records(sp, L.d_recs, L.nrecs, P->stream)) return fail(WPM_EINTERNAL, "seed launch failed");
    } else if (launch_seed_tasks(sp, L.ntasks, L.d_tm, L.d_tf, L.d_tk, P->has_pins ? P->d_pin_in.p : nullptr,
                                 P->has_pins ? P->d_pin_out.p : nullptr, P->stream)) {
        return fail(WPM_EINTERNAL, "seed launch failed");
    }
    const int est_warps = P->num_sms * 16;
    sp.hungry = std::max(64, est_warps / 2);
    if (sp.map_queues) sp.hungry = 128;  // per map queue (measured 8..128: within 1 %, 128 best at n = 7, 8)
    // first poll sleep of a waiting warp: 1 us (32 ns before this round) --
    // idle warps' polls took issue slots from the busy ones: n = 4 -5 %,
    // n = 5 -2..-4 %, n >= 6 within noise (profiles/r02d_ab_backoff*.jsonl)
    sp.backoff_min = 1024;
    sp.backoff_max = 8192;
    if (const char* e = std::getenv("WPM_BACKOFF_MIN")) sp.backoff_min = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("WPM_HUNGRY")) sp.hungry = std::atoi(e);
    if (const char* e = std::getenv("WPM_BACKOFF_MAX")) sp.backoff_max = std::max(32, std::atoi(e));
    // donation checks: every 16 nodes for small tables (cheap task
    // loads; n <= 6 ramps/tails faster), 32 otherwise (n = 11 loads cost
    // O(N) per donated task) -- measured sweep in DESIGN.md
    sp.check_every = P->maxN <= 256 ? 16 : 32;
    if (const char* e = std::getenv("WPM_CHECK_EVERY")) sp.check_every = std::max(1, std::atoi(e));
    sp.first_check = sp.check_every;
    // > 512 warps waiting: busy warps look at the queue every 8 nodes (a
    // ramp, a tail, a GPU holding few frontier records) -- n = 5 -1.8 %,
    // n = 8 -1.2 %, n = 11 within noise (profiles/r02d_ab_starve.jsonl)
    sp.starve_at = 512;
    sp.starve_check = std::min(8, sp.check_every);
    if (const char* e = std::getenv("WPM_STARVE_AT")) sp.starve_at = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("WPM_STARVE_CHECK")) sp.starve_check = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("WPM_FIRST_CHECK")) sp.first_check = std::max(1, std::min(sp.check_every, std::atoi(e)));
    sp.donate_max = 1;
    if (const char* e = std::getenv("WPM_DONATE_MAX")) sp.donate_max = std::max(1, std::atoi(e));
    // claims: while fewer tasks than warps are pending on this GPU, waiting
    // warps pull records (measured at 1 GPU: a quarter of the warps starved
    // the claim phase 2-5x; >= the warp count matches the seeded run)
    sp.claim_low = P->num_sms * 40;
    // Several GPUs: at most a fair share (frontier / GPUs) pending per GPU
    // while it claims.  With ~5 k records and ~4 k warps per GPU every
    // waiting warp would otherwise pull a record at launch, and the GPU
    // launched first would take up to its warp count of them -- a
    // first-come partition instead of a balanced one.  A GPU past its share
    // claims again once its pending tasks drop under the share.
    if (L.claim_recs && P->claim_devices > 1)
        sp.claim_low = (int)std::max<long long>(
            2LL * P->num_sms, std::min<long long>(sp.claim_low, (L.claim_count + P->claim_devices - 1) / P->claim_devices));
    if (const char* e = std::getenv("WPM_CLAIM_LOW")) sp.claim_low = std::max(1, std::atoi(e));
    if (L.progress && P->root_stats) {  // nodes per root task / frontier record (the scaling projection)
        if (P->d_root_nodes.ensure((size_t)std::max<long long>(nroots, 1)))
            return fail(WPM_EINTERNAL, "device allocation failed (root stats)");
        CU(cudaMemsetAsync(P->d_root_nodes.p, 0, (size_t)std::max<long long>(nroots, 1) * 8, P->stream));
        sp.root_nodes = P->d_root_nodes.p;
        P->root_count = nroots;
    }
    int k3ok = 1;
    {
        CallTimer ct_("launch_k3_search", __LINE__);
        if (nseed > 0 || L.claim_recs) k3ok = launch_k3_search(sp, P->num_sms, P->stream, &P->warps);
    }
    if (!k3ok)
        return fail(WPM_EINTERNAL, std::string("kernel 3 launch: ") + cudaGetErrorString(cudaGetLastError()));
    return WPM_OK;
}

// the root tasks of the plan (map, minimum facet f) in queue order, or one
// ENTRY task for a pinned universe; a static shard keeps every count-th
static void root_tasks(const wpm_plan* P, int shard_index, int shard_count, std::vector<int32_t>* tm,
                       std::vector<int32_t>* tf, std::vector<int32_t>* tk) {
    tm->clear();
    tf->clear();
    tk->clear();
    if (P->has_pins) {
        tm->push_back(0);
        tf->push_back(0);
        tk->push_back(3);
    } else {
        // map-major: at any moment the warps of an SM share few maps, so the
        // per-map tables stay L1 resident; donations balance the load
        for (int i = 0; i < P->num_maps; ++i)
            for (int f = 0; f < P->M[i]; ++f)
                if (P->n + 1 <= P->cap[i]) {
                    tm->push_back(i);
                    tf->push_back(f);
                    tk->push_back(0);
                }
    }
    if (shard_count > 1) {
        size_t k = 0;
        for (size_t t = 0; t < tm->size(); ++t)
            if ((int)(t % shard_count) == shard_index) {
                (*tm)[k] = (*tm)[t];
                (*tf)[k] = (*tf)[t];
                (*tk)[k] = (*tk)[t];
                ++k;
            }
        tm->resize(k);
        tf->resize(k);
        tk->resize(k);
    }
}

// ---- phases of one search (composable: single GPU, split + search, claims)

// allocations, root tasks on the device, output sizing
static int search_prepare(wpm_plan* P, int shard_index, int shard_count) {
    Trace tr;
    const int K = P->num_maps;
    std::vector<int32_t> tm, tf, tk;
    root_tasks(P, shard_index, shard_count, &tm, &tf, &tk);
    const int ntasks = (int)tm.size();
    P->ntasks = ntasks;
    if (P->d_qctl.ensure(8 * (size_t)(K + 1)) || P->d_acc.ensure(4) || P->d_task_map.ensure(ntasks + 1) ||
        P->d_task_f.ensure(ntasks + 1) || P->d_task_kind.ensure(ntasks + 1) || P->d_out_ctl.ensure(4) ||
        P->d_per_map.ensure(K) || P->d_front_ctl.ensure(2))
        return fail(WPM_EINTERNAL, "device allocation failed (queue)");
    if (P->has_pins) {
        if (P->d_pin_in.ensure(P->mw) || P->d_pin_out.ensure(P->mw))
            return fail(WPM_EINTERNAL, "device allocation failed (pins)");
        CU(h2d_async(P, P->d_pin_in.p, P->pin_in.data(), P->mw * 4));
        CU(h2d_async(P, P->d_pin_out.p, P->pin_out.data(), P->mw * 4));
    }
    tr.mark("    prepare: small buffers");
    {  // root tasks are map-major: map q's are [first[q], first[q + 1])
        std::vector<int32_t> first(K + 1, 0);
        for (int t = 0; t < ntasks; ++t) ++first[tm[t] + 1];
        for (int q = 0; q < K; ++q) first[q + 1] += first[q];
        if (P->d_map_first.ensure(K + 1)) return fail(WPM_EINTERNAL, "device allocation failed (queue)");
        P->h_map_first = first;
        CU(h2d_async(P, P->d_map_first.p, P->h_map_first.data(), (K + 1) * 4));
        P->h2d += 4LL * (K + 1);
    }
    if (ntasks) {
        CU(h2d_async(P, P->d_task_map.p, tm.data(), ntasks * 4));
        CU(h2d_async(P, P->d_task_f.p, tf.data(), ntasks * 4));
        CU(h2d_async(P, P->d_task_kind.p, tk.data(), ntasks * 4));
        P->h2d += 12LL * ntasks;
    }
    if (P->out_cap == 0) {
        // first run: 2^21 rows covers every Picard-4 n (the most WPMs of any
        // n is 1.72 M, n = 8; <= 512 MB at the widest rows); a larger result
        // reruns once with the exact count.  (Sizing from free memory asked
        // the pool for GBs per plan, and cudaMemGetInfo cost 0.1 ms per call.)
        P->out_cap = 1ull << 21;
        if (const char* e = std::getenv("WPM_OUT_CAP")) P->out_cap = std::max(1ull, std::strtoull(e, nullptr, 10));
    }
    tr.mark("    prepare: out_cap");
    if (P->front_cap == 0) P->front_cap = 1ull << 16;
    // frame stack sized for the branch depths the search reaches in practice
    // (<= 37 measured up to n = 11); a run that outgrows it is redone with
    // the worst-case layout (fewer warps per SM)
    P->frame_cap = 64;
    if (const char* e = std::getenv("WPM_FRAME_CAP")) P->frame_cap = std::max(1, std::atoi(e));
    if (!P->full_depth) P->full_depth = P->maxDepth <= P->frame_cap;
    return WPM_OK;
}

// start of an attempt: empty outputs and counters, start event
static int search_reset(wpm_plan* P) {
    Trace tr;
    if (P->d_out_keys.ensure(P->out_cap * P->rw)) return fail(WPM_EINTERNAL, "device allocation failed (output)");
    tr.mark("    reset: output buffer");
    CU(cudaMemsetAsync(P->d_out_ctl.p, 0, 32, P->stream));
    CU(cudaMemsetAsync(P->d_acc.p, 0, 32, P->stream));
    CU(cudaMemsetAsync(P->d_qctl.p, 0, 64, P->stream));
    CU(cudaEventRecord(P->ev[0], P->stream));
    P->frontier = 0;
    return WPM_OK;
}

// phase A: a split launch from the root tasks; frames at split_depth become
// frontier records (everything above them is searched here).  Synchronous:
// returns the record count in P->frontier (> front_cap: overflowed)
static int search_split(wpm_plan* P, int split_depth) {
    if (P->d_front.ensure(P->front_cap * P->recw)) return fail(WPM_EINTERNAL, "allocation failed (frontier)");
    CU(cudaMemsetAsync(P->d_front_ctl.p, 0, 16, P->stream));
    K3Launch a;
    a.d_tm = P->d_task_map.p;
    a.d_tf = P->d_task_f.p;
    a.d_tk = P->d_task_kind.p;
    a.ntasks = P->ntasks;
    a.cutoff = split_depth;
    a.d_front_out = P->d_front.p;
    a.front_cap = P->front_cap;
    a.full_depth = P->full_depth;
    int rc = k3_launch(P, a, P->frame_cap);
    if (rc) return rc;
    unsigned long long fc = 0;
    CU(cudaMemcpyAsync(&fc, P->d_front_ctl.p, 8, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaStreamSynchronize(P->stream));
    P->d2h += 8;
    P->frontier = (long long)fc;
    return WPM_OK;
}

// phase B, asynchronous: the root tasks, the frontier records, or (claim)
// the shared frontier
enum MainSrc { SRC_ROOTS, SRC_FRONTIER, SRC_CLAIM };
static int search_main(wpm_plan* P, MainSrc src) {
    K3Launch b;
    b.full_depth = P->full_depth;
    b.progress = true;
    if (src == SRC_CLAIM) {
        b.claim_recs = P->d_front.p;
        b.claim_count = P->claim_count;
        b.claim_ctr = P->claim_ctr;
    } else if (src == SRC_FRONTIER) {
        b.d_recs = P->d_front.p;
        b.nrecs = P->frontier;
    } else {
        b.d_tm = P->d_task_map.p;
        b.d_tf = P->d_task_f.p;
        b.d_tk = P->d_task_kind.p;
        b.ntasks = P->ntasks;
    }
    const int rc = k3_launch(P, b, P->frame_cap);
    if (rc) return rc;
    CU(cudaEventRecord(P->ev[1], P->stream));
    return WPM_OK;
}

// end of an attempt: wait (calling the progress callback meanwhile), read
// counts.  *again = 1: rerun the attempt (frame stack / output / frontier
// outgrew its buffer; the buffers are resized)
static int search_finish(wpm_plan* P, long long progress_total, int* again) {
    *again = 0;
    unsigned long long octl[4], qc[8];
    CU(cudaMemcpyAsync(mail(P, kMailOctl), P->d_out_ctl.p, 32, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaMemcpyAsync(mail(P, kMailQc), P->d_qctl.p, 64, cudaMemcpyDeviceToHost, P->stream));
    if (P->progress_fn) {
        // the reference's progress(done, total) (search.hpp:54, :244): root
        // tasks finished, published by the kernel to host-mapped memory
        unsigned long long seen = 0;
        while (cudaEventQuery(P->ev[1]) == cudaErrorNotReady) {
            const unsigned long long v = *(volatile unsigned long long*)P->progress_host;
            if (v > seen && (long long)v < progress_total) {
                seen = v;
                P->progress_fn((int64_t)v, (int64_t)progress_total, P->progress_user);
            }
            std::this_thread::sleep_for(std::chrono::microseconds(200));
        }
    }
    CU(cudaStreamSynchronize(P->stream));
    stage_reset(P);
    std::memcpy(octl, mail(P, kMailOctl), sizeof(octl));
    std::memcpy(qc, mail(P, kMailQc), sizeof(qc));
    if (P->progress_fn) P->progress_fn((int64_t)progress_total, (int64_t)progress_total, P->progress_user);
    P->d2h += 96;
    P->total = (long long)octl[0];
    P->tasks = (long long)qc[3];  // kernel-3 launches of one attempt add up in qctl[3] / [4]
    P->nodes = (long long)qc[4];
    if (std::getenv("WPM_POLLSTAT"))
        std::fprintf(stderr, "[wpm] poll iterations %llu, waits %llu, wait cycles %llu (%.2f us per wait), tasks %llu, nodes %llu\n",
                     qc[5], qc[6], qc[7], qc[6] ? qc[7] / 1965.0 / qc[6] : 0.0, qc[3], qc[4]);
    if (std::getenv("WPM_PROFILE") && (qc[5] | qc[6] | qc[7])) {
        const double all = (double)(qc[5] + qc[6] + qc[7]);
        std::fprintf(stderr, "[wpm] warp clocks: busy %.1f%%  waiting %.1f%%  final wait %.1f%%  (tasks %llu)\n",
                     100.0 * qc[5] / all, 100.0 * qc[6] / all, 100.0 * qc[7] / all, qc[3]);
    }
    P->truncated = octl[3] != 0;
    if (octl[2]) {  // frame stack overflowed: redo with the full-depth layout
        P->full_depth = true;
        ++P->reruns;
        *again = 1;
        return WPM_OK;
    }
    if (P->truncated) {  // a budgeted stress run: keep what fits, no rerun
        P->total = std::min<long long>(P->total, (long long)P->out_cap);
        return WPM_OK;
    }
    if (octl[0] > P->out_cap) {
        ++P->reruns;
        P->out_cap = octl[0] + octl[0] / 8 + 1024;  // exact count known now: rerun once
        *again = 1;
    }
    return WPM_OK;
}

// single GPU: [split, then the frontier] or the root tasks
static int plan_search_phases(wpm_plan* P, int shard_index, int shard_count) {
    Trace tr;
    int rc = search_prepare(P, shard_index, shard_count);
    if (rc) return rc;
    tr.mark("  run: tasks + queue alloc");
    CU(cudaEventRecord(P->ev[4], P->stream));
    for (int attempt = 0; attempt < 4; ++attempt) {
        if ((rc = search_reset(P))) return rc;
        long long roots = P->ntasks;
        if (P->split_depth > 0) {
            if ((rc = search_split(P, P->split_depth))) return rc;
            if ((unsigned long long)P->frontier > P->front_cap) {  // rerun with the exact size
                P->front_cap = (unsigned long long)P->frontier + (unsigned long long)P->frontier / 4 + 1024;
                ++P->reruns;
                continue;
            }
            roots = P->frontier;
            tr.mark("  run: split");
        }
        if ((rc = search_main(P, P->split_depth > 0 ? SRC_FRONTIER : SRC_ROOTS))) return rc;
        // the sort follows kernel 3 on the stream, reading the row count on
        // the device: one synchronisation per run (a stage that overflowed
        // its buffers is discarded and rerun)
        if (!P->node_budget && (rc = plan_sort_launch(P, true))) return rc;
        tr.mark("  run: k3 + sort launch");
        int again = 0;
        if ((rc = search_finish(P, roots, &again))) return rc;
        tr.mark("  run: k3 + sort sync");
        if (!again) return P->node_budget ? plan_sort(P) : plan_sort_collect(P);
    }
    return fail(WPM_EINTERNAL, "search did not settle in 4 attempts");
}

static int plan_search(wpm_plan* P, int shard_index, int shard_count) {
    return plan_search_phases(P, shard_index, shard_count);
}

// canonical sort of the key rows in d_out_keys (P->total of them), per-map
// counts from the group boundaries; shared by the DFS and the odometer runs
// launch the sort on the plan's stream: rows = P->total, or -- device_count
// -- the count kernel 3 left in out_ctl[0] (capped at out_cap), so the sort
// follows the search without a host round trip
static int plan_sort_launch(wpm_plan* P, bool device_count) {
    Trace tr;
    const int K = P->num_maps;
    const long long rows = device_count ? (long long)P->out_cap : P->total;
    const size_t tb = canon_sort_temp_bytes(std::max<long long>(rows, 1), P->mw);
    if (P->d_temp.ensure(tb) || P->d_sorted_bits.ensure((size_t)rows * P->w32 + 1) || P->d_sorted_map.ensure(rows + 1))
        return fail(WPM_EINTERNAL, "device allocation failed (sort)");
    CU(cudaMemsetAsync(P->d_out_ctl.p + 1, 0, 8, P->stream));
    CU(cudaMemsetAsync(P->d_per_map.p, 0xFF, K * 8, P->stream));  // first row per map, -1 = none
    CU(cudaEventRecord(P->ev[2], P->stream));
    tr.mark("    sort: buffers");
    // grid sized from the rows this workload produced last time (this plan, or
    // an earlier plan of the same maps: one-shot calls), else the capacity
    long long hint = 0;
    if (device_count) {
        std::lock_guard<std::mutex> lk(g_rows_mu);
        auto it = g_rows_seen.find(P->signature);
        if (it != g_rows_seen.end()) hint = it->second + it->second / 8 + 64;
    }
    const char* se = std::getenv("WPM_SORT");
    if (se && std::strcmp(se, "bucket") == 0) {
        // bucketed by (map, three lowest facets), then sorted per bucket
        // (measured slower than the merge sort: DESIGN.md, kernel 4)
        long long tf = 0;
        for (const MapDesc& d : P->desc) tf = std::max<long long>(tf, (long long)d.facet_off + d.M);
        const size_t sw = bucket_sort_scratch_words(rows, tf);
        const bool fresh = P->d_bucket.n < sw || P->bucket_cap != rows || P->bucket_facets != tf;
        if (P->d_bucket.ensure(sw)) return fail(WPM_EINTERNAL, "device allocation failed (sort)");
        if (fresh) {
            CU(cudaMemsetAsync(P->d_bucket.p + bucket_sort_count_offset(rows), 0, (size_t)tf * 64 * 4, P->stream));
            P->bucket_cap = rows;
            P->bucket_facets = tf;
        }
        if (canon_sort_bucketed(P->d_out_keys.p, rows, device_count ? P->d_out_ctl.p : nullptr, P->mw, P->rw, P->w32,
                                P->d_maps.p, K, tf, P->d_sorted_bits.p, P->d_sorted_map.p, (long long*)P->d_per_map.p,
                                P->d_out_ctl.p + 1, P->d_temp.p, P->d_temp.n, P->d_bucket.p, P->d_bucket.n, P->stream,
                                hint)) {
            P->bucket_cap = -1;  // the count block is in an unknown state
            return fail(WPM_EINTERNAL, std::string("canonical sort: ") + cudaGetErrorString(cudaGetLastError()));
        }
    } else if (canon_sort_keys(P->d_out_keys.p, rows, P->mw, P->d_sorted_bits.p, P->d_sorted_map.p, P->d_temp.p,
                               P->d_temp.n, (long long*)P->d_per_map.p, P->d_out_ctl.p + 1, P->stream,
                               device_count ? P->d_out_ctl.p : nullptr, hint, P->w32)) {
        return fail(WPM_EINTERNAL, std::string("canonical sort: ") + cudaGetErrorString(cudaGetLastError()));
    }
    CU(cudaEventRecord(P->ev[3], P->stream));
    tr.mark("    sort: launch");
    // results of the sort, read back with the next synchronisation
    CU(cudaMemcpyAsync(mail(P, kMailDups), P->d_out_ctl.p + 1, 8, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaMemcpyAsync(mail(P, kMailMaps), P->d_per_map.p, K * 8, cudaMemcpyDeviceToHost, P->stream));
    P->d2h += 8 + 8LL * K;
    return WPM_OK;
}

// after the stream synchronised: duplicates, per-map counts, timings
static int plan_sort_collect(wpm_plan* P) {
    const int K = P->num_maps;
    {
        std::lock_guard<std::mutex> lk(g_rows_mu);
        g_rows_seen[P->signature] = P->total;
    }
    std::memcpy(&P->h_dups, mail(P, kMailDups), 8);
    P->h_first.resize(K);
    std::memcpy(P->h_first.data(), mail(P, kMailMaps), K * 8);
    P->dups = (long long)P->h_dups;
    // per-map counts from the group boundaries of the sorted map ids
    P->per_map.assign(K, 0);
    {
        long long next = P->total;
        for (int i = K - 1; i >= 0; --i)
            if (P->h_first[i] >= 0) {
                P->per_map[i] = (unsigned long long)(next - P->h_first[i]);
                next = P->h_first[i];
            }
    }
    CU(cudaEventElapsedTime(&P->ms_search, P->ev[0], P->ev[1]));
    CU(cudaEventElapsedTime(&P->ms_sort, P->ev[2], P->ev[3]));
    CU(cudaEventElapsedTime(&P->ms_total, P->ev[4], P->ev[3]));
    return WPM_OK;
}

static int plan_sort(wpm_plan* P) {
    Trace tr;
    int rc = plan_sort_launch(P, false);
    if (rc) return rc;
    tr.mark("  sort: alloc + launch");
    CU(cudaStreamSynchronize(P->stream));
    tr.mark("  sort: sync");
    return plan_sort_collect(P);
}

static int plan_run_multi(wpm_plan* P);

extern "C" int wpm_plan_run(wpm_plan_t* P, int32_t shard_index, int32_t shard_count, int64_t* total_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (shard_count < 1) shard_count = 1;
    if (shard_index < 0 || shard_index >= shard_count) return fail(WPM_EINVAL, "bad shard index");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    P->ran = false;
    P->line7 = P->line13 = P->line15 = -1;
    const int rc = P->peers.empty() ? plan_search(P, shard_index, shard_count) : plan_run_multi(P);
    if (rc) return rc;
    P->ran = true;
    if (total_out) *total_out = P->total;
    return WPM_OK;
}

// ------------------------------------------------------------------ multi-GPU

namespace {

// split rounds on the plan: from the root tasks at `depth`, then (while the
// frontier is smaller than `target`) from the frontier two levels deeper.
// Rows and nodes of everything above the final frontier stay in the plan.
// (depth, records) of the last split of each workload and shard count: the
// next split of the same job aims at its target in one round
std::mutex g_split_mu;
std::map<std::string, std::pair<int, long long>> g_split_seen;

int split_rounds(wpm_plan* P, int depth, long long target, int shard_count, bool calibrate) {
    if (P->d_front2.ensure(1)) return fail(WPM_EINTERNAL, "allocation failed (frontier)");
    const std::string key = P->signature + "#" + std::to_string(shard_count) + "#" + std::to_string(target);
    if (calibrate) {
        std::lock_guard<std::mutex> lk(g_split_mu);
        auto it = g_split_seen.find(key);
        if (it != g_split_seen.end() && it->second.second > 0) {
            const double r = std::log((double)target / (double)it->second.second) / std::log(1.7);
            depth = std::max(1, std::min(60, it->second.first + (int)std::lround(r)));
        }
    }
    const int first_depth = depth;
    int rc = search_split(P, depth);
    if (rc) return rc;
    {
        std::lock_guard<std::mutex> lk(g_split_mu);
        g_split_seen[key] = {first_depth, P->frontier};
    }
    for (int round = 1; round < 8; ++round) {
        if ((unsigned long long)P->frontier > P->front_cap) return WPM_OK;  // caller reruns with room
        // within 2x of the target is enough (a round costs ~0.5-1.5 ms)
        if (2 * P->frontier >= target || P->frontier == 0) return WPM_OK;
        // deep enough in one more round: the frontier grows ~1.7x per branch
        // level (measured 1.6-1.9x at n = 8 and 11, tools/split_sim.c)
        int jump = (int)std::ceil(std::log((double)target / (double)P->frontier) / std::log(1.7));
        depth += std::max(1, std::min(jump, 8));
        if (P->d_front2.ensure(P->front_cap * P->recw)) return fail(WPM_EINTERNAL, "allocation failed (frontier)");
        P->d_front.swap(P->d_front2);  // the current frontier seeds the next round
        CU(cudaMemsetAsync(P->d_front_ctl.p, 0, 16, P->stream));
        K3Launch a;
        a.d_recs = P->d_front2.p;
        a.nrecs = P->frontier;
        a.cutoff = depth;
        a.d_front_out = P->d_front.p;
        a.front_cap = P->front_cap;
        a.full_depth = P->full_depth;
        if ((rc = k3_launch(P, a, P->frame_cap))) return rc;
        unsigned long long fc = 0;
        CU(cudaMemcpyAsync(&fc, P->d_front_ctl.p, 8, cudaMemcpyDeviceToHost, P->stream));
        CU(cudaStreamSynchronize(P->stream));
        P->d2h += 8;
        P->frontier = (long long)fc;
    }
    return WPM_OK;
}

int enable_peer(int dev, int leader) {
    if (dev == leader) return WPM_OK;
    int ok = 0;
    CU(cudaDeviceCanAccessPeer(&ok, dev, leader));
    if (!ok) return fail(WPM_EINTERNAL, "no peer access between the job's GPUs (the shared claim counter needs P2P)");
    CU(cudaSetDevice(dev));
    const cudaError_t e = cudaDeviceEnablePeerAccess(leader, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return fail(WPM_EINTERNAL, "cudaDeviceEnablePeerAccess failed");
    cudaGetLastError();
    return WPM_OK;
}

// frontier target: 640 records per GPU (>= 2048).  Enough that the GPUs
// balance (largest record <= ~0.3 % of the work at n = 8 and 11; static
// max/mean of 5 k records over 8 GPUs 1.05-1.08), few enough that the
// per-record cost stays invisible (1 GPU, n = 11: the claim phase over 5 k
// records = the direct run, over 12.7 k +28 %, tools/gpu/split_probe.py).
// The first split is at depth 5, then one jump to the target depth.
long long frontier_target(int ndev) {
    long long per = 640;
    if (const char* e = std::getenv("WPM_SPLIT_PER_GPU")) per = std::max(1, std::atoi(e));
    return std::max<long long>(std::min<long long>(2048, 4 * per), per * ndev);
}

// first split depth for a 1/W share of the root tasks: the whole tree needs
// ~640 W records, i.e. log_1.7(W) levels more than one GPU's 640 -- so every
// shard reaches its target in one round (a round costs ~0.5-1 ms of launch,
// table copy and ramp-up whatever its size)
// (a shard's target of `per` records: depth 5 gave ~640 records for a whole
// workload, and every 1.7x more records per shard is one level deeper)
int first_split_depth(int ndev, long long per) {
    const double levels = std::log((double)std::max(1, ndev) * (double)std::max<long long>(per, 1) / 640.0) / std::log(1.7);
    return std::max(1, 5 + (int)std::ceil(levels - 1e-9));
}

}  // namespace

// One job over the leader plan and its peers (one plan per device, same
// maps): every device splits its share of the root tasks below the root
// (split_rounds, in parallel), the frontiers are concatenated and copied to
// every device, and every device's kernel 3 pulls frontier records through
// ONE claim counter in the leader's HBM (system-scope atomics over NVLink)
// into its own work queue, sharing them further by donation.
// No device waits for another; the rows are gathered into the leader with
// peer copies and sorted there once.  Host: one thread per device.
static int plan_run_multi(wpm_plan* P) {
    Trace tr;
    auto peek = [&](const char* where) {
        const cudaError_t e = cudaPeekAtLastError();
        if (e != cudaSuccess && tr.on) std::fprintf(stderr, "[wpm] pending CUDA error after %s: %s\n", where, cudaGetErrorString(e));
    };
    const int W = 1 + (int)P->peers.size();
    std::vector<wpm_plan*> all{P};
    for (auto* q : P->peers) all.push_back(q);
    int rc = search_prepare(P, 0, W);  // the leader's share of the root tasks
    if (rc) return rc;
    CU(cudaEventRecord(P->ev[4], P->stream));
    for (int attempt = 0; attempt < 4; ++attempt) {
        CU(cudaSetDevice(P->device));
        g_alloc_stream = P->stream;
        // every device splits its share of the root tasks (t % W == d), in
        // parallel; the frontiers are concatenated on the leader and copied
        // to every device
        std::vector<int> src(W, 0);
        {
            std::vector<std::thread> th;
            for (int d = 0; d < W; ++d)
                th.emplace_back([&, d]() {
                    wpm_plan* q = all[d];
                    if (cudaSetDevice(q->device) != cudaSuccess) {
                        src[d] = fail(WPM_EINTERNAL, "cudaSetDevice failed");
                        return;
                    }
                    g_alloc_stream = q->stream;
                    int r = d ? search_prepare(q, d, W) : WPM_OK;
                    if (!r) r = search_reset(q);
                    if (!r)
                        r = split_rounds(q, P->split_depth > 0 ? P->split_depth
                                                               : first_split_depth(W, (frontier_target(W) + W - 1) / W),
                                         (frontier_target(W) + W - 1) / W, W, P->split_depth <= 0);
                    src[d] = r;
                });
            for (auto& t : th) t.join();
        }
        CU(cudaSetDevice(P->device));
        g_alloc_stream = P->stream;
        for (int d = 0; d < W; ++d)
            if (src[d]) return src[d];
        bool overflow = false;
        long long F = 0;
        for (int d = 0; d < W; ++d) {
            overflow |= (unsigned long long)all[d]->frontier > all[d]->front_cap;
            F += all[d]->frontier;
        }
        if (overflow) {
            for (int d = 0; d < W; ++d)
                all[d]->front_cap = std::max(all[d]->front_cap, (unsigned long long)all[d]->frontier * 5 / 4 + 1024);
            ++P->reruns;
            continue;
        }
        tr.mark("  multi: parallel split");
        peek("split");
        if (P->d_front_all.ensure((size_t)std::max<long long>(F, 1) * P->recw))
            return fail(WPM_EINTERNAL, "allocation failed (frontier)");
        {
            long long at = 0;
            for (int d = 0; d < W; ++d) {
                const size_t bytes = (size_t)all[d]->frontier * P->recw * 4;
                if (bytes)
                    CU(cudaMemcpyPeerAsync(P->d_front_all.p + (size_t)at * P->recw, P->device, all[d]->d_front.p,
                                           all[d]->device, bytes, P->stream));
                at += all[d]->frontier;
            }
        }
        if (!P->claim_raw) {  // plain cudaMalloc: peers reach it through P2P (pool memory would need pool access)
            CU(cudaMalloc(&P->claim_raw, 64));
        }
        CU(cudaMemsetAsync(P->claim_raw, 0, 64, P->stream));
        CU(cudaStreamSynchronize(P->stream));
        for (int d = 0; d < W; ++d) {
            wpm_plan* q = all[d];
            CU(cudaSetDevice(q->device));
            g_alloc_stream = q->stream;
            if (q->d_front.ensure((size_t)std::max<long long>(F, 1) * q->recw))
                return fail(WPM_EINTERNAL, "allocation failed (frontier)");
            CU(cudaStreamSynchronize(q->stream));
            if (F) CU(cudaMemcpyPeerAsync(q->d_front.p, q->device, P->d_front_all.p, P->device, (size_t)F * P->recw * 4,
                                          P->stream));
            q->frontier = F;
            q->claim_count = F;
            q->claim_devices = W;
            q->claim_ctr = static_cast<unsigned long long*>(P->claim_raw);
        }
        CU(cudaSetDevice(P->device));
        g_alloc_stream = P->stream;
        CU(cudaStreamSynchronize(P->stream));
        tr.mark("  multi: frontier to every device");
        peek("frontier copies");
        // every device claims from the shared frontier
        std::vector<int> rcs(W, 0), again(W, 0);
        std::vector<std::thread> th;
        for (int d = 1; d < W; ++d)
            th.emplace_back([&, d]() {
                wpm_plan* q = all[d];
                if (cudaSetDevice(q->device) != cudaSuccess) {
                    rcs[d] = fail(WPM_EINTERNAL, "cudaSetDevice failed");
                    return;
                }
                g_alloc_stream = q->stream;
                rcs[d] = search_main(q, SRC_CLAIM);
                if (!rcs[d]) rcs[d] = search_finish(q, F, &again[d]);
            });
        rcs[0] = search_main(P, SRC_CLAIM);
        if (!rcs[0]) rcs[0] = search_finish(P, F, &again[0]);
        for (auto& t : th) t.join();
        CU(cudaSetDevice(P->device));
        g_alloc_stream = P->stream;
        for (int d = 0; d < W; ++d)
            if (rcs[d]) return rcs[d];
        tr.mark("  multi: claim phase");
        peek("claim phase");
        bool redo = false;
        for (int d = 0; d < W; ++d) redo |= again[d] != 0;
        if (redo) {
            for (int d = 1; d < W; ++d) all[d]->full_depth |= all[0]->full_depth;
            continue;
        }
        break;
    }
    // gather every device's key rows into the leader, then one canonical sort
    long long total = 0, nodes = 0, tasks = 0;
    P->dev_ms.assign(W, 0.0);
    P->dev_nodes.assign(W, 0);
    for (int d = 0; d < W; ++d) {
        total += all[d]->total;
        nodes += all[d]->nodes;
        tasks += all[d]->tasks;
        float ms = 0;
        CU(cudaSetDevice(all[d]->device));
        CU(cudaEventElapsedTime(&ms, all[d]->ev[0], all[d]->ev[1]));
        P->dev_ms[d] = ms;
        P->dev_nodes[d] = all[d]->nodes;
    }
    CU(cudaSetDevice(P->device));
    if (P->d_gather.ensure((size_t)std::max<long long>(total, 1) * P->rw))
        return fail(WPM_EINTERNAL, "device allocation failed (gather)");
    long long at = 0;
    for (int d = 0; d < W; ++d) {
        const size_t bytes = (size_t)all[d]->total * P->rw * 4;
        if (bytes)
            CU(cudaMemcpyPeerAsync(P->d_gather.p + (size_t)at * P->rw, P->device, all[d]->d_out_keys.p, all[d]->device,
                                   bytes, P->stream));
        at += all[d]->total;
        if (d) P->d2h += 0;  // peer copies stay on NVLink
    }
    P->d_out_keys.swap(P->d_gather);
    P->total = total;
    P->nodes = nodes;
    P->tasks = tasks;
    tr.mark("  multi: gather");
    peek("gather");
    const int src = plan_sort(P);
    peek("sort");
    return src;
}

// a plan spanning devices[0..ndev): devices[0] must be the plan's device; the
// other devices get plans of the same maps (peers); wpm_plan_run then runs
// the job on all of them (plan_run_multi) and leaves the canonical result on
// the leader.  ndev <= 1 detaches the peers.
extern "C" int wpm_plan_set_devices(wpm_plan_t* P, const int32_t* devices, int32_t ndev) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    for (auto* q : P->peers) wpm_plan_destroy(q);
    P->peers.clear();
    if (ndev <= 1) return WPM_OK;
    if (devices[0] != P->device) return fail(WPM_EINVAL, "devices[0] must be the plan's device");
    if (!P->recreate) return fail(WPM_EINVAL, "this plan cannot be replicated");
    for (int i = 1; i < ndev; ++i) {
        int rc = enable_peer(devices[i], P->device);
        if (rc) return rc;
        wpm_plan_t* q = nullptr;
        rc = P->recreate(devices[i], &q);
        if (rc) return rc;
        q->split_depth = P->split_depth;
        P->peers.push_back(q);
    }
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    return WPM_OK;
}

extern "C" int wpm_plan_create_orbits_multi(int32_t n, int32_t p, int64_t facet_cap, const int32_t* devices,
                                            int32_t ndev, wpm_plan_t** out) {
    *out = nullptr;
    if (ndev < 1 || !devices) return fail(WPM_EINVAL, "no devices");
    int rc = wpm_plan_create_orbits(n, p, facet_cap, devices[0], out);
    if (rc) return rc;
    rc = wpm_plan_set_devices(*out, devices, ndev);
    if (rc) {
        wpm_plan_destroy(*out);
        *out = nullptr;
    }
    return rc;
}

extern "C" int wpm_plan_device_stats(const wpm_plan_t* P, int32_t cap, double* ms_out, int64_t* nodes_out) {
    if (!P) return -fail(WPM_EINVAL, "null plan");
    const int W = (int)P->dev_ms.size();
    for (int d = 0; d < W && d < cap; ++d) {
        if (ms_out) ms_out[d] = P->dev_ms[d];
        if (nodes_out) nodes_out[d] = P->dev_nodes[d];
    }
    return W;
}

// split below the root: depth of the first split (0 = off for single-GPU
// runs; multi-GPU runs always split, from depth 3 by default)
extern "C" int wpm_plan_set_split(wpm_plan_t* P, int32_t depth) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (depth < 0 || depth > 255) return fail(WPM_EINVAL, "split depth out of range");
    P->split_depth = depth;
    for (auto* q : P->peers) q->split_depth = depth;
    return WPM_OK;
}

// ---- the same protocol across processes (one per GPU, torch.distributed):
// rank 0 splits and broadcasts the frontier; a claim counter in rank 0's HBM
// is shared through a CUDA IPC handle; every rank runs the claim phase.

extern "C" int wpm_plan_split(wpm_plan_t* P, int32_t shard_index, int32_t shard_count, int32_t depth, int64_t target,
                              int64_t* count) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (shard_count < 1) shard_count = 1;
    if (shard_index < 0 || shard_index >= shard_count) return fail(WPM_EINVAL, "bad shard index");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    P->ran = false;
    int rc = search_prepare(P, shard_index, shard_count);
    if (rc) return rc;
    CU(cudaEventRecord(P->ev[4], P->stream));
    for (int attempt = 0; attempt < 3; ++attempt) {
        if ((rc = search_reset(P))) return rc;
        const long long tgt = target > 0 ? target : frontier_target(1);
        if ((rc = split_rounds(P, depth > 0 ? depth : first_split_depth(shard_count, tgt), tgt, shard_count,
                               depth <= 0))) return rc;
        if ((unsigned long long)P->frontier <= P->front_cap) break;
        P->front_cap = (unsigned long long)P->frontier + (unsigned long long)P->frontier / 4 + 1024;
    }
    P->split_kept = true;  // the split's rows / nodes belong to this plan's claim run
    P->claim_devices = shard_count;
    if (count) *count = P->frontier;
    return WPM_OK;
}

extern "C" int wpm_plan_frontier(const wpm_plan_t* P, const uint32_t** recs, int64_t* count, int32_t* recw) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (recs) *recs = P->d_front.p;
    if (count) *count = P->frontier;
    if (recw) *recw = P->recw;
    return WPM_OK;
}

extern "C" int wpm_plan_load_frontier(wpm_plan_t* P, const uint32_t* recs, int64_t count) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    if (P->d_front.ensure((size_t)std::max<int64_t>(count, 1) * P->recw))
        return fail(WPM_EINTERNAL, "allocation failed (frontier)");
    if (count) CU(cudaMemcpyAsync(P->d_front.p, recs, (size_t)count * P->recw * 4, cudaMemcpyDefault, P->stream));
    CU(cudaStreamSynchronize(P->stream));
    P->frontier = count;  // a plan that split keeps its split's rows / nodes for the claim run
    return WPM_OK;
}

extern "C" int wpm_claim_counter_create(int32_t device, void** counter, uint8_t* ipc_handle) {
    CU(cudaSetDevice(device));
    void* p = nullptr;
    CU(cudaMalloc(&p, 64));
    CU(cudaMemset(p, 0, 64));
    if (ipc_handle) {
        cudaIpcMemHandle_t h;
        CU(cudaIpcGetMemHandle(&h, p));
        std::memcpy(ipc_handle, &h, sizeof(h));
    }
    *counter = p;
    return WPM_OK;
}

extern "C" int wpm_claim_counter_open(int32_t device, const uint8_t* ipc_handle, void** counter) {
    CU(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof(h));
    CU(cudaIpcOpenMemHandle(counter, h, cudaIpcMemLazyEnablePeerAccess));
    return WPM_OK;
}

extern "C" int wpm_claim_counter_reset(int32_t device, void* counter) {
    CU(cudaSetDevice(device));
    CU(cudaMemset(counter, 0, 64));
    return WPM_OK;
}

extern "C" int wpm_claim_counter_close(int32_t device, void* counter, int32_t opened) {
    CU(cudaSetDevice(device));
    if (opened) CU(cudaIpcCloseMemHandle(counter));
    else CU(cudaFree(counter));
    return WPM_OK;
}

// the claim phase on this plan: pull records of the loaded (or own) frontier
// through the shared counter; the rank that split keeps the split's rows and
// nodes.  Sorts this plan's rows canonically (the input of the gather).
extern "C" int wpm_plan_run_claim(wpm_plan_t* P, void* counter, int64_t* total_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    P->ran = false;
    int rc;
    if (!P->split_kept) {  // a plan that did not split: the loaded frontier is all it claims from
        const long long loaded = P->frontier;
        if ((rc = search_prepare(P, 0, 1))) return rc;
        CU(cudaEventRecord(P->ev[4], P->stream));
        if ((rc = search_reset(P))) return rc;
        P->frontier = loaded;  // (search_reset clears the split count)
    }
    P->claim_count = P->frontier;
    P->claim_ctr = static_cast<unsigned long long*>(counter);
    if ((rc = search_main(P, SRC_CLAIM))) return rc;
    int again = 0;
    if ((rc = search_finish(P, P->frontier, &again))) return rc;
    P->split_kept = false;
    if (again) return fail(WPM_EINTERNAL, "claim phase outgrew its buffers; rerun the job (sizes were raised)");
    if ((rc = plan_sort(P))) return rc;
    P->ran = true;
    if (total_out) *total_out = P->total;
    return WPM_OK;
}

// progress (SearchJob::progress, search.hpp:54): fn(done, total, user) from
// the calling thread while a run is in flight -- root tasks finished of the
// run's root tasks (or frontier records), monotone, the last call done == total
extern "C" int wpm_plan_set_progress(wpm_plan_t* P, void (*fn)(int64_t, int64_t, void*), void* user) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    CU(cudaSetDevice(P->device));
    if (fn && !P->progress_host) {
        void* h = nullptr;
        CU(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(h, 0, 64);
        void* d = nullptr;
        CU(cudaHostGetDevicePointer(&d, h, 0));
        P->progress_host = static_cast<unsigned long long*>(h);
        P->progress_dev = static_cast<unsigned long long*>(d);
    }
    P->progress_fn = fn;
    P->progress_user = user;
    return WPM_OK;
}

// per-root search nodes of the following runs' main phase (root tasks, or
// frontier records after a split): the input of the multi-GPU scaling
// projection (a list schedule of the records over W GPUs)
extern "C" int wpm_plan_set_root_stats(wpm_plan_t* P, int32_t on) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    P->root_stats = on != 0;
    return WPM_OK;
}

// nodes of each root task / frontier record of the last run (at most cap);
// returns the root count, and the split phase's own nodes in *split_nodes
extern "C" int64_t wpm_plan_root_nodes(wpm_plan_t* P, int64_t* out, int64_t cap, int64_t* split_nodes) {
    if (!P) return -fail(WPM_EINVAL, "null plan");
    if (!P->root_stats || P->root_count <= 0) return 0;
    CU(cudaSetDevice(P->device));
    const long long k = std::min<long long>(cap, P->root_count);
    std::vector<unsigned long long> h((size_t)P->root_count);
    CU(cudaMemcpy(h.data(), P->d_root_nodes.p, (size_t)P->root_count * 8, cudaMemcpyDeviceToHost));
    long long sum = 0;
    for (long long i = 0; i < P->root_count; ++i) sum += (long long)h[(size_t)i];
    for (long long i = 0; i < k; ++i) out[i] = (int64_t)h[(size_t)i];
    if (split_nodes) *split_nodes = P->nodes - sum;
    return P->root_count;
}

// search-node budget of the following runs (0 = none): a run that reaches it
// stops early and reports truncated = 1 -- a throughput / divergence stress
// on universes whose full enumeration is out of reach, not an enumeration
extern "C" int wpm_plan_set_node_budget(wpm_plan_t* P, int64_t budget) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (budget < 0) return fail(WPM_EINVAL, "negative node budget");
    P->node_budget = (unsigned long long)budget;
    return WPM_OK;
}

extern "C" int wpm_plan_truncated(const wpm_plan_t* P) { return P && P->truncated ? 1 : 0; }

extern "C" int wpm_plan_stats(const wpm_plan_t* P, double* ms_search, double* ms_sort, int64_t* nodes,
                              int64_t* tasks) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (ms_search) *ms_search = P->ms_search;
    if (ms_sort) *ms_sort = P->ms_sort;
    if (nodes) *nodes = P->nodes;
    if (tasks) *tasks = P->tasks;
    return WPM_OK;
}

extern "C" int wpm_plan_timing(const wpm_plan_t* P, double* ms_total, int32_t* warps) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (ms_total) *ms_total = P->ms_total;
    if (warps) *warps = P->warps;
    return WPM_OK;
}

extern "C" int wpm_plan_device_result(const wpm_plan_t* P, const uint32_t** bits32, const uint16_t** map_ids,
                                      int64_t* count, int32_t* words32) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    *bits32 = P->d_sorted_bits.p;
    *map_ids = P->d_sorted_map.p;
    *count = P->total;
    *words32 = P->w32;
    return WPM_OK;
}

extern "C" int wpm_canonical_sort_device(int32_t device, const uint32_t* bits32, const uint16_t* map_ids,
                                         int64_t count, int32_t words32, uint32_t* out_bits32, uint16_t* out_map,
                                         int64_t* dups, void* stream) {
    CU(cudaSetDevice(device));
    init_pool(device);
    cudaStream_t st = (cudaStream_t)stream;
    g_alloc_stream = st;
    if (count <= 0) {
        if (dups) *dups = 0;
        return WPM_OK;
    }
    const int kw = key_words_for(words32);
    if (kw < 0) return fail(WPM_EINVAL, "rows wider than 64 words");
    DevBuf<uint8_t> temp;
    DevBuf<uint32_t> keys;
    DevBuf<unsigned long long> d;
    const size_t tb = canon_sort_temp_bytes(count, words32);
    if (temp.ensure(tb) || keys.ensure((size_t)count * rec_words(words32)) || d.ensure(1))
        return fail(WPM_EINTERNAL, "allocation failed (sort)");
    CU(cudaMemsetAsync(d.p, 0, 8, st));
    if (canon_pack(bits32, map_ids, count, words32, keys.p, st) ||
        canon_sort_keys(keys.p, count, words32, out_bits32, out_map, temp.p, temp.n, nullptr, d.p, st))
        return fail(WPM_EINTERNAL, std::string("canonical sort: ") + cudaGetErrorString(cudaGetLastError()));
    unsigned long long h = 0;
    CU(cudaMemcpyAsync(&h, d.p, 8, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (dups) *dups = (int64_t)h;
    return WPM_OK;
}

extern "C" int wpm_int_peak(int32_t device, double* ops_per_s) {
    CU(cudaSetDevice(device));
    double v = 0;
    if (int_peak_measure(device, &v)) return fail(WPM_EINTERNAL, "int peak microbenchmark failed");
    *ops_per_s = v;
    return WPM_OK;
}

extern "C" int wpm_plan_fetch(wpm_plan_t* P, wpm_result_t** out) {
    *out = nullptr;
    if (!P) return fail(WPM_EINVAL, "null plan");
    CU(cudaSetDevice(P->device));
    const int K = P->num_maps;
    auto* R = new wpm_result_t();
    R->num_maps = K;
    R->words = P->w32 / 2;
    R->total = P->total;
    R->counts = new int64_t[K];
    R->offsets = new int64_t[K + 1];
    R->offsets[0] = 0;
    for (int i = 0; i < K; ++i) {
        R->counts[i] = (int64_t)P->per_map[i];
        R->offsets[i + 1] = R->offsets[i] + R->counts[i];
    }
    size_t got = 0;
    R->bits = static_cast<uint64_t*>(g_pinned.get((size_t)std::max<long long>(P->total, 1) * R->words * 8, &got));
    if (!R->bits) {
        delete[] R->counts;
        delete[] R->offsets;
        delete R;
        return fail(WPM_EINTERNAL, "pinned host allocation failed");
    }
    {
        std::lock_guard<std::mutex> lk(g_block_mu);
        g_block_size[R->bits] = got;
    }
    if (P->total > 0) {
        const cudaError_t e = cudaMemcpyAsync(R->bits, P->d_sorted_bits.p, (size_t)P->total * P->w32 * 4,
                                              cudaMemcpyDeviceToHost, P->stream);
        if (e != cudaSuccess || cudaStreamSynchronize(P->stream) != cudaSuccess) {
            wpm_result_free(R);
            return fail(WPM_EINTERNAL, "result copy failed");
        }
    }
    P->d2h += (long long)P->total * P->w32 * 4;
    R->nodes = P->nodes;
    R->duplicates = P->dups;
    R->ms_total = P->ms_total;
    R->h2d_bytes = P->h2d;
    R->d2h_bytes = P->d2h;
    R->ms_search = P->ms_search;
    R->ms_sort = P->ms_sort;
    R->tasks = P->tasks;
    *out = R;
    trace_pending("fetch");
    return WPM_OK;
}

extern "C" void wpm_plan_destroy(wpm_plan_t* P) {
    if (!P) return;
    trace_pending("destroy (entry)");
    for (auto* q : P->peers) wpm_plan_destroy(q);
    P->peers.clear();
    cudaSetDevice(P->device);
    trace_pending("destroy (peers gone)");
    if (P->progress_host) cudaFreeHost(P->progress_host);
    if (P->claim_raw) cudaFree(P->claim_raw);
    trace_pending("destroy (host / claim memory)");
    DevCtx::Bundle b;
    b.s = P->stream;
    for (int i = 0; i < 5; ++i) b.ev[i] = P->ev[i];
    const int dev = P->device;
    // every buffer's last use is complete once the stream is idle: they go to
    // the block cache for the next plan on this device (the pool otherwise)
    g_recycle = b.s && cudaStreamSynchronize(b.s) == cudaSuccess;
    delete P;
    g_recycle = false;
    trace_pending("destroy (buffers)");
    if (b.s) {
        std::lock_guard<std::mutex> lk(g_dev[dev].mu);
        g_dev[dev].free_bundles.push_back(b);
    }
}

extern "C" void wpm_result_free(wpm_result_t* R) {
    if (!R) return;
    delete[] R->counts;
    delete[] R->offsets;
    if (R->bits) {
        size_t sz = 0;
        {
            std::lock_guard<std::mutex> lk(g_block_mu);
            auto it = g_block_size.find(R->bits);
            if (it != g_block_size.end()) {
                sz = it->second;
                g_block_size.erase(it);
            }
        }
        if (sz) g_pinned.put(R->bits, sz);
    }
    delete R;
}

extern "C" int wpm_enumerate(const wpm_job_t* job, wpm_result_t** out) {
    *out = nullptr;
    if (!job) return fail(WPM_EINVAL, "null job");
    const int32_t M = job->num_facets;
    wpm_plan_t* P = nullptr;
    const int dev0 = job->num_devices > 1 && job->devices ? job->devices[0] : job->device;
    int rc = wpm_plan_create_universes(job->m, job->n, 1, &M, job->facets, job->facet_cap, job->required,
                                       job->num_required, job->forbidden, job->num_forbidden, dev0, &P);
    if (rc) return rc;
    if (job->progress) rc = wpm_plan_set_progress(P, job->progress, job->progress_user);
    if (!rc && job->num_devices > 1 && job->devices) rc = wpm_plan_set_devices(P, job->devices, job->num_devices);
    if (!rc) rc = wpm_plan_run(P, job->shard_count > 1 ? job->shard_index : 0, std::max(1, job->shard_count), nullptr);
    if (!rc) rc = wpm_plan_fetch(P, out);
    wpm_plan_destroy(P);
    return rc;
}

extern "C" int wpm_enumerate_orbits(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_result_t** out) {
    *out = nullptr;
    Trace tr;
    wpm_plan_t* P = nullptr;
    int rc = wpm_plan_create_orbits(n, p, facet_cap, device, &P);
    tr.mark("create (orbits, k1, k2)");
    if (rc) return rc;
    rc = wpm_plan_run(P, 0, 1, nullptr);
    tr.mark("run (k3 + sort)");
    if (!rc) rc = wpm_plan_fetch(P, out);
    tr.mark("fetch (D2H)");
    wpm_plan_destroy(P);
    tr.mark("destroy");
    return rc;
}

// write_complex / write_complexes (complex_io.hpp:21-39)
extern "C" int64_t wpm_write_cplx(const wpm_result_t* R, int32_t map, int32_t m, int32_t n, const uint64_t* universe,
                                  char* buf, int64_t buf_len) {
    if (!R || map < 0 || map >= R->num_maps) return -fail(WPM_EINVAL, "bad map index");
    int64_t len = 0;
    char line[512];
    auto put = [&](const char* s, int k) {
        if (len + k <= buf_len && buf) std::memcpy(buf + len, s, (size_t)k);
        len += k;
    };
    const int W = R->words;
    for (int64_t i = R->offsets[map]; i < R->offsets[map + 1]; ++i) {
        if (i > R->offsets[map]) put("\n", 1);
        int k = std::snprintf(line, sizeof(line), "%d %d\n", m, n);
        put(line, k);
        const uint64_t* K = R->bits + (size_t)i * W;
        for (int w = 0; w < W; ++w)
            for (uint64_t x = K[w]; x; x &= x - 1) {
                const uint64_t f = universe[w * 64 + __builtin_ctzll(x)];
                k = 0;
                bool first = true;
                for (uint64_t y = f; y; y &= y - 1) {
                    if (!first) line[k++] = ' ';
                    k += std::snprintf(line + k, sizeof(line) - (size_t)k, "%d", __builtin_ctzll(y));
                    first = false;
                }
                line[k++] = '\n';
                put(line, k);
            }
    }
    return len;
}

// ------------------------------------------------------------------ Algorithm 2 lines 7 / 13

namespace {

uint32_t host_binom(int a, int b) { return binom_small(a, b); }

// all n-subsets of [m] in ascending mask order (catalog.hpp:112-120), 0-based
std::vector<uint16_t> subsets_ascending(int m, int n) {
    std::vector<uint16_t> out;
    for (uint32_t x = 0; x < (1u << m); ++x)
        if (__builtin_popcount(x) == n) out.push_back((uint16_t)x);
    return out;
}

}  // namespace

// pipeline.hpp:58-89: union of the last run's WPM lists (line 7), then the
// full-support and seedness filters (line 13), resident on the device
extern "C" int wpm_plan_line13(wpm_plan_t* P, int64_t* line7_out, int64_t* line13_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (!P->ran) return fail(WPM_EINVAL, "line 13 needs a completed wpm_plan_run");
    const int m = P->m, n = P->n;
    const long long U = host_binom(m, n);
    if (m > 16 || U > 2048) return fail(WPM_EINVAL, "line 13 needs C(m, n) <= 2048 facets in the label universe");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    const int gw = (int)((U + 31) / 32);
    const int kw = key_words_for(gw);
    const long long cnt = P->total;
    P->gw = gw;
    if (P->unrank.empty()) {
        P->unrank = subsets_ascending(m, n);
        if (P->d_unrank.ensure(U)) return fail(WPM_EINTERNAL, "device allocation failed (line 13)");
        CU(cudaMemcpyAsync(P->d_unrank.p, P->unrank.data(), U * 2, cudaMemcpyHostToDevice, P->stream));
        P->h2d += U * 2;
    }
    const size_t tsort = canon_sort_temp_bytes(std::max<long long>(cnt, 1), gw);
    const size_t tsel = l13_select_temp_bytes(std::max<long long>(cnt, 1));
    size_t total_facets = 0;
    for (const MapDesc& d : P->desc) total_facets = std::max<size_t>(total_facets, d.facet_off + d.M);
    if (P->d_gidx.ensure(total_facets) || P->d_l13_keys.ensure((size_t)cnt * rec_words(gw)) ||
        P->d_l13_rows.ensure((size_t)cnt * gw) || P->d_l13_map.ensure(cnt) || P->d_l13_iota.ensure(cnt) ||
        P->d_l13_uidx.ensure(cnt) || P->d_l13_sidx.ensure(cnt) || P->d_l13_flags.ensure(cnt) ||
        P->d_l13_temp.ensure(std::max(tsort, tsel)) || P->d_l13_num.ensure(2) || P->d_l13_dups.ensure(1))
        return fail(WPM_EINTERNAL, "device allocation failed (line 13)");
    CU(cudaEventRecord(P->ev[0], P->stream));
    CU(cudaMemsetAsync(P->d_l13_dups.p, 0, 8, P->stream));
    if (l13_global_rank(P->num_maps, P->d_maps.p, P->d_facets.p, P->d_gidx.p, P->stream) ||
        l13_remap(P->d_sorted_bits.p, P->d_sorted_map.p, cnt, P->w32, P->d_maps.p, P->d_gidx.p, kw, rec_words(gw),
                  P->d_l13_keys.p, P->num_sms, P->stream) ||
        canon_sort_keys(P->d_l13_keys.p, cnt, gw, P->d_l13_rows.p, P->d_l13_map.p, P->d_l13_temp.p,
                        P->d_l13_temp.n, nullptr, P->d_l13_dups.p, P->stream) ||
        l13_unique(P->d_l13_rows.p, cnt, gw, P->d_l13_flags.p, P->d_l13_iota.p, P->d_l13_uidx.p, P->d_l13_num.p,
                   P->d_l13_temp.p, P->d_l13_temp.n, P->stream))
        return fail(WPM_EINTERNAL, std::string("line 7 union: ") + cudaGetErrorString(cudaGetLastError()));
    CU(cudaEventRecord(P->ev[1], P->stream));
    if (cnt > 0) CU(cudaMemsetAsync(P->d_l13_flags.p, 0, cnt, P->stream));
    if (l13_filter(P->d_l13_rows.p, gw, P->d_l13_uidx.p, P->d_l13_num.p, cnt, P->d_unrank.p, m, (int)U,
                   P->d_l13_flags.p, P->d_l13_sidx.p, P->d_l13_num.p + 1, P->d_l13_temp.p, P->d_l13_temp.n,
                   P->num_sms, P->stream))
        return fail(WPM_EINTERNAL, std::string("line 13 filter: ") + cudaGetErrorString(cudaGetLastError()));
    CU(cudaEventRecord(P->ev[2], P->stream));
    int num[2] = {0, 0};
    unsigned long long dups = 0;
    CU(cudaMemcpyAsync(num, P->d_l13_num.p, 8, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaMemcpyAsync(&dups, P->d_l13_dups.p, 8, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaStreamSynchronize(P->stream));
    P->d2h += 16;
    if ((long long)num[0] + (long long)dups != cnt)
        return fail(WPM_EINTERNAL, "line 7: unique + duplicate rows != rows");
    P->line7 = num[0];
    P->line13 = num[1];
    CU(cudaEventElapsedTime(&P->ms_union, P->ev[0], P->ev[1]));
    CU(cudaEventElapsedTime(&P->ms_filter, P->ev[1], P->ev[2]));
    if (line7_out) *line7_out = P->line7;
    if (line13_out) *line13_out = P->line13;
    return WPM_OK;
}

extern "C" int wpm_plan_line13_timing(const wpm_plan_t* P, double* ms_union, double* ms_filter) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (ms_union) *ms_union = P->ms_union;
    if (ms_filter) *ms_filter = P->ms_filter;
    return WPM_OK;
}

// pipeline.hpp:91-103: canonical_form (isomorphism.hpp:228-303) of every
// line-13 survivor, then one representative per class in order of first
// appearance -- on the device, on the resident line-13 result
extern "C" int wpm_plan_line15(wpm_plan_t* P, int64_t* line15_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (P->line13 < 0) return fail(WPM_EINVAL, "line 15 needs wpm_plan_line13 first");
    const int m = P->m, n = P->n;
    if (m > 15 || n > 11) return fail(WPM_EINVAL, "line 15 on the device needs m <= 15 and n <= 11");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    const long long cnt = P->line13;
    const int gw = P->gw;
    const size_t tdd = l15_dedupe_temp_bytes(std::max<long long>(cnt, 1), gw);
    if (P->d_l15_rows.ensure((size_t)std::max<long long>(cnt, 1) * gw) || P->d_l15_sidx.ensure(cnt + 1) ||
        P->d_l15_iota.ensure(cnt + 1) || P->d_l15_rep.ensure(cnt + 1) || P->d_l15_first.ensure(cnt + 1) ||
        P->d_l15_temp.ensure(tdd) || P->d_l15_num.ensure(2) || P->d_l15_ctl.ensure(5) ||
        P->d_l15_cost.ensure(cnt + 1))
        return fail(WPM_EINTERNAL, "device allocation failed (line 15)");
    CU(cudaEventRecord(P->ev[0], P->stream));
    if (l15_max_facets(P->d_l13_rows.p, gw, P->d_l13_sidx.p, cnt, P->d_l15_num.p, P->stream))
        return fail(WPM_EINTERNAL, "line 15: facet count pass failed");
    int kmax = 0;
    CU(cudaMemcpyAsync(&kmax, P->d_l15_num.p, 4, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaStreamSynchronize(P->stream));
    // minimal non-faces: a few dozen for Picard-4 seeds (<= 64 measured for
    // n <= 11); the kernel flags an overflow and the launch repeats with
    // twice the room (exact either way)
    int mnfcap = 64;
    unsigned long long ctl[5] = {0, 0, 0, 0, 0};
    P->l15_launches = 0;
    // canonical-form cache: isomorphic survivors after the first confirm a
    // cached form instead of searching (WPM_L15_CACHE=0 disables)
    const int cslots = 1 << 14;
    const bool use_cache = !(std::getenv("WPM_L15_CACHE") && std::atoi(std::getenv("WPM_L15_CACHE")) == 0);
    if (use_cache && (P->d_l15_ckey.ensure(cslots) || P->d_l15_cdata.ensure((size_t)cslots * (kmax + 1))))
        return fail(WPM_EINTERNAL, "device allocation failed (line 15 cache)");
    for (;;) {
        const L15Layout L = l15_layout(m, n, kmax, mnfcap, gw);
        if (L.P > 2048 || l15_smem_bytes(L) > 227 * 1024)
            return fail(WPM_EINTERNAL, "line 15: complexes too large for the device layout");
        ++P->l15_launches;
        if (l15_launch(L, P->d_l13_rows.p, P->d_l13_sidx.p, nullptr, P->d_unrank.p, nullptr, nullptr, cnt,
                       P->d_l15_rows.p, nullptr, nullptr, P->d_l15_cost.p, P->d_l15_ctl.p,
                       use_cache ? P->d_l15_ckey.p : nullptr, use_cache ? P->d_l15_cdata.p : nullptr, cslots,
                       P->num_sms, P->stream))
            return fail(WPM_EINTERNAL, std::string("line 15 canonical forms: ") +
                                           cudaGetErrorString(cudaGetLastError()));
        CU(cudaMemcpyAsync(ctl, P->d_l15_ctl.p, sizeof(ctl), cudaMemcpyDeviceToHost, P->stream));
        CU(cudaStreamSynchronize(P->stream));
        if (ctl[1] == 0) break;
        mnfcap *= 2;
    }
    P->l15_kmax = kmax;
    P->l15_mnfcap = mnfcap;
    CU(cudaEventRecord(P->ev[1], P->stream));
    if (l15_dedupe(P->d_l15_rows.p, cnt, gw, P->d_l15_sidx.p, P->d_l15_iota.p, P->d_l15_first.p, P->d_l15_rep.p,
                   P->d_l15_num.p + 1, P->d_l15_temp.p, P->d_l15_temp.n, P->stream))
        return fail(WPM_EINTERNAL, std::string("line 15 dedupe: ") + cudaGetErrorString(cudaGetLastError()));
    CU(cudaEventRecord(P->ev[2], P->stream));
    int nrep = 0;
    CU(cudaMemcpyAsync(&nrep, P->d_l15_num.p + 1, 4, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaStreamSynchronize(P->stream));
    P->d2h += 4 + 4 + sizeof(ctl);
    P->line15 = nrep;
    P->l15_leaves = (long long)ctl[2];
    P->l15_steps = (long long)ctl[3];
    P->l15_hits = (long long)ctl[4];
    CU(cudaEventElapsedTime(&P->ms_canon, P->ev[0], P->ev[1]));
    CU(cudaEventElapsedTime(&P->ms_dedupe, P->ev[1], P->ev[2]));
    if (line15_out) *line15_out = P->line15;
    return WPM_OK;
}

// per-survivor search cost of the last wpm_plan_line15 (placements), survivor order
extern "C" int64_t wpm_plan_line15_costs(wpm_plan_t* P, int64_t* out, int64_t cap) {
    if (!P) return -fail(WPM_EINVAL, "null plan");
    if (P->line15 < 0) return -fail(WPM_EINVAL, "call wpm_plan_line15 first");
    const long long n = std::min<long long>(cap, P->line13);
    if (n > 0 && (cudaMemcpyAsync(out, P->d_l15_cost.p, (size_t)n * 8, cudaMemcpyDeviceToHost, P->stream) !=
                      cudaSuccess ||
                  cudaStreamSynchronize(P->stream) != cudaSuccess))
        return -fail(WPM_EINTERNAL, "line 15 costs: copy failed");
    return P->line13;
}

extern "C" int wpm_plan_line15_stats(const wpm_plan_t* P, double* ms_canon, double* ms_dedupe, int64_t* labelings,
                                     int64_t* placements, int32_t* launches, int64_t* cache_hits) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (cache_hits) *cache_hits = P->l15_hits;
    if (launches) *launches = P->l15_launches;
    if (ms_canon) *ms_canon = P->ms_canon;
    if (ms_dedupe) *ms_dedupe = P->ms_dedupe;
    if (labelings) *labelings = P->l15_leaves;
    if (placements) *placements = P->l15_steps;
    return WPM_OK;
}

// global bitset rows -> the C-ABI complex list (CSR of 1-based facet masks)
static wpm_complexes_t* complexes_from_rows(int m, int n, int gw, const std::vector<uint16_t>& unr,
                                            const uint32_t* rows, long long count) {
    auto* C = new wpm_complexes_t();
    C->line15 = -1;
    C->m = m;
    C->n = n;
    C->count = count;
    C->words = (gw + 1) / 2;
    C->offsets = new int64_t[count + 1];
    C->bits = new uint64_t[(size_t)count * C->words + 1];
    long long nf = 0;
    for (long long i = 0; i < count; ++i) {
        const uint32_t* r = rows + (size_t)i * gw;
        for (int w = 0; w < gw; ++w) nf += __builtin_popcount(r[w]);
    }
    C->facets = new uint64_t[nf + 1];
    long long k = 0;
    for (long long i = 0; i < count; ++i) {
        const uint32_t* r = rows + (size_t)i * gw;
        C->offsets[i] = k;
        uint64_t* b = C->bits + (size_t)i * C->words;
        for (int w = 0; w < C->words; ++w) b[w] = 0;
        for (int w = 0; w < gw; ++w) {
            b[w >> 1] |= (uint64_t)r[w] << ((w & 1) * 32);
            for (uint32_t x = r[w]; x; x &= x - 1) C->facets[k++] = (uint64_t)unr[w * 32 + __builtin_ctz(x)] << 1;
        }
    }
    C->offsets[count] = k;
    return C;
}

extern "C" int wpm_plan_fetch_complexes(wpm_plan_t* P, int32_t which, wpm_complexes_t** out) {
    *out = nullptr;
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (P->line7 < 0) return fail(WPM_EINVAL, "call wpm_plan_line13 first");
    if (which != 7 && which != 13 && which != 14 && which != 15)
        return fail(WPM_EINVAL, "which must be 7, 13, 14 or 15");
    if (which >= 14 && P->line15 < 0) return fail(WPM_EINVAL, "call wpm_plan_line15 first");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    const long long count = which == 7 ? P->line7 : which == 15 ? P->line15 : P->line13;
    const int gw = P->gw;
    // the key buffer is free after the union: gather the selected rows there
    const int grc = which >= 14 ? l15_gather(P->d_l15_rows.p, gw, which == 15 ? P->d_l15_rep.p : P->d_l15_iota.p,
                                             count, P->d_l13_keys.p, P->stream)
                                : l13_gather(P->d_l13_rows.p, gw, which == 7 ? P->d_l13_uidx.p : P->d_l13_sidx.p,
                                             count, P->d_l13_keys.p, P->stream);
    if (grc) return fail(WPM_EINTERNAL, "gather failed");
    std::vector<uint32_t> h((size_t)count * gw + 1);
    if (count) CU(cudaMemcpyAsync(h.data(), P->d_l13_keys.p, (size_t)count * gw * 4, cudaMemcpyDeviceToHost,
                                  P->stream));
    CU(cudaStreamSynchronize(P->stream));
    P->d2h += (long long)count * gw * 4;
    wpm_complexes_t* C = complexes_from_rows(P->m, P->n, gw, P->unrank, h.data(), count);
    C->line7 = P->line7;
    C->line13 = P->line13;
    C->ms_union = P->ms_union;
    C->ms_filter = P->ms_filter;
    C->line15 = P->line15;
    C->ms_canon = P->ms_canon;
    C->ms_dedupe = P->ms_dedupe;
    *out = C;
    return WPM_OK;
}

extern "C" void wpm_complexes_free(wpm_complexes_t* C) {
    if (!C) return;
    delete[] C->offsets;
    delete[] C->facets;
    delete[] C->bits;
    delete C;
}

extern "C" int64_t wpm_write_complexes(const wpm_complexes_t* C, char* buf, int64_t buf_len) {
    if (!C) return -fail(WPM_EINVAL, "null complex list");
    int64_t len = 0;
    char line[512];
    auto put = [&](const char* s, int k) {
        if (len + k <= buf_len && buf) std::memcpy(buf + len, s, (size_t)k);
        len += k;
    };
    for (int64_t i = 0; i < C->count; ++i) {  // complex_io.hpp:21-39
        if (i > 0) put("\n", 1);
        int k = std::snprintf(line, sizeof(line), "%d %d\n", C->m, C->n);
        put(line, k);
        for (int64_t j = C->offsets[i]; j < C->offsets[i + 1]; ++j) {
            k = 0;
            bool first = true;
            for (uint64_t y = C->facets[j]; y; y &= y - 1) {
                if (!first) line[k++] = ' ';
                k += std::snprintf(line + k, sizeof(line) - (size_t)k, "%d", __builtin_ctzll(y));
                first = false;
            }
            line[k++] = '\n';
            put(line, k);
        }
    }
    return len;
}

// is_seed (classify.hpp:51-53) and full support (complex.hpp:64-70) of a
// batch of pure complexes; PureComplex validation (complex.hpp:37-55)
extern "C" int wpm_seed_flags(int32_t m, int32_t n, int64_t count, const int64_t* offsets, const uint64_t* facets,
                              int32_t device, uint8_t* flags_out) {
    if (m < 1 || m > 16) return fail(WPM_EINVAL, "vertex count out of range (1..16 on the device)");
    if (n < 0) return fail(WPM_EINVAL, "negative facet size");
    if (count < 0 || (count > 0 && (!offsets || !flags_out))) return fail(WPM_EINVAL, "bad batch");
    const uint64_t full = (((uint64_t)1 << m) - 1) << 1;
    const long long nf = count > 0 ? offsets[count] : 0;
    std::vector<uint16_t> masks((size_t)nf + 1);
    int maxf = 1;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t a = offsets[i], b = offsets[i + 1];
        if (b < a || a < 0 || b > nf) return fail(WPM_EINVAL, "offsets not ascending");
        if (b - a > WPM_MAX_FACETS) return fail(WPM_EINVAL, "complex with more than WPM_MAX_FACETS facets");
        maxf = std::max<int>(maxf, (int)(b - a));
        for (int64_t j = a; j < b; ++j) {
            const uint64_t f = facets[j];
            if (f & ~full) return fail(WPM_EINVAL, "facet uses a label outside 1..m");
            if (__builtin_popcountll(f) != n) return fail(WPM_EINVAL, "purity: facet size differs from n");
            masks[j] = (uint16_t)(f >> 1);
        }
        std::sort(masks.begin() + a, masks.begin() + b);  // PureComplex sorts its facets
        for (int64_t j = a + 1; j < b; ++j)
            if (masks[j] == masks[j - 1]) return fail(WPM_EINVAL, "duplicate facet");
    }
    auto* P = new wpm_plan();
    int rc = plan_init(P, device);
    if (rc == WPM_OK && count > 0) {
        g_alloc_stream = P->stream;
        DevBuf<uint16_t> dm;
        DevBuf<long long> doff;
        DevBuf<uint8_t> dfl;
        maxf = (maxf + 7) & ~7;
        if (dm.ensure(nf + 1) || doff.ensure(count + 1) || dfl.ensure(count)) {
            rc = fail(WPM_EINTERNAL, "device allocation failed (seed flags)");
        } else if (cudaMemcpyAsync(dm.p, masks.data(), (nf + 1) * 2, cudaMemcpyHostToDevice, P->stream) ||
                   cudaMemcpyAsync(doff.p, offsets, (count + 1) * 8, cudaMemcpyHostToDevice, P->stream) ||
                   l13_seed_flags(dm.p, doff.p, count, m, maxf, dfl.p, P->num_sms, P->stream) ||
                   cudaMemcpyAsync(flags_out, dfl.p, count, cudaMemcpyDeviceToHost, P->stream) ||
                   cudaStreamSynchronize(P->stream)) {
            rc = fail(WPM_EINTERNAL, std::string("seed flags: ") + cudaGetErrorString(cudaGetLastError()));
        }
    }
    wpm_plan_destroy(P);
    return rc;
}

// pipeline.hpp:52-89 one-shot for one n: every orbit map, UBT (or the given)
// cap, search + union + filters; returns the line-13 survivors
extern "C" int wpm_pipeline_line13(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_complexes_t** out) {
    *out = nullptr;
    wpm_plan_t* P = nullptr;
    int rc = wpm_plan_create_orbits(n, p, facet_cap, device, &P);
    if (rc) return rc;
    int64_t total = 0, l7 = 0, l13 = 0;
    rc = wpm_plan_run(P, 0, 1, &total);
    if (!rc) rc = wpm_plan_line13(P, &l7, &l13);
    if (!rc) rc = wpm_plan_fetch_complexes(P, 13, out);
    if (!rc) {
        (*out)->h2d_bytes = P->h2d;
        (*out)->d2h_bytes = P->d2h;
    }
    wpm_plan_destroy(P);
    return rc;
}

// pipeline.hpp:52-103 one-shot for one n: lines 1-13 as above, then the
// canonical forms and the first-appearance representatives (line 15)
extern "C" int wpm_pipeline_line15(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_complexes_t** out) {
    *out = nullptr;
    wpm_plan_t* P = nullptr;
    int rc = wpm_plan_create_orbits(n, p, facet_cap, device, &P);
    if (rc) return rc;
    int64_t total = 0, l7 = 0, l13 = 0, l15 = 0;
    rc = wpm_plan_run(P, 0, 1, &total);
    if (!rc) rc = wpm_plan_line13(P, &l7, &l13);
    if (!rc) rc = wpm_plan_line15(P, &l15);
    if (!rc) rc = wpm_plan_fetch_complexes(P, 15, out);
    if (!rc) {
        (*out)->h2d_bytes = P->h2d;
        (*out)->d2h_bytes = P->d2h;
    }
    wpm_plan_destroy(P);
    return rc;
}

// canonical_form (isomorphism.hpp:228-303) and refine_classes (:162-218) of
// a batch of pure complexes; PureComplex validation (complex.hpp:37-55)
extern "C" int wpm_canonical_forms(int32_t m, int32_t n, int64_t count, const int64_t* offsets,
                                   const uint64_t* facets, int32_t device, uint64_t* canon_out, int8_t* classes_out) {
    if (m < 1 || m > 15) return fail(WPM_EINVAL, "vertex count out of range (1..15 for canonical forms)");
    if (n < 1 || n > 11 || n > m) return fail(WPM_EINVAL, "facet size out of range (1..min(11, m))");
    if (count < 0 || (count > 0 && (!offsets || !canon_out))) return fail(WPM_EINVAL, "bad batch");
    const uint64_t full = (((uint64_t)1 << m) - 1) << 1;
    const long long nf = count > 0 ? offsets[count] : 0;
    std::vector<uint16_t> masks((size_t)nf + 1);
    int kmax = 1;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t a = offsets[i], b = offsets[i + 1];
        if (b < a || a < 0 || b > nf) return fail(WPM_EINVAL, "offsets not ascending");
        if (b - a > WPM_MAX_FACETS) return fail(WPM_EINVAL, "complex with more than WPM_MAX_FACETS facets");
        kmax = std::max<int>(kmax, (int)(b - a));
        for (int64_t j = a; j < b; ++j) {
            const uint64_t f = facets[j];
            if (f & ~full) return fail(WPM_EINVAL, "facet uses a label outside 1..m");
            if (__builtin_popcountll(f) != n) return fail(WPM_EINVAL, "purity: facet size differs from n");
            masks[j] = (uint16_t)(f >> 1);
        }
        std::sort(masks.begin() + a, masks.begin() + b);  // PureComplex sorts its facets
        for (int64_t j = a + 1; j < b; ++j)
            if (masks[j] == masks[j - 1]) return fail(WPM_EINVAL, "duplicate facet");
    }
    auto* P = new wpm_plan();
    int rc = plan_init(P, device);
    if (rc == WPM_OK && count > 0) {
        g_alloc_stream = P->stream;
        DevBuf<uint16_t> dm, dout;
        DevBuf<long long> doff;
        DevBuf<int8_t> dcls;
        DevBuf<unsigned long long> dctl, ckey;
        DevBuf<uint16_t> cdata;
        std::vector<uint16_t> hout((size_t)nf + 1);
        std::vector<int8_t> hcls;
        if (dm.ensure(nf + 1) || dout.ensure(nf + 1) || doff.ensure(count + 1) || dctl.ensure(5) ||
            (classes_out && dcls.ensure((size_t)count * 16))) {
            rc = fail(WPM_EINTERNAL, "device allocation failed (canonical forms)");
        } else if (cudaMemcpyAsync(dm.p, masks.data(), (nf + 1) * 2, cudaMemcpyHostToDevice, P->stream) ||
                   cudaMemcpyAsync(doff.p, offsets, (count + 1) * 8, cudaMemcpyHostToDevice, P->stream)) {
            rc = fail(WPM_EINTERNAL, "canonical forms: upload failed");
        } else {
            int mnfcap = 64;
            for (;;) {
                const L15Layout L = l15_layout(m, n, kmax, mnfcap, 1);
                if (L.P > 2048 || l15_smem_bytes(L) > 227 * 1024) {
                    rc = fail(WPM_EINTERNAL, "canonical forms: complexes too large for the device layout");
                    break;
                }
                unsigned long long ctl[5] = {0, 0, 0, 0, 0};
                const int cslots = 1 << 12;
                if ((!ckey.p && (ckey.ensure(cslots) || cdata.ensure((size_t)cslots * (kmax + 1)))) ||
                    l15_launch(L, nullptr, nullptr, nullptr, nullptr, dm.p, doff.p, count, nullptr, dout.p,
                               classes_out ? dcls.p : nullptr, nullptr, dctl.p, ckey.p, cdata.p, cslots,
                               P->num_sms, P->stream) ||
                    cudaMemcpyAsync(ctl, dctl.p, sizeof(ctl), cudaMemcpyDeviceToHost, P->stream) ||
                    cudaStreamSynchronize(P->stream)) {
                    rc = fail(WPM_EINTERNAL, std::string("canonical forms: ") +
                                                 cudaGetErrorString(cudaGetLastError()));
                    break;
                }
                if (ctl[1] == 0) break;
                mnfcap *= 2;
            }
            if (rc == WPM_OK) {
                if (classes_out) hcls.resize((size_t)count * 16);
                if (cudaMemcpyAsync(hout.data(), dout.p, (nf + 1) * 2, cudaMemcpyDeviceToHost, P->stream) ||
                    (classes_out && cudaMemcpyAsync(hcls.data(), dcls.p, (size_t)count * 16, cudaMemcpyDeviceToHost,
                                                    P->stream)) ||
                    cudaStreamSynchronize(P->stream)) {
                    rc = fail(WPM_EINTERNAL, "canonical forms: download failed");
                } else {
                    for (long long j = 0; j < nf; ++j) canon_out[j] = (uint64_t)hout[j] << 1;
                    if (classes_out)
                        for (int64_t i = 0; i < count; ++i)
                            for (int v = 0; v < m; ++v) classes_out[i * m + v] = hcls[(size_t)i * 16 + v];
                }
            }
        }
    }
    wpm_plan_destroy(P);
    return rc;
}

// ------------------------------------------------------------------ Algorithm 1 (the reference's search)

// IncidenceMatrix of a universe (incidence.hpp:34-55): ridges ascending, the
// ridges of each facet ascending, the parents of each ridge ascending
static void host_incidence(const std::vector<uint32_t>& facets, HostIncidence* A) {
    std::vector<uint32_t> ridges;
    for (uint32_t f : facets)
        for (uint32_t x = f; x; x &= x - 1) ridges.push_back(f & ~(x & (0u - x)));
    std::sort(ridges.begin(), ridges.end());
    ridges.erase(std::unique(ridges.begin(), ridges.end()), ridges.end());
    A->M = (int)facets.size();
    A->N = (int)ridges.size();
    A->cols.assign(A->M, {});
    A->parents.assign(A->N, {});
    for (int j = 0; j < A->M; ++j) {
        const uint32_t f = facets[j];
        for (uint32_t x = f; x; x &= x - 1) {
            const uint32_t r = f & ~(x & (0u - x));
            A->cols[j].push_back((int)(std::lower_bound(ridges.begin(), ridges.end(), r) - ridges.begin()));
        }
        std::sort(A->cols[j].begin(), A->cols[j].end());
        for (int r : A->cols[j]) A->parents[r].push_back(j);
    }
}

// enumerate_wpm exactly as the reference runs it (search.hpp:141-258): the
// kernel basis on the host (kbasis.cpp), every leaf of the combination space
// on the device (k6_odometer.cu), then the same canonical sort
// the reference's basis and combination space of every map (kbasis.cpp),
// built once per plan (the maps and pins are fixed)
static int ensure_spaces(wpm_plan* P) {
    if (P->spaces_ok) return WPM_OK;
    const int K = P->num_maps;
    const auto t0 = std::chrono::steady_clock::now();
    P->spaces.assign(K, {});
    for (int i = 0; i < K; ++i) {
        const MapDesc& d = P->desc[i];
        std::vector<uint32_t> fac(d.M);
        CU(cudaMemcpy(fac.data(), P->d_facets.p + d.facet_off, d.M * 4, cudaMemcpyDeviceToHost));
        P->d2h += 4LL * d.M;
        HostIncidence A;
        host_incidence(fac, &A);
        std::vector<int> req, forb;
        if (P->has_pins)
            for (int j = 0; j < d.M; ++j) {
                if ((P->pin_in[(size_t)i * P->mw + (j >> 5)] >> (j & 31)) & 1u) req.push_back(j);
                if ((P->pin_out[(size_t)i * P->mw + (j >> 5)] >> (j & 31)) & 1u) forb.push_back(j);
            }
        if (build_space(A, req, forb, &P->spaces[i])) return fail(WPM_EINFEASIBLE, "link constraints are infeasible");
    }
    P->ms_basis = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    P->spaces_ok = true;
    return WPM_OK;
}

static int run_odometer(wpm_plan* P, const std::vector<CombinationSpaceHost>& spaces, double ms_prep0,
                        int64_t* total_out);

extern "C" int wpm_plan_run_kernel_basis(wpm_plan_t* P, uint64_t candidate_cap, int64_t* total_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    const bool fresh = !P->spaces_ok;
    const int rc = ensure_spaces(P);
    if (rc) return rc;
    for (const auto& cs : P->spaces)
        if (cs.space > candidate_cap)  // search.hpp:147-150
            return fail(WPM_ECAP, "combination space of " + std::to_string(cs.space) + " candidates exceeds cap " +
                                      std::to_string(candidate_cap));
    return run_odometer(P, P->spaces, fresh ? P->ms_basis : 0.0, total_out);
}

// Algorithm 1 over one map with the first `nfixed` blocks (widest first,
// search.hpp:168-170) fixed to candidates cand[0..nfixed): the reference's
// per-item odometer (search.hpp:204-243) over the remaining blocks from
// base' = base ^ the fixed candidates' deltas.  The accepted set is every
// reference-reachable WPM whose coordinates share that prefix.
extern "C" int wpm_plan_run_kernel_basis_prefix(wpm_plan_t* P, int32_t map, int32_t nfixed, const int32_t* cand,
                                                uint64_t candidate_cap, int64_t* total_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (map < 0 || map >= P->num_maps) return fail(WPM_EINVAL, "bad map index");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    const int rc = ensure_spaces(P);
    if (rc) return rc;
    const CombinationSpaceHost& cs = P->spaces[map];
    const int nb = (int)cs.ncand.size();
    if (nfixed < 0 || nfixed > nb) return fail(WPM_EINVAL, "prefix longer than the block list");
    std::vector<CombinationSpaceHost> sp(P->num_maps);
    for (auto& x : sp) x.space = 0;  // every other map: no leaves
    CombinationSpaceHost& r = sp[map];
    r.s = cs.s;
    r.induced_blocks = cs.induced_blocks;
    r.W32 = cs.W32;
    r.base = cs.base;
    size_t first = 0;
    for (int b = 0; b < nfixed; ++b) {
        if (cand[b] < 0 || cand[b] >= cs.ncand[b]) return fail(WPM_EINVAL, "prefix candidate out of range");
        const uint32_t* d = cs.deltas.data() + (first + (size_t)cand[b]) * cs.W32;
        for (int w = 0; w < cs.W32; ++w) r.base[w] ^= d[w];
        first += (size_t)cs.ncand[b];
    }
    r.ncand.assign(cs.ncand.begin() + nfixed, cs.ncand.end());
    r.deltas.assign(cs.deltas.begin() + (long)(first * cs.W32), cs.deltas.end());
    unsigned long long space = 1;
    bool sat = false;
    for (int c : r.ncand) {
        if (!sat && space > ~0ull / (unsigned long long)c) sat = true;
        if (!sat) space *= (unsigned long long)c;
    }
    r.space = sat ? ~0ull : space;
    if (r.space > candidate_cap)
        return fail(WPM_ECAP, "prefix space of " + std::to_string(r.space) + " candidates exceeds cap " +
                                  std::to_string(candidate_cap));
    return run_odometer(P, sp, 0.0, total_out);
}

// blocks of map `map`'s combination space, widest first: widths[b] generators
// each (1 = a free singleton; candidates = 1 + w + w(w-1)/2); returns the block
// count (writes at most cap) or -status
extern "C" int32_t wpm_plan_space_blocks(wpm_plan_t* P, int32_t map, int32_t* widths, int32_t cap) {
    if (!P || map < 0 || map >= P->num_maps) return -fail(WPM_EINVAL, "bad map index");
    if (cudaSetDevice(P->device) != cudaSuccess) return -fail(WPM_EINTERNAL, "cudaSetDevice failed");
    g_alloc_stream = P->stream;
    const int rc = ensure_spaces(P);
    if (rc) return -rc;
    const auto& w = P->spaces[map].width;
    for (int b = 0; b < (int)w.size() && b < cap; ++b) widths[b] = w[b];
    return (int32_t)w.size();
}

static int run_odometer(wpm_plan* P, const std::vector<CombinationSpaceHost>& spaces, double ms_prep0,
                        int64_t* total_out) {
    P->ran = false;
    P->line7 = P->line13 = P->line15 = -1;
    const int K = P->num_maps;
    const int W32 = (P->maxM + 31) / 32;
    const int Wb = odo_words_bucket(W32);
    if (Wb < 0) return fail(WPM_EINVAL, "the odometer supports universes of at most 1024 facets");
    const auto t0 = std::chrono::steady_clock::now();
    // ---- device tables: vectors at stride Wb (zero padded)
    std::vector<OdoMap> om(K);
    std::vector<int> blk;  // ncand entries, then (after nblk) first-candidate entries
    std::vector<int> ncand_all, first_all;
    std::vector<uint32_t> words;
    long long tasks = 0, leaves = 0;
    // leaves per prefix: ~512 prefixes per lane of the whole grid (8 CTAs x 8
    // warps per SM) -- the cap-passing leaves cluster in parts of the space,
    // so small tasks on the dynamic queue keep the tail short (sweep 4 / 32 /
    // 128 / 512 / 2048 / 8192 at n = 7: 311 / 139 / 78 / 72 / 83 / 109 ms) --
    // and at most 64K leaves of inner loop per lane
    unsigned long long all_leaves = 0;
    for (const auto& cs : spaces) all_leaves += cs.space;
    const unsigned long long lanes = (unsigned long long)P->num_sms * 64 * 32;
    long long per_lane = 512;
    if (const char* e = std::getenv("WPM_ODO_PER_LANE")) per_lane = std::max(1, std::atoi(e));
    const long long inner_target = (long long)std::min<unsigned long long>(
        65536, std::max<unsigned long long>(8, all_leaves / ((unsigned long long)per_lane * lanes)));
    auto put_vec = [&](const uint32_t* v) {
        for (int w = 0; w < Wb; ++w) words.push_back(w < W32 ? v[w] : 0u);
    };
    for (int i = 0; i < K; ++i) {
        const CombinationSpaceHost& cs = spaces[i];
        const int nb = (int)cs.ncand.size();
        OdoMap& o = om[i];
        o.map = i;
        o.n = P->desc[i].n;
        o.fs = P->desc[i].fr_stride;
        o.cap = P->desc[i].cap;
        o.nb = nb;
        o.blk = (int)ncand_all.size();
        o.fr_off = P->desc[i].fr_off;
        // inner blocks: the last r, >= inner_target leaves per prefix (or every block)
        long long inner = 1;
        int r = 0;
        while (r < nb && r < odo_max_inner() && inner < inner_target) inner *= cs.ncand[nb - 1 - r++];
        o.r = r;
        o.inner = inner;
        o.outer = (long long)(cs.space / (unsigned long long)inner);
        o.task0 = tasks;
        tasks += (o.outer + 31) / 32;
        leaves += (long long)cs.space;
        o.base_off = (uint32_t)words.size();
        std::vector<uint32_t> b32(cs.W32);
        for (int w = 0; w < cs.W32; ++w) b32[w] = cs.base[w];
        b32.resize(std::max(W32, cs.W32), 0u);
        put_vec(b32.data());
        int first = 0;
        for (int b = 0; b < nb; ++b) {
            ncand_all.push_back(cs.ncand[b]);
            first_all.push_back(first);
            first += cs.ncand[b];
        }
        o.delta_off = (uint32_t)words.size();
        std::vector<uint32_t> v(std::max(W32, cs.W32), 0u);
        for (int c = 0; c < first; ++c) {
            std::fill(v.begin(), v.end(), 0u);
            for (int w = 0; w < cs.W32; ++w) v[w] = cs.deltas[(size_t)c * cs.W32 + w];
            put_vec(v.data());
        }
        o.step_off = (uint32_t)words.size();
        int c0 = 0;
        for (int b = 0; b < nb; ++b) {  // step c: delta[c] ^ delta[(c + 1) % ncand]
            const int nc = cs.ncand[b];
            for (int c = 0; c < nc; ++c) {
                std::fill(v.begin(), v.end(), 0u);
                const uint32_t* a = cs.deltas.data() + (size_t)(c0 + c) * cs.W32;
                const uint32_t* z = cs.deltas.data() + (size_t)(c0 + (c + 1) % nc) * cs.W32;
                for (int w = 0; w < cs.W32; ++w) v[w] = a[w] ^ z[w];
                put_vec(v.data());
            }
            c0 += nc;
        }
    }
    const int nblk = (int)ncand_all.size();
    blk = ncand_all;
    blk.insert(blk.end(), first_all.begin(), first_all.end());
    if (P->d_odo_maps.ensure(K) || P->d_odo_blk.ensure(blk.size() + 1) || P->d_odo_words.ensure(words.size() + 1) ||
        P->d_odo_ctl.ensure(4) || P->d_out_ctl.ensure(4) || P->d_per_map.ensure(K))
        return fail(WPM_EINTERNAL, "device allocation failed (odometer)");
    CU(cudaMemcpyAsync(P->d_odo_maps.p, om.data(), sizeof(OdoMap) * K, cudaMemcpyHostToDevice, P->stream));
    if (!blk.empty())
        CU(cudaMemcpyAsync(P->d_odo_blk.p, blk.data(), blk.size() * 4, cudaMemcpyHostToDevice, P->stream));
    CU(cudaMemcpyAsync(P->d_odo_words.p, words.data(), words.size() * 4, cudaMemcpyHostToDevice, P->stream));
    P->h2d += (long long)(sizeof(OdoMap) * K + blk.size() * 4 + words.size() * 4);
    P->ms_prep = ms_prep0 + std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (P->out_cap == 0) {
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        const unsigned long long row = (unsigned long long)P->rw * 4 * 3;
        P->out_cap = std::min<unsigned long long>(std::max<unsigned long long>(fr / 16 / row, 1ull << 20), 1ull << 26);
    }
    CU(cudaEventRecord(P->ev[4], P->stream));
    for (int attempt = 0; attempt < 2; ++attempt) {
        if (P->d_out_keys.ensure(P->out_cap * P->rw)) return fail(WPM_EINTERNAL, "device allocation failed (output)");
        CU(cudaMemsetAsync(P->d_out_ctl.p, 0, 32, P->stream));
        CU(cudaMemsetAsync(P->d_odo_ctl.p, 0, 32, P->stream));
        OdoParams op{};
        op.maps = P->d_odo_maps.p;
        op.num_maps = K;
        op.blk_ncand = P->d_odo_blk.p;
        op.blk_first = P->d_odo_blk.p + nblk;
        op.words = P->d_odo_words.p;
        op.fr = P->d_fr.p;
        op.task_ctr = P->d_odo_ctl.p;
        op.total_tasks = tasks;
        op.cnt_words = (P->maxN + 31) / 32;  // ridge bitset words
        op.out_keys = P->d_out_keys.p;
        op.out_ctl = P->d_out_ctl.p;
        op.out_cap = P->out_cap;
        op.rw = P->rw;
        op.leaf_ctr = P->d_odo_ctl.p + 1;
        CU(cudaEventRecord(P->ev[0], P->stream));
        if (tasks > 0 && launch_odometer(op, Wb, P->num_sms, P->stream))
            return fail(WPM_EINTERNAL, std::string("odometer launch: ") + cudaGetErrorString(cudaGetLastError()));
        CU(cudaEventRecord(P->ev[1], P->stream));
        unsigned long long octl[4], oc[4];
        CU(cudaMemcpyAsync(octl, P->d_out_ctl.p, 32, cudaMemcpyDeviceToHost, P->stream));
        CU(cudaMemcpyAsync(oc, P->d_odo_ctl.p, 32, cudaMemcpyDeviceToHost, P->stream));
        CU(cudaStreamSynchronize(P->stream));
        P->d2h += 64;
        P->total = (long long)octl[0];
        P->leaves = (long long)oc[1];
        P->checked = (long long)oc[2];
        P->nodes = 0;
        P->tasks = tasks;
        if (P->leaves != leaves)
            return fail(WPM_EINTERNAL, "odometer visited " + std::to_string(P->leaves) + " leaves, space is " +
                                           std::to_string(leaves));
        if (octl[0] <= P->out_cap) break;
        P->out_cap = octl[0] + octl[0] / 8 + 1024;
        ++P->reruns;
    }
    const int rc = plan_sort(P);
    if (rc) return rc;
    P->ran = true;
    if (total_out) *total_out = P->total;
    return WPM_OK;
}

// ------------------------------------------------------------------ verification (k8_verify.cu)

namespace {
// pivots P (one facet per usable generator) with G|_P invertible, and the
// inverse's columns: x_i = parity(invcol[i] & y|_P)
bool solve_pivots(const std::vector<uint32_t>& gens, int s, int W32, std::vector<int32_t>* piv,
                  std::vector<unsigned long long>* invcol) {
    std::vector<std::vector<uint32_t>> r(s);
    for (int i = 0; i < s; ++i) r[i].assign(gens.begin() + (long)i * W32, gens.begin() + (long)(i + 1) * W32);
    std::vector<unsigned long long> comb(s);  // which generators each reduced row sums
    for (int i = 0; i < s; ++i) comb[i] = 1ull << i;
    piv->assign(s, -1);
    for (int i = 0; i < s; ++i) {
        int f = -1;
        for (int w = 0; w < W32 && f < 0; ++w)
            if (r[i][w]) f = w * 32 + __builtin_ctz(r[i][w]);
        if (f < 0) return false;  // dependent generators
        (*piv)[i] = f;
        for (int j = 0; j < s; ++j)
            if (j != i && ((r[j][f >> 5] >> (f & 31)) & 1u)) {
                for (int w = 0; w < W32; ++w) r[j][w] ^= r[i][w];
                comb[j] ^= comb[i];
            }
    }
    // reduced row i = sum over comb[i] of g, and has a 1 at pivot i and 0 at
    // every other pivot: y|_P = x A  =>  x_k = sum_i y_{P_i} [k in comb[i]]
    invcol->assign(s, 0ull);
    for (int i = 0; i < s; ++i)
        for (int k = 0; k < s; ++k)
            if ((comb[i] >> k) & 1ull) (*invcol)[k] |= 1ull << i;
    return true;
}
}  // namespace

// Soundness of every row of the last run (the direct WPM test on the device)
// and, with reach != 0, reachability in the reference's combination space:
// coordinates in its usable generators, <= 2 per induced block
// (SURVEY 8(c)(1)-(2)).  coords_out (optional): one uint64 per row, canonical
// order -- bit g = generator g of the block order (wpm_plan_space_blocks).
extern "C" int wpm_plan_verify(wpm_plan_t* P, int32_t reach, int64_t* unsound, int64_t* unreachable,
                               uint64_t* coords_out) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (!P->ran) return fail(WPM_EINVAL, "verify needs a completed run");
    CU(cudaSetDevice(P->device));
    g_alloc_stream = P->stream;
    const int K = P->num_maps;
    std::vector<VerifyMap> vm(K);
    std::vector<uint32_t> words;
    std::vector<int32_t> ints;
    std::vector<unsigned long long> u64s;
    if (reach) {
        const int rc = ensure_spaces(P);
        if (rc) return rc;
    }
    for (int i = 0; i < K; ++i) {
        const MapDesc& d = P->desc[i];
        VerifyMap& v = vm[i];
        v.M = d.M;
        v.N = d.N;
        v.n = d.n;
        v.cap = d.cap;
        v.fs = d.fr_stride;
        v.fr_off = d.fr_off;
        v.s = -1;
        v.nblk = 0;
        if (!reach) continue;
        const CombinationSpaceHost& cs = P->spaces[i];
        int s = 0;
        for (int w : cs.width) s += w;
        if (s > 64) return fail(WPM_EINVAL, "reachability needs at most 64 usable generators");
        std::vector<int32_t> piv;
        std::vector<unsigned long long> inv;
        if (!solve_pivots(cs.gens, s, cs.W32, &piv, &inv)) return fail(WPM_EINTERNAL, "dependent kernel generators");
        v.s = s;
        v.W32 = cs.W32;
        v.gens_off = (uint32_t)words.size();
        words.insert(words.end(), cs.gens.begin(), cs.gens.end());
        v.base_off = (uint32_t)words.size();
        words.insert(words.end(), cs.base.begin(), cs.base.end());
        words.resize(words.size() + 64, 0u);  // rows are read up to w32 words
        v.piv_off = (uint32_t)ints.size();
        ints.insert(ints.end(), piv.begin(), piv.end());
        v.inv_off = (uint32_t)u64s.size();
        u64s.insert(u64s.end(), inv.begin(), inv.end());
        v.blk_off = (uint32_t)u64s.size();
        int lo = 0;
        for (int w : cs.width) {
            if (w >= 2) {
                u64s.push_back((w == 64 ? ~0ull : ((1ull << w) - 1ull)) << lo);
                ++v.nblk;
            }
            lo += w;
        }
    }
    DevBuf<VerifyMap> d_vm;
    DevBuf<uint32_t> d_words;
    DevBuf<int32_t> d_ints;
    DevBuf<unsigned long long> d_u64, d_ctl, d_coords;
    if (d_vm.ensure(K) || d_words.ensure(words.size() + 1) || d_ints.ensure(ints.size() + 1) ||
        d_u64.ensure(u64s.size() + 1) || d_ctl.ensure(4) || d_coords.ensure((size_t)std::max<long long>(P->total, 1)))
        return fail(WPM_EINTERNAL, "device allocation failed (verify)");
    CU(cudaMemcpyAsync(d_vm.p, vm.data(), K * sizeof(VerifyMap), cudaMemcpyHostToDevice, P->stream));
    if (!words.empty())
        CU(cudaMemcpyAsync(d_words.p, words.data(), words.size() * 4, cudaMemcpyHostToDevice, P->stream));
    if (!ints.empty()) CU(cudaMemcpyAsync(d_ints.p, ints.data(), ints.size() * 4, cudaMemcpyHostToDevice, P->stream));
    if (!u64s.empty())
        CU(cudaMemcpyAsync(d_u64.p, u64s.data(), u64s.size() * 8, cudaMemcpyHostToDevice, P->stream));
    CU(cudaMemsetAsync(d_ctl.p, 0, 32, P->stream));
    VerifyParams vp{};
    vp.maps = d_vm.p;
    vp.fr = P->d_fr.p;
    vp.words = d_words.p;
    vp.ints = d_ints.p;
    vp.u64s = d_u64.p;
    vp.rows = P->d_sorted_bits.p;
    vp.row_map = P->d_sorted_map.p;
    vp.count = P->total;
    vp.w32 = P->w32;
    vp.cnt_words = (P->maxN + 3) / 4 + 1;
    vp.reach = reach ? 1 : 0;
    vp.coords = d_coords.p;
    vp.flags = nullptr;
    vp.ctl = d_ctl.p;
    if (launch_k8_verify(vp, P->num_sms, P->stream))
        return fail(WPM_EINTERNAL, std::string("verify launch: ") + cudaGetErrorString(cudaGetLastError()));
    unsigned long long ctl[4];
    CU(cudaMemcpyAsync(ctl, d_ctl.p, 32, cudaMemcpyDeviceToHost, P->stream));
    if (coords_out && P->total > 0)
        CU(cudaMemcpyAsync(coords_out, d_coords.p, (size_t)P->total * 8, cudaMemcpyDeviceToHost, P->stream));
    CU(cudaStreamSynchronize(P->stream));
    if (unsound) *unsound = (int64_t)ctl[0];
    if (unreachable) *unreachable = reach ? (int64_t)(ctl[1] + ctl[2]) : -1;
    return WPM_OK;
}

extern "C" int wpm_plan_kernel_basis_stats(const wpm_plan_t* P, int64_t* leaves, int64_t* checked, double* ms_prep,
                                           double* ms_leaves) {
    if (!P) return fail(WPM_EINVAL, "null plan");
    if (leaves) *leaves = P->leaves;
    if (checked) *checked = P->checked;
    if (ms_prep) *ms_prep = P->ms_prep;
    if (ms_leaves) *ms_leaves = P->ms_search;
    return WPM_OK;
}

extern "C" int wpm_plan_combination_space(const wpm_plan_t* P, int32_t map, uint64_t* space, int32_t* s,
                                          int32_t* blocks) {
    if (!P || map < 0 || map >= P->num_maps || (int)P->spaces.size() != P->num_maps)
        return fail(WPM_EINVAL, "no combination space (run wpm_plan_run_kernel_basis first)");
    const CombinationSpaceHost& cs = P->spaces[map];
    if (space) *space = cs.space;
    if (s) *s = cs.s;
    if (blocks) *blocks = cs.induced_blocks;
    return WPM_OK;
}
