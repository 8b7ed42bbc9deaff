// k4_canon.cu -- canonical order of the emitted WPMs: one persistent
// merge-sort kernel (cooperative launch, grid-wide barriers between passes).
//
// Replaces the merge + sort + unique of enumerate_wpm (search.hpp:247-257):
// complexes are ordered by their facet lists (std::vector<VertexSet>
// operator<, facets ascending), i.e. lexicographically on the ascending
// facet-index lists with a proper prefix first.  On characteristic bitsets
// that is decided at d = the lowest facet in exactly one of A, B: the list
// holding d is smaller unless the other list ends before d.
//
// Records are what kernel 3 emits: w32 bitset words, zero padding, the map
// id in the last word -- rw = rec_words(w32), a multiple of 4 (16-byte
// vectors move them) -- ordered by (map, canonical order).
// A prefix of the facet list does not bound the work (rows of one map share
// long prefixes: 8-facet prefixes still tie up to 1,260 rows at n = 11), so
// the sort compares whole records:
//   phase 1  every CTA sorts tiles of T records in shared memory (bitonic
//            network over record indices; the records stay put);
//   phase 2  merge passes, runs of T, 2T, 4T, ...: each CTA owns chunks of C
//            output records, finds its input ranges by merge-path binary
//            searches on the L2-resident records, stages them in shared
//            memory and merges (every thread a merge-path diagonal);
//   phase 3  the C-ABI split: rows (w32 words) + map ids, the first row of
//            each map, adjacent duplicates counted (the DFS partitions the
//            space, so 0 -- a checked invariant, not a dedupe).
// One launch per sort; passes are separated by grid.sync().
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "wpm_internal.h"

namespace cg = cooperative_groups;

namespace wpm {

namespace {

constexpr int SORT_THREADS = 512;

struct SortParams {
    const uint32_t* in;    // count * rw records (kernel-3 output)
    uint32_t* buf0;        // ping-pong record buffers (buf0 may alias nothing)
    uint32_t* buf1;
    long long count;                      // rows, or the cap of *count_dev
    const unsigned long long* count_dev;  // optional: the row count on the device
    int w32, rw;
    int ow;                // words per output row (>= w32; zero beyond w32)
    int tile;              // records per phase-1 tile (power of two)
    int chunk;             // output records per merge chunk (<= tile)
    uint32_t* out_bits;    // count * w32
    uint16_t* out_map;
    long long* first_row;  // per map (may be null)
    unsigned long long* dups;
    int tie;               // >= 0: a payload word that breaks ties (a total order over equal rows)
    uint32_t* out_payload; // optional: that payload word of every sorted record
};

// canonical record order: map, then the facet-list order on the bitsets
__device__ __forceinline__ bool rec_less(const uint32_t* A, const uint32_t* B, int w32, int mp, int tie) {
    const uint32_t ma = A[mp], mb = B[mp];  // the map id (the record's last word)
    if (ma != mb) return ma < mb;
    for (int w = 0; w < w32; ++w) {
        const uint32_t a = A[w], b = B[w];
        const uint32_t x = a ^ b;
        if (!x) continue;
        const uint32_t low = x & (0u - x);
        const bool a_has = (a & low) != 0u;
        const uint32_t* O = a_has ? B : A;
        bool more = (O[w] & ~((low << 1) - 1u)) != 0u;
        for (int v = w + 1; v < w32 && !more; ++v) more = O[v] != 0u;
        return a_has ? more : !more;
    }
    return tie >= 0 && A[tie] < B[tie];
}

// copy nw words (a multiple of 4; 16-byte aligned) global -> shared in
// 16-byte vectors, four loads in flight per thread
__device__ __forceinline__ void stage16(uint32_t* dst, const uint32_t* src, long long nw) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint4* s = reinterpret_cast<const uint4*>(src);
    const long long nv = nw >> 2;
    const int bd = blockDim.x;
    long long i = threadIdx.x;
    for (; i + 3 * bd < nv; i += 4 * bd) {
        const uint4 a = __ldcg(s + i), b = __ldcg(s + i + bd), c = __ldcg(s + i + 2 * bd), e = __ldcg(s + i + 3 * bd);
        d[i] = a;
        d[i + bd] = b;
        d[i + 2 * bd] = c;
        d[i + 3 * bd] = e;
    }
    for (; i < nv; i += bd) d[i] = __ldcg(s + i);
}

// merge-path split of diagonal d between sorted A[0..na) and B[0..nb):
// the number of A elements among the first d outputs (A wins ties)
__device__ __forceinline__ long long merge_split(const uint32_t* A, long long na, const uint32_t* B, long long nb,
                                                 long long d, int w32, int rw, int tie) {
    long long lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
    while (lo < hi) {
        const long long a = (lo + hi) >> 1;  // take a from A, d - a from B
        // A[a] vs B[d - a - 1]: if B[d-a-1] < A[a] then fewer A needed
        if (rec_less(B + (size_t)(d - a - 1) * rw, A + (size_t)a * rw, w32, rw - 1, tie)) hi = a;
        else lo = a + 1;
    }
    return lo;
}

// the same split searched by a whole warp: 32 probes per round (a 33-ary
// search), so a merge-path search over L2-resident runs costs log33 rounds
// of dependent loads instead of log2
__device__ __forceinline__ long long merge_split_warp(const uint32_t* A, long long na, const uint32_t* B, long long nb,
                                                      long long d, int w32, int rw, int tie, int lane) {
    long long lo = d > nb ? d - nb : 0, hi = d < na ? d : na;  // answer in [lo, hi]
    while (hi - lo > 0) {
        const long long span = hi - lo;
        // probe a_i = lo + (i + 1) * span / 33 for lanes i < 32 (distinct once span >= 33)
        const long long a = lo + ((long long)(lane + 1) * span) / 33;
        bool pred = true;  // pred(a): B[d-a-1] < A[a]  (monotone in a)
        if (a < hi) pred = rec_less(B + (size_t)(d - a - 1) * rw, A + (size_t)a * rw, w32, rw - 1, tie);
        const unsigned t = __ballot_sync(0xFFFFFFFFu, pred);
        const int f = t ? __ffs(t) - 1 : 32;
        // the answer lies in (a_{f-1}, a_f]: a_{-1} = lo - 1, a_32 = hi
        const long long nlo = f == 0 ? lo : lo + ((long long)f * span) / 33 + 1;
        const long long nhi = f == 32 ? hi : lo + ((long long)(f + 1) * span) / 33;
        lo = nlo;
        hi = nhi;
    }
    return lo;
}

__global__ void __launch_bounds__(SORT_THREADS, 2) k4_sort(const __grid_constant__ SortParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    cg::grid_group grid = cg::this_grid();
    const int T = p.tile, rw = p.rw, w32 = p.w32;
    const long long N = p.count_dev ? min((long long)*p.count_dev, p.count) : p.count;
    uint32_t* recs = sm;                                       // T records
    uint16_t* idx = reinterpret_cast<uint16_t*>(sm + (size_t)T * rw);  // T indices (bitonic)
    const long long ntiles = (N + T - 1) / T;
    // ---- phase 1: sort tiles of T records (in -> buf0)
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const long long base = tile * T;
        const int cnt = (int)min((long long)T, N - base);
        stage16(recs, p.in + (size_t)base * rw, (long long)cnt * rw);
        for (int i = threadIdx.x; i < T; i += blockDim.x) idx[i] = (uint16_t)i;
        __syncthreads();
        for (int k = 2; k <= T; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < T; i += blockDim.x) {
                    const int l = i ^ j;
                    if (l > i) {
                        const int a = idx[i], b = idx[l];
                        // indices >= cnt are +inf padding
                        const bool b_lt_a = a >= cnt ? b < cnt || b < a
                                                     : (b < cnt && rec_less(recs + (size_t)b * rw, recs + (size_t)a * rw, w32, rw - 1, p.tie));
                        const bool up = (i & k) == 0;
                        if (up == b_lt_a) {
                            idx[i] = (uint16_t)b;
                            idx[l] = (uint16_t)a;
                        }
                    }
                }
                __syncthreads();
            }
        uint4* dst = reinterpret_cast<uint4*>(p.buf0 + (size_t)base * rw);
        const int rv = rw >> 2;
        for (int i = threadIdx.x; i < cnt * rv; i += blockDim.x) {
            const int r = i / rv, c = i - r * rv;
            dst[i] = reinterpret_cast<const uint4*>(recs + (size_t)idx[r] * rw)[c];
        }
        __syncthreads();
    }
    grid.sync();
    // ---- phase 2: merge passes (runs of L -> 2L), C = T output records per chunk
    const uint32_t* src = p.buf0;
    uint32_t* dst = p.buf1;
    __shared__ long long s_rng[4];
    const int C = p.chunk;
    for (long long L = T; L < N; L <<= 1) {
        const long long nchunks = (N + C - 1) / C;
        for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
            const long long o0 = c * C, o1 = min(N, o0 + C);
            const long long run = o0 / (2 * L), rbase = run * 2 * L;
            const long long na = min(L, N - rbase), nb = max(0ll, min(L, N - rbase - L));
            const uint32_t* A = src + (size_t)rbase * rw;
            const uint32_t* B = A + (size_t)na * rw;
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            if (warp < 2) {
                const long long r = merge_split_warp(A, na, B, nb, (warp ? o1 : o0) - rbase, w32, rw, p.tie, lane);
                if (lane == 0) s_rng[warp] = r;
            }
            __syncthreads();
            const long long a0 = s_rng[0], a1 = s_rng[1];
            const long long b0 = (o0 - rbase) - a0, b1 = (o1 - rbase) - a1;
            const int ca = (int)(a1 - a0), cb = (int)(b1 - b0);
            // stage A[a0..a1) then B[b0..b1) in shared memory
            stage16(recs, A + (size_t)a0 * rw, (long long)ca * rw);
            stage16(recs + (size_t)ca * rw, B + (size_t)b0 * rw, (long long)cb * rw);
            __syncthreads();
            const uint32_t* SA = recs;
            const uint32_t* SB = recs + (size_t)ca * rw;
            const int total = ca + cb;
            const int per = (total + blockDim.x - 1) / blockDim.x;
            const int d0 = min(total, (int)threadIdx.x * per), d1 = min(total, d0 + per);
            if (d0 < d1) {  // each thread: its merge-path diagonal, then `per` sources
                int ia = (int)merge_split(SA, ca, SB, cb, d0, w32, rw, p.tie);
                int ib = d0 - ia;
                for (int d = d0; d < d1; ++d) {
                    const bool take_a = ib >= cb || (ia < ca && !rec_less(SB + (size_t)ib * rw, SA + (size_t)ia * rw, w32, rw - 1, p.tie));
                    idx[d] = (uint16_t)(take_a ? ia++ : ca + ib++);
                }
            }
            __syncthreads();
            // coalesced write of the merged chunk
            uint4* out = reinterpret_cast<uint4*>(dst + (size_t)o0 * rw);
            const int rv = rw >> 2;
            for (int i = threadIdx.x; i < total * rv; i += blockDim.x) {
                const int r = i / rv, c = i - r * rv;
                out[i] = reinterpret_cast<const uint4*>(recs + (size_t)idx[r] * rw)[c];
            }
            __syncthreads();
        }
        grid.sync();
        const uint32_t* t = src;
        src = dst;
        dst = const_cast<uint32_t*>(t);
    }
    // ---- phase 3: the C-ABI layout, group boundaries, duplicates
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int ow = p.ow;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N * ow; i += stride) {
        const long long r = i / ow, c = i - r * ow;
        p.out_bits[i] = c < w32 ? src[(size_t)r * rw + c] : 0u;
    }
    unsigned long long nd = 0;
    for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < N; r += stride) {
        const uint32_t* R = src + (size_t)r * rw;
        const uint32_t* Q = R - rw;  // the previous record (r > 0)
        if (p.out_map) p.out_map[r] = (uint16_t)R[rw - 1];
        if (p.out_payload) p.out_payload[r] = R[p.tie];
        if (r == 0 || Q[rw - 1] != R[rw - 1]) {
            if (p.first_row) p.first_row[R[rw - 1]] = r;
        } else {
            bool same = true;
            for (int i = 0; i < w32; ++i) same &= R[i] == Q[i];
            nd += same;
        }
    }
    if (nd && p.dups) atomicAdd(p.dups, nd);
}

int g_sort_sms[64] = {0};

}  // namespace

int key_words_for(int w32) { return w32 >= 1 && w32 <= 64 ? w32 : -1; }

// temp = the two ping-pong record buffers (the input stays intact)
size_t canon_sort_temp_bytes(long long count, int w32) {
    return (size_t)2 * (size_t)count * (size_t)rec_words(w32) * 4 + 256;
}

int canon_sort_keys(uint32_t* d_keys, long long count, int w32, uint32_t* d_sorted_bits, uint16_t* d_sorted_map,
                    void* d_temp, size_t temp_bytes, long long* d_first_row, unsigned long long* d_dups,
                    cudaStream_t st, const unsigned long long* d_count, long long grid_rows, int out_words) {
    return canon_sort_records(d_keys, count, w32, rec_words(w32), -1, d_sorted_bits, d_sorted_map, nullptr, d_temp,
                              temp_bytes, d_first_row, d_dups, st, d_count, grid_rows, out_words);
}

int canon_sort_records(uint32_t* d_keys, long long count, int w32, int rw, int tie, uint32_t* d_sorted_bits,
                       uint16_t* d_sorted_map, uint32_t* d_payload, void* d_temp, size_t temp_bytes,
                       long long* d_first_row, unsigned long long* d_dups, cudaStream_t st,
                       const unsigned long long* d_count, long long grid_rows, int out_words) {
    if (count <= 0) return 0;
    if (out_words <= 0) out_words = w32;
    if (out_words < w32) return 1;
    if (rw % 4 || rw < w32 + 1) return 1;
    if (temp_bytes < (size_t)2 * (size_t)count * (size_t)rw * 4) return 1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 1;
    if (!g_sort_sms[dev] && cudaDeviceGetAttribute(&g_sort_sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 1;
    // tile = chunk = the largest power of two <= 2048 that still gives every
    // SM a tile (N / SMs) and keeps a tile's records <= 100 KB of shared
    // memory (two CTAs per SM).  Swept 256-4096 at n = 4, 5, 6, 8, 11: the best
    // tile follows the row count (n = 4: 256, n = 5: 1024, n = 6 / 8: 2048)
    // and the record width (n = 11, 128-byte records: 256-512).
    const long long rows_hint = grid_rows > 0 ? std::min(grid_rows, count) : count;
    int T = 2048;
    while (T > 128 && ((long long)T > rows_hint / g_sort_sms[dev] || (size_t)T * rw * 4 > 100u * 1024u)) T >>= 1;
    if (const char* e = std::getenv("WPM_SORT_TILE")) {
        T = std::max(64, std::atoi(e));
        while (T > 64 && (size_t)T * rw * 4 + (size_t)T * 2 > 200u * 1024u) T >>= 1;
    }
    int Cc = T;
    if (const char* e = std::getenv("WPM_SORT_CHUNK")) Cc = std::max(32, std::min(T, std::atoi(e)));
    const size_t smem = (size_t)T * rw * 4 + (size_t)T * 2 + 16;
    if (cudaFuncSetAttribute(k4_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_sort, SORT_THREADS, smem) != cudaSuccess || per_sm < 1)
        return 1;
    // the kernel strides over its tiles / chunks, so any grid is correct; size
    // it for the expected rows (fewer idle CTAs in every grid barrier)
    const long long rows_for_grid = grid_rows > 0 ? std::min(grid_rows, count) : count;
    const long long work = std::max((rows_for_grid + T - 1) / T, (rows_for_grid + Cc - 1) / Cc);
    const int grid = (int)std::min<long long>(work, (long long)per_sm * g_sort_sms[dev]);
    SortParams sp{};
    sp.in = d_keys;
    sp.buf0 = static_cast<uint32_t*>(d_temp);
    sp.buf1 = sp.buf0 + (size_t)count * rw;
    sp.count = count;
    sp.count_dev = d_count;
    sp.w32 = w32;
    sp.rw = rw;
    sp.ow = out_words;
    sp.tile = T;
    sp.chunk = Cc;
    sp.out_bits = d_sorted_bits;
    sp.out_map = d_sorted_map;
    sp.first_row = d_first_row;
    sp.dups = d_dups;
    sp.tie = tie;
    sp.out_payload = d_payload;
    void* args[] = {&sp};
    if (cudaLaunchCooperativeKernel((const void*)k4_sort, dim3(grid), dim3(SORT_THREADS), args, smem, st) != cudaSuccess)
        return 1;
    return 0;
}

__global__ void pack_records(const uint32_t* __restrict__ bits, const uint16_t* __restrict__ map, long long n, int w32,
                             uint32_t* __restrict__ recs) {
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const int rw = rec_words(w32);
    uint32_t* r = recs + (size_t)row * rw;
    for (int i = 0; i < rw - 1; ++i) r[i] = i < w32 ? bits[(size_t)row * w32 + i] : 0u;
    r[rw - 1] = map[row];
}

int canon_pack(const uint32_t* d_bits, const uint16_t* d_map, long long count, int w32, uint32_t* d_keys,
               cudaStream_t st) {
    if (count <= 0) return 0;
    pack_records<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d_bits, d_map, count, w32, d_keys);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace wpm
