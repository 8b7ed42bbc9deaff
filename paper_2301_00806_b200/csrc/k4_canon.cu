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

// bitonic network over the indices of cnt staged records (padded to a power
// of two; indices >= cnt sort last): idx[0..cnt) ends in record order.  A
// compare-exchange at distance j < 32 stays inside one warp (thread t owns
// elements t + m * blockDim, blockDim a multiple of 32), so only the stages
// at j >= 32 and the ones next to them need the CTA barrier -- 10 of the 55
// stages of a 1024-record tile.  Ends with a CTA barrier.
__device__ __forceinline__ void bitonic_idx(const uint32_t* recs, uint16_t* idx, int cnt, int w32, int rw, int tie) {
    int P2 = 1;
    while (P2 < cnt) P2 <<= 1;
    for (int i = threadIdx.x; i < P2; i += blockDim.x) idx[i] = (uint16_t)i;
    __syncthreads();
    for (int k = 2; k <= P2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const int a = idx[i], b = idx[l];
                    const bool b_lt_a = a >= cnt ? b < cnt || b < a
                                                 : (b < cnt && rec_less(recs + (size_t)b * rw, recs + (size_t)a * rw, w32, rw - 1, tie));
                    if (((i & k) == 0) == b_lt_a) {
                        idx[i] = (uint16_t)b;
                        idx[l] = (uint16_t)a;
                    }
                }
            }
            const int next_j = j > 1 ? j >> 1 : (2 * k <= P2 ? k : 0);
            if (j >= 32 || next_j >= 32) __syncthreads();
            else __syncwarp();
        }
    __syncthreads();
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
        __syncthreads();
        bitonic_idx(recs, idx, cnt, w32, rw, p.tie);
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

// ---- the bucketed sort (the plan's sort of kernel-3 rows).  Every row's
// first facets decide its place among most others: with f0 < f1 < f2 its
// three lowest facets, the canonical order is (map, f0, f1, f2, the rest), so
// rows are counted and scattered into buckets (map, f0, s1, s2) --
// s1 = min(f1 - f0 - 1, 7), s2 = min(f2 - f1 - 1, 7) when s1 < 7, else 0 --
// whose order is the canonical order, and only rows of one bucket still
// need comparing.  The buckets are sorted where they lie: a window of T/2
// output positions owns the buckets that start in it; consecutive buckets
// of <= T rows in all are sorted together in shared memory (bitonic) and
// written out in the C-ABI layout; a bucket of > T rows is sorted by its CTA
// alone (tiles, then merge passes through global memory).
constexpr int BK_PER_FACET = 64;

struct BucketParams {
    const uint32_t* in;                   // kernel-3 records
    long long cap;
    const unsigned long long* count_dev;  // rows on the device (<= cap)
    int w32, rw, ow;
    const MapDesc* maps;
    int num_maps;
    long long B;                          // buckets (BK_PER_FACET per facet of all maps)
    uint32_t* bid;                        // cap: bucket of each input row
    uint32_t* cnt;                        // B: zero on entry, zeroed again on exit
    uint32_t* off;                        // B + 1
    uint32_t* cur;                        // B: scatter cursors
    uint32_t* bsum;                       // gridDim.x
    uint32_t* buf;                        // cap * rw: rows in bucket order
    uint32_t* tmp;                        // cap * rw: merge ping-pong (big buckets)
    int tile;                             // T: rows sorted at once in shared memory
    uint32_t* out_bits;
    uint16_t* out_map;
    long long* first_row;
    unsigned long long* dups;
    int stop;                             // experiment: leave after this phase (0 = run all)
};

__device__ __forceinline__ uint32_t bucket_of(const uint32_t* R, int w32, int rw, const MapDesc* maps) {
    const uint32_t map = R[rw - 1];
    int f[3] = {0, -1, -1};
    int k = 0;
    for (int w = 0; w < w32 && k < 3; ++w) {
        uint32_t x = R[w];
        while (x && k < 3) {
            f[k++] = w * 32 + __ffs(x) - 1;
            x &= x - 1u;
        }
    }
    int s1 = 0, s2 = 0;
    if (f[1] >= 0) {
        s1 = min(f[1] - f[0] - 1, 7);
        if (s1 < 7 && f[2] >= 0) s2 = min(f[2] - f[1] - 1, 7);
    }
    return (maps[map].facet_off + (uint32_t)f[0]) * BK_PER_FACET + (uint32_t)(s1 * 8 + s2);
}

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    uint32_t t = 0;
    for (int i = 0; i < nw; ++i) t += red[i];
    return t;
}

// bitonic sort of cnt (<= T) staged records by index (idx[0..cnt) sorted)
__device__ __forceinline__ void tile_bitonic(const uint32_t* recs, uint16_t* idx, int cnt, int w32, int rw) {
    bitonic_idx(recs, idx, cnt, w32, rw, -1);
}

__device__ __forceinline__ bool same_bits(const uint32_t* A, const uint32_t* B, int w32) {
    bool same = true;
    for (int i = 0; i < w32; ++i) same &= A[i] == B[i];
    return same;
}

// rows idx[0..cnt) of the staged records -> output rows at `at` (C-ABI
// layout); adjacent equal rows counted (prev: the row before `at` in this
// bucket, or null)
__device__ __forceinline__ unsigned long long write_out(const BucketParams& p, const uint32_t* recs, const uint16_t* idx,
                                                        int cnt, long long at, const uint32_t* prev) {
    const int w32 = p.w32, rw = p.rw, ow = p.ow;
    for (int i = threadIdx.x; i < cnt * ow; i += blockDim.x) {
        const int r = i / ow, c = i - r * ow;
        p.out_bits[(size_t)at * ow + i] = c < w32 ? recs[(size_t)idx[r] * rw + c] : 0u;
    }
    unsigned long long nd = 0;
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
        const uint32_t* R = recs + (size_t)idx[r] * rw;
        p.out_map[at + r] = (uint16_t)R[rw - 1];
        if (r > 0) nd += same_bits(R, recs + (size_t)idx[r - 1] * rw, w32);
        else if (prev) nd += same_bits(R, prev, w32);
    }
    return nd;
}

// one bucket of > T rows [bs, be), sorted by this CTA alone from its
// bucket-order rows in buf: tiles of T into tmp, then merge passes (buf and
// tmp of this range as ping-pong), the last one writing the C-ABI rows
__device__ unsigned long long big_bucket(const BucketParams& p, long long bs, long long be, uint32_t* recs,
                                         uint16_t* idx, long long* s_w) {
    const int T = p.tile, rw = p.rw, w32 = p.w32;
    const long long sz = be - bs;
    unsigned long long nd = 0;
    for (long long t0 = bs; t0 < be; t0 += T) {
        const int cnt = (int)min((long long)T, be - t0);
        stage16(recs, p.buf + (size_t)t0 * rw, (long long)cnt * rw);
        __syncthreads();
        tile_bitonic(recs, idx, cnt, w32, rw);
        uint4* dst = reinterpret_cast<uint4*>(p.tmp + (size_t)t0 * rw);
        const int rv = rw >> 2;
        for (int i = threadIdx.x; i < cnt * rv; i += blockDim.x) {
            const int r = i / rv, c = i - r * rv;
            dst[i] = reinterpret_cast<const uint4*>(recs + (size_t)idx[r] * rw)[c];
        }
        __syncthreads();
    }
    const uint32_t* src = p.tmp;
    uint32_t* dstb = p.buf;
    for (long long L = T; L < sz; L <<= 1) {
        const bool last = 2 * L >= sz;
        for (long long rs = bs; rs < be; rs += 2 * L) {
            const long long na = min(L, be - rs), nb = max(0ll, min(L, be - rs - L));
            const uint32_t* A = src + (size_t)rs * rw;
            const uint32_t* Bp = A + (size_t)na * rw;
            for (long long o0 = 0; o0 < na + nb; o0 += T) {
                const long long o1 = min(na + nb, o0 + T);
                const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
                if (warp < 2) {
                    const long long r = merge_split_warp(A, na, Bp, nb, warp ? o1 : o0, w32, rw, -1, lane);
                    if (lane == 0) s_w[warp] = r;
                }
                __syncthreads();
                const long long a0 = s_w[0], a1 = s_w[1], b0 = o0 - a0, b1 = o1 - a1;
                const int ca = (int)(a1 - a0), cb = (int)(b1 - b0);
                stage16(recs, A + (size_t)a0 * rw, (long long)ca * rw);
                stage16(recs + (size_t)ca * rw, Bp + (size_t)b0 * rw, (long long)cb * rw);
                __syncthreads();
                const uint32_t* SA = recs;
                const uint32_t* SB = recs + (size_t)ca * rw;
                const int total = ca + cb;
                const int pt = (total + blockDim.x - 1) / blockDim.x;
                const int d0 = min(total, (int)threadIdx.x * pt), d1 = min(total, d0 + pt);
                if (d0 < d1) {
                    int ia = (int)merge_split(SA, ca, SB, cb, d0, w32, rw, -1);
                    int ib = d0 - ia;
                    for (int d = d0; d < d1; ++d) {
                        const bool take_a = ib >= cb || (ia < ca && !rec_less(SB + (size_t)ib * rw, SA + (size_t)ia * rw, w32, rw - 1, -1));
                        idx[d] = (uint16_t)(take_a ? ia++ : ca + ib++);
                    }
                }
                __syncthreads();
                if (last) {
                    // the previous output row of this bucket (written by this CTA)
                    nd += write_out(p, recs, idx, total, rs + o0, nullptr);
                    if (threadIdx.x == 0 && rs + o0 > bs) {
                        const uint32_t* R = recs + (size_t)idx[0] * rw;
                        const uint32_t* Q = p.out_bits + (size_t)(rs + o0 - 1) * p.ow;
                        nd += same_bits(R, Q, w32);
                    }
                } else {
                    uint4* out = reinterpret_cast<uint4*>(dstb + (size_t)(rs + o0) * rw);
                    const int rv = rw >> 2;
                    for (int i = threadIdx.x; i < total * rv; i += blockDim.x) {
                        const int r = i / rv, c = i - r * rv;
                        out[i] = reinterpret_cast<const uint4*>(recs + (size_t)idx[r] * rw)[c];
                    }
                }
                __syncthreads();
            }
        }
        const uint32_t* t = src;
        src = dstb;
        dstb = const_cast<uint32_t*>(t);
    }
    return nd;
}

__global__ void __launch_bounds__(SORT_THREADS, 2) k4_bucket(const __grid_constant__ BucketParams p) {
    extern __shared__ __align__(16) uint32_t sm[];
    __shared__ uint32_t red[SORT_THREADS / 32];
    __shared__ long long s_w[4];
    cg::grid_group grid = cg::this_grid();
    const int T = p.tile, rw = p.rw, w32 = p.w32;
    const long long N = p.count_dev ? min((long long)*p.count_dev, p.cap) : p.cap;
    const long long B = p.B;
    const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x, gs = (long long)gridDim.x * blockDim.x;
    // ---- 1: bucket of every row, counts
    for (long long i = gt; i < N; i += gs) {
        const uint32_t b = bucket_of(p.in + (size_t)i * rw, w32, rw, p.maps);
        p.bid[i] = b;
        atomicAdd(&p.cnt[b], 1u);
    }
    grid.sync();
    if (p.stop == 1) return;
    // ---- 2: exclusive scan of the counts (a chunk per CTA)
    const long long per = (B + gridDim.x - 1) / gridDim.x;
    const long long c0 = min(B, (long long)blockIdx.x * per), c1 = min(B, c0 + per);
    {
        uint32_t v = 0;
        for (long long j = c0 + threadIdx.x; j < c1; j += blockDim.x) v += p.cnt[j];
        v = block_sum(v, red);
        if (threadIdx.x == 0) p.bsum[blockIdx.x] = v;
    }
    grid.sync();
    {
        uint32_t pre = 0;
        for (int k = threadIdx.x; k < (int)blockIdx.x; k += blockDim.x) pre += p.bsum[k];
        pre = block_sum(pre, red);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (long long base = c0; base < c1; base += blockDim.x) {
            const long long j = base + threadIdx.x;
            const uint32_t v = j < c1 ? p.cnt[j] : 0u;
            uint32_t x = v;  // inclusive warp scan
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= o) x += y;
            }
            __syncthreads();
            if (lane == 31) red[warp] = x;
            __syncthreads();
            uint32_t wpre = 0, tot = 0;
            for (int i = 0; i < nw; ++i) {
                wpre += i < warp ? red[i] : 0u;
                tot += red[i];
            }
            if (j < c1) {
                const uint32_t e = pre + wpre + x - v;
                p.off[j] = e;
                p.cur[j] = e;
            }
            pre += tot;
        }
        if (gt == 0) p.off[B] = (uint32_t)N;
    }
    grid.sync();
    if (p.stop == 2) return;
    // ---- 3: scatter into bucket order; the buckets each window owns; first
    // row of each map; the counts back to zero for the next sort
    for (long long i = gt; i < N; i += gs) {
        const uint32_t pos = atomicAdd(&p.cur[p.bid[i]], 1u);
        const uint4* src = reinterpret_cast<const uint4*>(p.in + (size_t)i * rw);
        uint4* dst = reinterpret_cast<uint4*>(p.buf + (size_t)pos * rw);
        for (int c = 0; c < (rw >> 2); ++c) dst[c] = __ldcg(src + c);
    }
    for (long long j = gt; j < B; j += gs) {
        p.cnt[j] = 0u;
    }
    for (long long q = gt; q < p.num_maps; q += gs) {
        const long long b0 = (long long)p.maps[q].facet_off * BK_PER_FACET, b1 = b0 + (long long)p.maps[q].M * BK_PER_FACET;
        if (p.first_row) p.first_row[q] = p.off[b1] > p.off[b0] ? (long long)p.off[b0] : -1;
    }
    grid.sync();
    if (p.stop == 3) return;
    // ---- 4: tiles of T positions sorted in shared memory.  Only the first
    // and the last bucket of a tile can reach past it; every other row is in
    // its final place and is written out.  Rows of those straddling buckets
    // go to tmp (sorted pieces) for step 5.
    uint32_t* recs = sm;
    uint16_t* idx = reinterpret_cast<uint16_t*>(sm + (size_t)T * rw);
    __shared__ uint32_t s_edge[4];
    unsigned long long nd = 0;
    const long long ntile = (N + T - 1) / T;
    for (long long t = blockIdx.x; t < ntile; t += gridDim.x) {
        const long long t0 = t * T;
        const int cnt = (int)min((long long)T, N - t0);
        stage16(recs, p.buf + (size_t)t0 * rw, (long long)cnt * rw);
        __syncthreads();
        tile_bitonic(recs, idx, cnt, w32, rw);
        if (threadIdx.x == 0) {
            const uint32_t bf = bucket_of(recs + (size_t)idx[0] * rw, w32, rw, p.maps);
            const uint32_t bl = bucket_of(recs + (size_t)idx[cnt - 1] * rw, w32, rw, p.maps);
            s_edge[0] = bf;
            s_edge[1] = bl;
            s_edge[2] = (long long)p.off[bf] < t0;                    // the first bucket started before
            s_edge[3] = (long long)p.off[bl + 1] > t0 + cnt;          // the last one goes on after
        }
        __syncthreads();
        const uint32_t bf = s_edge[0], bl = s_edge[1];
        const bool sf = s_edge[2] != 0u, sl = s_edge[3] != 0u;
        const int ow = p.ow;
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const uint32_t* R = recs + (size_t)idx[i] * rw;
            const uint32_t b = bucket_of(R, w32, rw, p.maps);
            const long long q = t0 + i;
            if ((sf && b == bf) || (sl && b == bl)) {
                uint4* d = reinterpret_cast<uint4*>(p.tmp + (size_t)q * rw);
                for (int c = 0; c < (rw >> 2); ++c) d[c] = reinterpret_cast<const uint4*>(R)[c];
                continue;
            }
            uint32_t* o = p.out_bits + (size_t)q * ow;
            for (int c = 0; c < ow; ++c) o[c] = c < w32 ? R[c] : 0u;
            p.out_map[q] = (uint16_t)R[rw - 1];
            if (i > 0) {
                const uint32_t* Q = recs + (size_t)idx[i - 1] * rw;
                if (bucket_of(Q, w32, rw, p.maps) == b) nd += same_bits(R, Q, w32);
            }
        }
        __syncthreads();
    }
    grid.sync();
    if (p.stop == 4) return;
    // ---- 5: each straddling bucket once, by the CTA of the tile boundary
    // after its start: <= T rows re-sorted whole in shared memory (its
    // sorted pieces from tmp), more by this CTA's merge passes
    for (long long t = 1 + blockIdx.x; t < ntile; t += gridDim.x) {
        const long long x = t * T;
        // the bucket holding position x (buf is in bucket order)
        const uint32_t b = bucket_of(p.buf + (size_t)x * rw, w32, rw, p.maps);
        const long long bs = p.off[b], be = p.off[b + 1];
        if (bs >= x || bs < x - T) continue;  // no straddle here, or not its first boundary
        if (be - bs <= T) {
            const int cnt = (int)(be - bs);
            stage16(recs, p.tmp + (size_t)bs * rw, (long long)cnt * rw);
            __syncthreads();
            tile_bitonic(recs, idx, cnt, w32, rw);
            nd += write_out(p, recs, idx, cnt, bs, nullptr);
            __syncthreads();
        } else {
            nd += big_bucket(p, bs, be, recs, idx, s_w);
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
    const int per_sm = occupancy_cached(reinterpret_cast<const void*>(k4_sort), SORT_THREADS, smem);
    if (per_sm < 1) return 1;
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

// the bucketed sort's scratch (uint32 words) for cap rows of a plan with
// total_facets facets; the count words (B of them, at offset cap) must be
// zero before the first sort -- every sort leaves them zero
size_t bucket_sort_scratch_words(long long cap, long long total_facets) {
    const long long B = total_facets * BK_PER_FACET;
    return (size_t)(cap + 3 * B + 1 + 1024 + 16);
}
size_t bucket_sort_count_offset(long long cap) { return (size_t)cap; }

int canon_sort_bucketed(const uint32_t* d_keys, long long cap, const unsigned long long* d_count, int w32, int rw,
                        int out_words, const MapDesc* d_maps, int num_maps, long long total_facets,
                        uint32_t* d_sorted_bits, uint16_t* d_sorted_map, long long* d_first_row,
                        unsigned long long* d_dups, void* d_temp, size_t temp_bytes, uint32_t* d_scratch,
                        size_t scratch_words, cudaStream_t st, long long grid_rows) {
    if (cap <= 0) return 0;
    if (rw % 4 || rw < w32 + 1 || out_words < w32) return 1;
    if (temp_bytes < (size_t)2 * (size_t)cap * (size_t)rw * 4) return 1;
    if (scratch_words < bucket_sort_scratch_words(cap, total_facets)) return 1;
    const long long B = total_facets * BK_PER_FACET;
    if (B >= 0xFFFFFFFFll || cap >= 0xFFFFFFFFll) return 1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 1;
    if (!g_sort_sms[dev] && cudaDeviceGetAttribute(&g_sort_sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 1;
    // T: the largest power of two <= 4096 whose records fit ~100 KB of
    // shared memory (two CTAs per SM)
    const size_t extra = 16;
    int T = 4096;
    while (T > 64 && (size_t)T * rw * 4 + (size_t)T * 2 + extra > 100u * 1024u) T >>= 1;
    if (const char* e = std::getenv("WPM_BUCKET_TILE")) T = std::max(64, std::min(T, std::atoi(e)));
    const size_t smem = (size_t)T * rw * 4 + (size_t)T * 2 + extra;
    if (cudaFuncSetAttribute(k4_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k4_bucket, SORT_THREADS, smem) != cudaSuccess || per_sm < 1)
        return 1;
    const long long rows = grid_rows > 0 ? std::min(grid_rows, cap) : cap;
    const long long work = std::max<long long>(1, (rows + T - 1) / T);
    int grid = (int)std::min<long long>(std::min<long long>(work, 1024), (long long)per_sm * g_sort_sms[dev]);
    if (std::getenv("WPM_BUCKET_FULLGRID")) grid = per_sm * g_sort_sms[dev];
    BucketParams bp{};
    bp.in = d_keys;
    bp.cap = cap;
    bp.count_dev = d_count;
    bp.w32 = w32;
    bp.rw = rw;
    bp.ow = out_words;
    bp.maps = d_maps;
    bp.num_maps = num_maps;
    bp.B = B;
    uint32_t* q = d_scratch;
    bp.bid = q;
    q += cap;
    bp.cnt = q;
    q += B;
    bp.off = q;
    q += B + 1;
    bp.cur = q;
    q += B;
    bp.bsum = q;
    bp.buf = static_cast<uint32_t*>(d_temp);
    bp.tmp = bp.buf + (size_t)cap * rw;
    bp.tile = T;
    bp.out_bits = d_sorted_bits;
    bp.out_map = d_sorted_map;
    bp.first_row = d_first_row;
    bp.dups = d_dups;
    if (const char* e = std::getenv("WPM_BUCKET_STOP")) bp.stop = std::atoi(e);
    void* args[] = {&bp};
    if (cudaLaunchCooperativeKernel((const void*)k4_bucket, dim3(grid), dim3(SORT_THREADS), args, smem, st) != cudaSuccess)
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
