// k4_canon.cu -- canonical order of the emitted WPMs.
//
// Replaces the merge + sort + unique of enumerate_wpm (search.hpp:247-257):
// complexes are ordered by their facet lists (std::vector<VertexSet>
// operator<, facets ascending), i.e. lexicographically on the ascending
// facet-index lists with a proper prefix first.  On characteristic bitsets
// that is decided at d = the lowest facet in exactly one of A, B: the list
// holding d is smaller unless the other list ends before d.
//
// Kernel 3 emits each WPM as a fixed-width key row -- W uint32 words of the
// characteristic bitset (zero padded, W a bucket >= the plan's width)
// followed by the map id.  Narrow rows (W <= 4, M <= 128, i.e. n <= 5) are
// merge-sorted (CUB) as keys themselves: no indirection, comparisons in
// registers.  W is the exact word count there (n = 5 has M <= 88: 16-byte
// keys instead of 20).  Wider rows merge-sort row indices instead, the comparator
// reading the rows from L2 (moving 36-132 B keys through every merge pass
// measured 2-4x slower).  A split/gather pass then writes the canonical rows
// (the C-ABI width) and map ids, records per-map group boundaries and counts
// adjacent duplicates (the DFS partitions the space, so the count is 0 -- a
// checked invariant, not a dedupe).
#include <cub/device/device_merge_sort.cuh>

#include <cstdint>

#include "wpm_internal.h"

namespace wpm {

template <int W>
struct RowKey {
    uint32_t w[W];
    uint32_t map;
};

template <int W>
struct RowLess {
    __device__ __forceinline__ bool operator()(const RowKey<W>& A, const RowKey<W>& B) const {
        if (A.map != B.map) return A.map < B.map;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t x = A.w[i] ^ B.w[i];
            if (!x) continue;
            const uint32_t low = x & (0u - x);
            const bool a_has = (A.w[i] & low) != 0u;
            const RowKey<W>& O = a_has ? B : A;
            bool more = (O.w[i] & ~((low << 1) - 1u)) != 0u;
#pragma unroll
            for (int v = i + 1; v < W; ++v) more |= O.w[v] != 0u;
            return a_has ? more : !more;
        }
        return false;
    }
};

// split the sorted key rows into the C-ABI layout: rows of w32 words + map ids;
// group boundaries (first row per map) and adjacent-duplicate count
template <int W>
__global__ void split_rows(const RowKey<W>* __restrict__ keys, long long n, int w32, uint32_t* __restrict__ out,
                           uint16_t* __restrict__ out_map, unsigned long long* dups, long long* __restrict__ first_row) {
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    const RowKey<W>& k = keys[row];
    for (int i = 0; i < w32; ++i) out[(size_t)row * w32 + i] = k.w[i];
    out_map[row] = (uint16_t)k.map;
    if (row == 0 || keys[row - 1].map != k.map) {
        if (first_row) first_row[k.map] = row;
    } else {
        bool same = true;
        const RowKey<W>& p = keys[row - 1];
#pragma unroll
        for (int i = 0; i < W; ++i) same &= p.w[i] == k.w[i];
        if (same) atomicAdd(dups, 1ull);
    }
}

// pack externally supplied rows (w32 words + uint16 map ids) into key rows
template <int W>
__global__ void pack_rows(const uint32_t* __restrict__ bits, const uint16_t* __restrict__ map, long long n, int w32,
                          RowKey<W>* __restrict__ keys) {
    const long long row = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    RowKey<W> k;
#pragma unroll
    for (int i = 0; i < W; ++i) k.w[i] = i < w32 ? bits[(size_t)row * w32 + i] : 0u;
    k.map = map[row];
    keys[row] = k;
}

// ---- wide rows: merge-sort row indices instead (moving > 20-byte keys costs
// more than the comparator's L2 reads); the comparator reads the key rows
struct IdxLess {
    const uint32_t* keys;
    int rw, w32;
    __device__ __forceinline__ bool operator()(const uint32_t& a, const uint32_t& b) const {
        const uint32_t* A = keys + (size_t)a * rw;
        const uint32_t* B = keys + (size_t)b * rw;
        const uint32_t ma = A[rw - 1], mb = B[rw - 1];
        if (ma != mb) return ma < mb;
        for (int w = 0; w < w32; ++w) {
            const uint32_t x = A[w] ^ B[w];
            if (!x) continue;
            const uint32_t low = x & (0u - x);
            const bool a_has = (A[w] & low) != 0u;
            const uint32_t* O = a_has ? B : A;
            bool more = (O[w] & ~((low << 1) - 1u)) != 0u;
            for (int v = w + 1; v < w32 && !more; ++v) more = O[v] != 0u;
            return a_has ? more : !more;
        }
        return false;
    }
};

__global__ void iota_u32(uint32_t* idx, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) idx[i] = (uint32_t)i;
}

__global__ void gather_rows(const uint32_t* __restrict__ keys, int rw, const uint32_t* __restrict__ idx, long long n,
                            int w32, uint32_t* __restrict__ out, uint16_t* __restrict__ out_map,
                            unsigned long long* dups, long long* __restrict__ first_row) {
    // one warp per row
    const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const uint32_t* S = keys + (size_t)idx[row] * rw;
    const uint32_t* P = row > 0 ? keys + (size_t)idx[row - 1] * rw : S;
    const bool new_group = row == 0 || P[rw - 1] != S[rw - 1];
    if (lane == 0 && new_group && first_row) first_row[S[rw - 1]] = row;
    bool same = !new_group;
    for (int w = lane; w < w32; w += 32) {
        const uint32_t v = S[w];
        out[(size_t)row * w32 + w] = v;
        if (P[w] != v) same = false;
    }
    same = __all_sync(0xFFFFFFFFu, same);
    if (lane == 0) {
        out_map[row] = (uint16_t)S[rw - 1];
        if (same) atomicAdd(dups, 1ull);
    }
}


int key_words_for(int w32) {
#ifdef WPM_KEY_FINE
    static const int buckets[] = {1, 2, 3, 4, 5, 6, 8, 16, 24, 32, 48, 64};
#else
    static const int buckets[] = {1, 2, 3, 4, 8, 16, 24, 32, 48, 64};
#endif
    for (int b : buckets)
        if (w32 <= b) return b;
    return -1;
}

template <int W>
static size_t temp_bytes_w(long long count) {
    size_t bytes = 0;
    cub::DeviceMergeSort::SortKeys(nullptr, bytes, (RowKey<W>*)nullptr, (int)count, RowLess<W>());
    return bytes;
}

template <int W>
static int sort_w(uint32_t* d_keys, long long count, int w32, uint32_t* d_sorted_bits, uint16_t* d_sorted_map,
                  void* d_temp, size_t temp_bytes, long long* d_first_row, unsigned long long* d_dups,
                  cudaStream_t st) {
    auto* keys = reinterpret_cast<RowKey<W>*>(d_keys);
    size_t bytes = temp_bytes;
    if (cub::DeviceMergeSort::SortKeys(d_temp, bytes, keys, (int)count, RowLess<W>(), st) != cudaSuccess) return 1;
    split_rows<W><<<(unsigned)((count + 255) / 256), 256, 0, st>>>(keys, count, w32, d_sorted_bits, d_sorted_map,
                                                                    d_dups, d_first_row);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

#ifdef WPM_KEY_FINE
#define WPM_KEY_FINE_CASES(CALL) \
    case 5: CALL(5);             \
    case 6: CALL(6);
#else
#define WPM_KEY_FINE_CASES(CALL)
#endif
#define WPM_KEY_DISPATCH(KW, CALL) \
    switch (KW) {                  \
        case 1: CALL(1);           \
        case 2: CALL(2);           \
        case 3: CALL(3);           \
        case 4: CALL(4);           \
        WPM_KEY_FINE_CASES(CALL)   \
        case 8: CALL(8);           \
        case 16: CALL(16);         \
        case 24: CALL(24);         \
        case 32: CALL(32);         \
        case 48: CALL(48);         \
        case 64: CALL(64);         \
        default: break;            \
    }

// temp = merge-sort scratch (+ the index array on the wide-row path)
size_t canon_sort_temp_bytes(long long count, int w32) {
    const int kw = key_words_for(w32);
    switch (kw) {
        case 1: return temp_bytes_w<1>(count);
        case 2: return temp_bytes_w<2>(count);
        case 3: return temp_bytes_w<3>(count);
        case 4: return temp_bytes_w<4>(count);
#ifdef WPM_KEY_DIRECT6
        case 5: return temp_bytes_w<5>(count);
        case 6: return temp_bytes_w<6>(count);
#endif
        default: break;
    }
    size_t bytes = 0;
    cub::DeviceMergeSort::SortKeys(nullptr, bytes, (uint32_t*)nullptr, (int)count, IdxLess{nullptr, kw + 1, w32});
    return bytes + ((size_t)count * 4 + 256);
}

int canon_sort_keys(uint32_t* d_keys, long long count, int w32, uint32_t* d_sorted_bits, uint16_t* d_sorted_map,
                    void* d_temp, size_t temp_bytes, long long* d_first_row, unsigned long long* d_dups,
                    cudaStream_t st) {
    if (count <= 0) return 0;
    const int kw = key_words_for(w32);
#define SW(W)                                                                                                  \
    case W:                                                                                                    \
        return sort_w<W>(d_keys, count, w32, d_sorted_bits, d_sorted_map, d_temp, temp_bytes, d_first_row, d_dups, st);
    switch (kw) {
        SW(1) SW(2) SW(3) SW(4)
#ifdef WPM_KEY_DIRECT6
        SW(5) SW(6)
#endif
        default: break;
    }
#undef SW
    const size_t idx_bytes = (size_t)count * 4 + 256;
    uint32_t* idx = reinterpret_cast<uint32_t*>(d_temp);
    void* sort_temp = static_cast<uint8_t*>(d_temp) + idx_bytes;
    size_t bytes = temp_bytes - idx_bytes;
    iota_u32<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(idx, count);
    const IdxLess cmp{d_keys, kw + 1, w32};
    if (cub::DeviceMergeSort::SortKeys(sort_temp, bytes, idx, (int)count, cmp, st) != cudaSuccess) return 1;
    const long long threads = count * 32;
    gather_rows<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(d_keys, kw + 1, idx, count, w32, d_sorted_bits,
                                                                     d_sorted_map, d_dups, d_first_row);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int canon_pack(const uint32_t* d_bits, const uint16_t* d_map, long long count, int w32, uint32_t* d_keys,
               cudaStream_t st) {
    if (count <= 0) return 0;
    const int kw = key_words_for(w32);
#define PK(W)                                                                                                    \
    pack_rows<W><<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d_bits, d_map, count, w32,                      \
                                                                    reinterpret_cast<RowKey<W>*>(d_keys));       \
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
    WPM_KEY_DISPATCH(kw, PK)
#undef PK
    return 1;
}

}  // namespace wpm
