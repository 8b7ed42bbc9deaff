// k4_canon.cu -- canonical order of the emitted WPMs.
//
// Replaces the merge + sort + unique of enumerate_wpm (search.hpp:247-257):
// complexes are ordered by their facet lists (std::vector<VertexSet>
// operator<, facets ascending), i.e. lexicographically on the ascending
// facet-index lists with a proper prefix first.  On characteristic bitsets
// that is decided at d = the lowest facet in exactly one of A, B: the list
// holding d is smaller unless the other list ends before d.  A merge sort of
// row indices with that comparator (rows stay put, L2 resident), then one
// gather pass that also counts adjacent duplicates (the DFS partitions the
// space, so the count is 0 -- a checked invariant, not a dedupe).
#include <cub/device/device_merge_sort.cuh>

#include <cstdint>

#include "wpm_internal.h"

namespace wpm {

struct CanonLess {
    const uint32_t* bits;
    const uint16_t* map;
    int w32;
    __device__ __forceinline__ bool operator()(const uint32_t& a, const uint32_t& b) const {
        const uint16_t ma = map[a], mb = map[b];
        if (ma != mb) return ma < mb;
        const uint32_t* A = bits + (size_t)a * w32;
        const uint32_t* B = bits + (size_t)b * w32;
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

__global__ void gather_rows(const uint32_t* __restrict__ bits, const uint16_t* __restrict__ map,
                            const uint32_t* __restrict__ idx, long long n, int w32, uint32_t* __restrict__ out,
                            uint16_t* __restrict__ out_map, unsigned long long* dups,
                            long long* __restrict__ first_row) {
    // one warp per row; first_row[map] = index of the map's first row (group boundaries)
    const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const uint32_t src = idx[row];
    const bool new_group = row == 0 || map[idx[row - 1]] != map[src];
    if (lane == 0 && new_group && first_row) first_row[map[src]] = row;
    bool same = !new_group;
    const uint32_t* S = bits + (size_t)src * w32;
    const uint32_t* P = row > 0 ? bits + (size_t)idx[row - 1] * w32 : S;
    for (int w = lane; w < w32; w += 32) {
        const uint32_t v = S[w];
        out[(size_t)row * w32 + w] = v;
        if (P[w] != v) same = false;
    }
    same = __all_sync(0xFFFFFFFFu, same);
    if (lane == 0) {
        out_map[row] = map[src];
        if (same) atomicAdd(dups, 1ull);
    }
}

size_t canon_sort_temp_bytes(long long count, int w32) {
    size_t bytes = 0;
    CanonLess cmp{nullptr, nullptr, w32};
    cub::DeviceMergeSort::SortKeys(nullptr, bytes, (uint32_t*)nullptr, (int)count, cmp);
    return bytes;
}

int canon_sort(const uint32_t* d_bits, const uint16_t* d_map, long long count, int w32, uint32_t* d_sorted_bits,
               uint16_t* d_sorted_map, void* d_temp, size_t temp_bytes, uint32_t* d_idx_a, long long* d_first_row,
               unsigned long long* d_dups, cudaStream_t st) {
    if (count <= 0) return 0;
    iota_u32<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d_idx_a, count);
    CanonLess cmp{d_bits, d_map, w32};
    size_t bytes = temp_bytes;
    if (cub::DeviceMergeSort::SortKeys(d_temp, bytes, d_idx_a, (int)count, cmp, st) != cudaSuccess) return 1;
    const long long threads = count * 32;
    gather_rows<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(d_bits, d_map, d_idx_a, count, w32,
                                                                     d_sorted_bits, d_sorted_map, d_dups,
                                                                     d_first_row);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace wpm
