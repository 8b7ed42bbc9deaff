// k1_universe.cu -- kernel 1: the candidate-facet generator.
//
// Replaces binary_matroid + gf2col::independent (charmap.hpp:92-141) and
// matroid_universe (pipeline.hpp:33-35): a facet is an n-subset of the m
// columns of the mod-2 characteristic map that is linearly independent.
// Data-parallel over C(m, n) subsets x maps: one CTA per map, one thread per
// subset.  Thread t unranks the t-th n-subset in colex order -- colex order of
// subsets IS ascending bitmask order, the canonical VertexSet order
// (vertex_set.hpp:55) -- so an order-preserving block compaction emits the
// universe already sorted (PureComplex ctor sort, complex.hpp:33).  The
// independence test is bitmask GF(2) elimination keyed by leading bit.
#include <cstdint>

#include "wpm_dev.cuh"
#include "wpm_internal.h"

namespace wpm {

__device__ __forceinline__ uint32_t colex_unrank(const uint32_t (*c_binom)[17], uint32_t t, int k, int m) {
    uint32_t mask = 0;
    int c = m - 1;
    for (int i = k; i >= 1; --i) {
        while (c_binom[c][i] > t) --c;  // largest c with C(c, i) <= t
        mask |= 1u << c;
        t -= c_binom[c][i];
        --c;
    }
    return mask;
}

__device__ __forceinline__ int gf2_rank_of(const uint32_t* cols, uint32_t sel) {
    uint32_t basis[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) basis[b] = 0;
    int r = 0;
    while (sel) {
        const int v = __ffs(sel) - 1;
        sel &= sel - 1;
        uint32_t x = cols[v];
        while (x) {
            const int b = 31 - __clz(x);
            if (basis[b]) {
                x ^= basis[b];
            } else {
                basis[b] = x;
                ++r;
                break;
            }
        }
    }
    return r;
}

__global__ void __launch_bounds__(1024) k1_universe(Binom bn, int n, int m, const uint32_t* __restrict__ cols,
                                                    uint32_t* __restrict__ facets, int facet_stride,
                                                    int32_t* __restrict__ M_out) {
    const int map = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ uint32_t s_cols[32];
    __shared__ int s_warp[32];
    __shared__ int s_rank_ok;
    __shared__ uint32_t c_binom[17][17];
    for (int i = tid; i < 17 * 17; i += blockDim.x) c_binom[i / 17][i % 17] = bn.c[i / 17][i % 17];
    if (tid < m) s_cols[tid] = cols[map * m + tid];
    __syncthreads();
    if (tid == 0) s_rank_ok = gf2_rank_of(s_cols, (m >= 32) ? 0xFFFFFFFFu : ((1u << m) - 1u)) == n;
    __syncthreads();
    if (!s_rank_ok) {  // binary_matroid throws on a rank-deficient map (charmap.hpp:118-121)
        if (tid == 0) M_out[map] = -1;
        return;
    }
    const uint32_t total = c_binom[m][n];
    int running = 0;
    uint32_t* out = facets + (size_t)map * facet_stride;
    for (uint32_t base = 0; base < total; base += blockDim.x) {
        const uint32_t t = base + tid;
        bool ok = false;
        uint32_t mask0 = 0;
        if (t < total) {
            mask0 = colex_unrank(c_binom, t, n, m);
            ok = gf2_rank_of(s_cols, mask0) == n;
        }
        const unsigned b = __ballot_sync(0xFFFFFFFFu, ok);
        if (lane == 0) s_warp[warp] = __popc(b);
        __syncthreads();
        int before = 0, block_total = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            if (w < warp) before += s_warp[w];
            block_total += s_warp[w];
        }
        const int pos = running + before + __popc(b & ((1u << lane) - 1u));
        if (ok && pos < facet_stride) out[pos] = mask0 << 1;  // 1-based labels
        running += block_total;
        __syncthreads();
    }
    if (tid == 0) M_out[map] = running;
}

int launch_k1_universe(int n, int m, int num_maps, const uint32_t* d_cols, uint32_t* d_facets,
                       int facet_stride, int32_t* d_M, cudaStream_t st) {
    // few maps (n >= 9: 1-7 CTAs on 148 SMs): 1024 threads per map cut the
    // serial subset loop 4x (n = 11: one CTA over 1365 subsets)
    const int threads = num_maps <= 32 ? 1024 : 256;
    k1_universe<<<num_maps, threads, 0, st>>>(make_binom(), n, m, d_cols, d_facets, facet_stride, d_M);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace wpm
