// k2_incidence.cu -- kernel 2: the ridge -> candidate-facet incidence tables.
//
// Replaces ridges_of (complex.hpp:107-119) and incidence_matrix
// (incidence.hpp:34-55).  One CTA per map.  Every (n-1)-subset of [m] has a
// colex rank < C(m, n-1) (<= 11440 for m <= 16), so the ridge set is a flag
// array in shared memory and its order-preserving block scan IS the
// canonical ridge order (ascending bitmask).  A second shared table maps the
// colex rank of an n-subset to its facet index, so the candidate facets of a
// ridge r are {r + v : v not in r} looked up directly -- ascending v gives
// ascending facet masks, the reference's parent order (incidence.hpp:47-52).
// fr[f] lists f's ridges ascending: dropping a higher vertex gives a smaller
// mask, so vertices are walked high to low.
#include <cstdint>

#include "wpm_dev.cuh"
#include "wpm_internal.h"

namespace wpm {

__device__ __forceinline__ uint32_t colex_rank(const uint32_t (*cb)[17], uint32_t mask0) {
    uint32_t r = 0;
    int i = 1;
    while (mask0) {
        const int c = __ffs(mask0) - 1;
        mask0 &= mask0 - 1;
        r += cb[c][i++];
    }
    return r;
}

__device__ __forceinline__ uint32_t colex_unrank2(const uint32_t (*cb)[17], uint32_t t, int k, int m) {
    uint32_t mask = 0;
    int c = m - 1;
    for (int i = k; i >= 1; --i) {
        while (cb[c][i] > t) --c;
        mask |= 1u << c;
        t -= cb[c][i];
        --c;
    }
    return mask;
}

__global__ void __launch_bounds__(1024) k2_incidence(Binom bn, const MapDesc* __restrict__ maps,
                                                     const uint32_t* __restrict__ facets,
                                                     uint32_t* __restrict__ ridges, uint16_t* __restrict__ fr,
                                                     uint16_t* __restrict__ rp, uint8_t* __restrict__ npar,
                                                     int32_t* __restrict__ N_out, int32_t* __restrict__ err) {
    extern __shared__ uint32_t smem[];
    __shared__ uint32_t cb[17][17];
    __shared__ int s_warp[32];
    __shared__ int s_bad;
    const int map = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nthreads = blockDim.x;
    const MapDesc d = maps[map];
    const int M = d.M, n = d.n, m = d.m;
    for (int i = tid; i < 17 * 17; i += nthreads) cb[i / 17][i % 17] = bn.c[i / 17][i % 17];
    if (tid == 0) s_bad = 0;
    const int CF = (int)binom_small(m, n), CR = (int)binom_small(m, n - 1);
    uint32_t* rflag = smem;                                // CR entries, then prefix sums
    uint16_t* fidx = reinterpret_cast<uint16_t*>(smem + CR);  // CF entries
    for (int i = tid; i < CR; i += nthreads) rflag[i] = 0;
    for (int i = tid; i < CF; i += nthreads) fidx[i] = NONE16;
    __syncthreads();
    const uint32_t* F = facets + d.facet_off;
    for (int j = tid; j < M; j += nthreads) {
        const uint32_t f0 = F[j] >> 1;
        fidx[colex_rank(cb, f0)] = (uint16_t)j;
        for (uint32_t b = f0; b; b &= b - 1) rflag[colex_rank(cb, f0 & ~(b & (~b + 1)))] = 1;
    }
    __syncthreads();
    // block-wide exclusive scan of rflag (contiguous chunk per thread)
    const int chunk = (CR + nthreads - 1) / nthreads;
    const int lo = tid * chunk, hi = min(CR, lo + chunk);
    int local = 0;
    for (int i = lo; i < hi; ++i) local += (int)rflag[i];
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (nthreads >> 5); ++w) {
        if (w < warp) before += s_warp[w];
        total += s_warp[w];
    }
    int run = before + incl - local;
    for (int i = lo; i < hi; ++i) {
        const uint32_t fl = rflag[i];
        rflag[i] = fl ? (uint32_t)run : 0xFFFFFFFFu;  // ridge index, or none
        run += (int)fl;
    }
    __syncthreads();
    const int N = total;
    uint32_t* R = ridges + d.ridge_off;
    for (int i = tid; i < CR; i += nthreads)
        if (rflag[i] != 0xFFFFFFFFu) R[rflag[i]] = colex_unrank2(cb, (uint32_t)i, n - 1, m) << 1;
    // facet -> ridges (ascending)
    uint16_t* FRm = fr + d.fr_off;
    for (int j = tid; j < M; j += nthreads) {
        const uint32_t f0 = F[j] >> 1;
        int k = 0;
        for (int v = m - 1; v >= 0; --v)
            if ((f0 >> v) & 1u) FRm[j * d.fr_stride + k++] = (uint16_t)rflag[colex_rank(cb, f0 & ~(1u << v))];
    }
    // ridge -> candidate facets (ascending)
    uint16_t* RPm = rp + d.rp_off;
    uint8_t* NPm = npar + d.np_off;
    for (int i = tid; i < CR; i += nthreads) {
        const uint32_t ri = rflag[i];
        if (ri == 0xFFFFFFFFu) continue;
        const uint32_t r0 = colex_unrank2(cb, (uint32_t)i, n - 1, m);
        int c = 0;
        for (int v = 0; v < m; ++v) {
            if ((r0 >> v) & 1u) continue;
            const uint16_t g = fidx[colex_rank(cb, r0 | (1u << v))];
            if (g == NONE16) continue;
            if (c < d.rp_stride) RPm[ri * d.rp_stride + c] = g;
            ++c;
        }
        if (c > d.rp_stride) s_bad = 1;
        NPm[ri] = (uint8_t)min(c, d.rp_stride);
        for (int q = c; q < d.rp_stride; ++q) RPm[ri * d.rp_stride + q] = NONE16;
    }
    __syncthreads();
    if (tid == 0) {
        N_out[map] = N;
        if (s_bad) atomicExch(err, 1);
    }
}

int launch_k2_incidence(int num_maps, const MapDesc* d_maps, int max_m, int max_n, const uint32_t* d_facets,
                        uint32_t* d_ridges, uint16_t* d_fr, uint16_t* d_rp, uint8_t* d_npar, int32_t* d_N,
                        int32_t* d_err, cudaStream_t st) {
    // smem: C(m, n-1) uint32 flags + C(m, n) uint16 facet ids, sized for the largest (m, n)
    size_t smem = 0;
    for (int n = 1; n <= max_n; ++n) {
        const size_t s = (size_t)binom_small(max_m, n - 1) * 4 + (size_t)binom_small(max_m, n) * 2 + 16;
        if (s > smem) smem = s;
    }
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(k2_incidence, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    // few maps: 1024 threads per map (n = 11: one CTA, 320 us at 256 threads)
    const int threads = num_maps <= 32 ? 1024 : 256;
    k2_incidence<<<num_maps, threads, smem, st>>>(make_binom(), d_maps, d_facets, d_ridges, d_fr, d_rp, d_npar, d_N,
                                                   d_err);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace wpm
