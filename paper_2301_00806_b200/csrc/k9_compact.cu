// k9_compact.cu -- stream compaction: the flagged indices (or values) of an
// array, in order, in one cooperative launch.  Used by the line-7 / line-13
// selects (k5_line13.cu) and the line-15 first-appearance dedupe
// (k7_line15.cu) in place of a library select.
//
// Each CTA owns a contiguous range: it counts its flags, one grid barrier,
// every CTA sums the counts of the CTAs before it (<= a few hundred), then
// walks its range 1024 items at a time with a ballot / warp-count block scan
// and scatters.  The last CTA writes the total.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>

#include "wpm_internal.h"

namespace cg = cooperative_groups;

namespace wpm {

namespace {

constexpr int CT = 1024;

__global__ void __launch_bounds__(CT, 1) k_compact(const uint32_t* __restrict__ in, const uint8_t* __restrict__ flags,
                                                   long long n, uint32_t* __restrict__ out, int* __restrict__ d_num,
                                                   unsigned* __restrict__ block_cnt) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned s_warp[32];
    __shared__ unsigned s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long per = (n + gridDim.x - 1) / gridDim.x;
    const long long lo = std::min<long long>(n, (long long)blockIdx.x * per), hi = std::min<long long>(n, lo + per);
    // phase 1: this CTA's count
    unsigned c = 0;
    for (long long i = lo + tid; i < hi; i += CT) c += flags[i] != 0;
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if (lane == 0) s_warp[warp] = c;
    __syncthreads();
    if (tid == 0) {
        unsigned t = 0;
        for (int w = 0; w < CT / 32; ++w) t += s_warp[w];
        block_cnt[blockIdx.x] = t;
    }
    grid.sync();
    // the CTAs before this one
    unsigned before = 0;
    for (int b = tid; b < (int)blockIdx.x; b += CT) before += block_cnt[b];
    before = __reduce_add_sync(0xFFFFFFFFu, before);
    __syncthreads();
    if (lane == 0) s_warp[warp] = before;
    __syncthreads();
    if (tid == 0) {
        unsigned t = 0;
        for (int w = 0; w < CT / 32; ++w) t += s_warp[w];
        s_base = t;
    }
    __syncthreads();
    unsigned base = s_base;
    // phase 2: ordered scatter, CT items per step
    for (long long i0 = lo; i0 < hi; i0 += CT) {
        const long long i = i0 + tid;
        const bool f = i < hi && flags[i] != 0;
        const unsigned b = __ballot_sync(0xFFFFFFFFu, f);
        __syncthreads();  // s_warp reuse
        if (lane == 0) s_warp[warp] = __popc(b);
        __syncthreads();
        unsigned wbefore = 0, total = 0;
        for (int w = 0; w < CT / 32; ++w) {
            const unsigned x = s_warp[w];
            wbefore += w < warp ? x : 0u;
            total += x;
        }
        if (f) out[base + wbefore + __popc(b & ((1u << lane) - 1u))] = in ? in[i] : (uint32_t)i;
        base += total;
    }
    if (blockIdx.x == gridDim.x - 1 && tid == 0) *d_num = (int)base;
}

int g_compact_sms[64] = {0};

}  // namespace

size_t compact_temp_bytes() { return 4096 * sizeof(unsigned); }

int compact_flagged(const uint32_t* in, const uint8_t* flags, long long n, uint32_t* out, int* d_num, void* d_temp,
                    cudaStream_t st) {
    if (n <= 0) return cudaMemsetAsync(d_num, 0, sizeof(int), st) == cudaSuccess ? 0 : 1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 1;
    if (!g_compact_sms[dev] &&
        cudaDeviceGetAttribute(&g_compact_sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return 1;
    // one CTA per SM (cooperative), at least 4096 items per CTA
    const int grid = (int)std::max<long long>(1, std::min<long long>(g_compact_sms[dev], (n + 4095) / 4096));
    unsigned* block_cnt = static_cast<unsigned*>(d_temp);
    void* args[] = {(void*)&in, (void*)&flags, (void*)&n, (void*)&out, (void*)&d_num, (void*)&block_cnt};
    if (cudaLaunchCooperativeKernel((const void*)k_compact, dim3(grid), dim3(CT), args, 0, st) != cudaSuccess) return 1;
    return 0;
}

}  // namespace wpm
