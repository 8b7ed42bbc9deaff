// k8_verify.cu -- kernel 8: device verification of an enumeration result.
//
// For every emitted WPM K (one warp per row):
//   soundness      K is nonempty, inside the universe, |K| <= cap, and every
//                  ridge lies in exactly 0 or 2 facets of K -- the direct
//                  weak-pseudo-manifold test (complex.hpp:224-233, the
//                  predicate behind wpm_counts_ok, search.hpp:114-131);
//   reachability   K ^ base lies in the span of the reference basis's usable
//                  generators with at most two generators from any induced
//                  block -- i.e. the reference's combination space
//                  (search.hpp:81-104, kernel_basis.hpp:84-235) contains K, so
//                  enumerate_wpm would emit it.  The
//                  coordinates are solved as test_gf2.cpp:15-50 does, by
//                  elimination: on the host a set P of s pivot facets where the
//                  generators restricted to P are invertible, so
//                  x = (K ^ base)|_P * A^-1, then K ^ base == sum x_i g_i is
//                  checked word by word.  x is written out (the prefix-sampled
//                  completeness check, groups rows by it).
#include <cstdint>

#include "wpm_internal.h"

namespace wpm {

namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;

__global__ void __launch_bounds__(256) k8_verify(const __grid_constant__ VerifyParams p) {
    extern __shared__ __align__(16) uint32_t vsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int wpb = blockDim.x >> 5;
    uint32_t* cnt = vsm + (size_t)wid * p.cnt_words;  // ridge counts, one byte each
    const long long nwarps = (long long)gridDim.x * wpb;
    for (long long row = (long long)blockIdx.x * wpb + wid; row < p.count; row += nwarps) {
        const uint32_t* K = p.rows + (size_t)row * p.w32;
        const VerifyMap vm = p.maps[p.row_map[row]];
        const int mw = (vm.M + 31) >> 5;
        // ---- soundness
        int size = 0;
        bool outside = false;
        for (int w = lane; w < p.w32; w += 32) {
            uint32_t v = K[w];
            if (w == mw - 1 && (vm.M & 31)) outside |= (v >> (vm.M & 31)) != 0u;
            if (w >= mw) outside |= v != 0u;
            size += __popc(v);
        }
        size = (int)__reduce_add_sync(FULL, (unsigned)size);
        bool bad = __any_sync(FULL, outside) || size == 0 || size > vm.cap;
        for (int i = lane; i < ((vm.N + 3) >> 2); i += 32) cnt[i] = 0u;
        __syncwarp();
        for (int w = lane; w < mw; w += 32)
            for (uint32_t v = K[w]; v; v &= v - 1u) {
                const int f = w * 32 + __ffs(v) - 1;
                for (int k = 0; k < vm.n; ++k) {
                    const int r = p.fr[vm.fr_off + f * vm.fs + k];
                    atomicAdd(&cnt[r >> 2], 1u << ((r & 3) * 8));
                }
            }
        __syncwarp();
        bool odd = false;
        for (int i = lane; i < ((vm.N + 3) >> 2); i += 32) {
            const uint32_t c = cnt[i];
            for (int b = 0; b < 4; ++b) {
                const uint32_t x = (c >> (8 * b)) & 0xFFu;
                odd |= x != 0u && x != 2u;
            }
        }
        bad |= __any_sync(FULL, odd);
        uint8_t flag = bad ? 1 : 0;
        // ---- reachability in the reference basis
        unsigned long long x = 0;
        if (p.reach && vm.s >= 0) {
            const uint32_t* base = p.words + vm.base_off;
            unsigned long long yp = 0;
            for (int h = 0; h < 2; ++h) {
                const int i = lane + 32 * h;
                bool bit = false;
                if (i < vm.s) {
                    const int f = p.ints[vm.piv_off + i];
                    bit = (((K[f >> 5] ^ base[f >> 5]) >> (f & 31)) & 1u) != 0u;
                }
                yp |= (unsigned long long)__ballot_sync(FULL, bit) << (32 * h);
            }
            for (int h = 0; h < 2; ++h) {
                const int i = lane + 32 * h;
                const bool xi = i < vm.s && (__popcll(p.u64s[vm.inv_off + i] & yp) & 1);
                x |= (unsigned long long)__ballot_sync(FULL, xi) << (32 * h);
            }
            bool miss = false;
            const uint32_t* g = p.words + vm.gens_off;
            for (int w = lane; w < mw; w += 32) {
                uint32_t acc = 0;
                for (unsigned long long b = x; b; b &= b - 1ull) acc ^= g[(size_t)(__ffsll(b) - 1) * vm.W32 + w];
                miss |= acc != (K[w] ^ base[w]);
            }
            const bool span_bad = __any_sync(FULL, miss);
            bool blk = false;
            for (int b = lane; b < vm.nblk; b += 32) blk |= __popcll(x & p.u64s[vm.blk_off + b]) > 2;
            const bool blk_bad = __any_sync(FULL, blk);
            flag |= (span_bad ? 2 : 0) | (blk_bad ? 4 : 0);
        }
        if (lane == 0) {
            if (p.coords) p.coords[row] = x;
            if (p.flags) p.flags[row] = flag;
            if (flag & 1) atomicAdd(&p.ctl[0], 1ull);
            if (flag & 2) atomicAdd(&p.ctl[1], 1ull);
            if (flag & 4) atomicAdd(&p.ctl[2], 1ull);
        }
        __syncwarp();
    }
}

}  // namespace

int launch_k8_verify(const VerifyParams& p, int num_sms, cudaStream_t st) {
    if (p.count <= 0) return 0;
    const int threads = 256, wpb = threads / 32;
    const size_t smem = (size_t)wpb * p.cnt_words * 4;
    if (cudaFuncSetAttribute(k8_verify, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    long long blocks = (p.count + wpb - 1) / wpb;
    blocks = blocks < (long long)num_sms * 8 ? blocks : (long long)num_sms * 8;
    k8_verify<<<(unsigned)blocks, threads, smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace wpm
