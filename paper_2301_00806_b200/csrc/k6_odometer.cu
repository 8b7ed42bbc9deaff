// k6_odometer.cu -- Algorithm 1 of the paper, the reference's own search, on
// the device (§8(f) row 3: the apples-to-apples comparison).
//
// The reference (search.hpp:141-258) enumerates the combination space of a
// convenient kernel basis: every leaf K = base ^ (one XOR delta per block)
// (search.hpp:156-166, :192-243), skips the empty set and the leaves over the
// count cap (:204-210), and keeps K iff every touched ridge lies in exactly two
// facets of K (wpm_counts_ok, :114-131).  This kernel visits exactly the same
// leaves:
//   * the blocks (widest first, as :168-170) split into an OUTER part, one
//     prefix per lane, and an INNER part of the last r blocks (sized on the
//     host so that every lane of the grid gets several prefixes), walked
//     by a warp-uniform odometer: each step XORs one precomputed step delta
//     delta[d] ^ delta[d+1 mod c] (a broadcast load) into the lane's K;
//   * per leaf: W XORs, W POPCs, one compare, one ballot;
//   * the leaves inside the cap are queued per warp in shared memory (32
//     entries, interleaved) and checked 32 at a time, one per lane
//     (wpm_counts_ok): every (facet, ridge) incidence marks a "seen once" /
//     "seen twice" bit in lane-private shared-memory bitsets (word i of lane
//     l at i * 32 + l: bank-conflict free for any pattern); a third
//     incidence rejects at once.  The leaf loop itself stays branch-light.  Every K is in the GF(2) kernel of the
//     incidence matrix, so all ridge counts are even and "no count >= 3" is
//     "every touched count == 2";
//   * accepted K go out as key rows (map id last) into the same canonical
//     sort as kernel 3's output.
#include <cstdint>

#include "wpm_internal.h"

namespace wpm {

namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr int ODO_WARPS = 8;
constexpr int MAX_INNER = 64;

// __ldg of step / delta words (read-only, L1-resident, warp-uniform address
// for the inner odometer -> one broadcast transaction)
template <int W>
__device__ __forceinline__ void xor_words(uint32_t (&K)[W], const uint32_t* __restrict__ src) {
#pragma unroll
    for (int w = 0; w < W; ++w) K[w] ^= __ldg(src + w);
}

// wpm_counts_ok (search.hpp:114-131) for up to 32 queued candidates, one per
// lane: every (facet, ridge) incidence marks a "seen once" / "seen twice" bit
// in the lane's private bitsets; a third incidence rejects at once.  The
// accepted K go out as key rows (kw bitset words, zero padded, + map id).
template <int W>
__device__ __forceinline__ void flush_queue(const OdoParams& p, const uint32_t* Q, int qn, uint32_t* seen1,
                                            uint32_t* seen2, int nw, const uint16_t* frm, int fs, int n, int map,
                                            int lane, unsigned long long& checked) {
    uint32_t K[W];
    bool ok = lane < qn;
#pragma unroll
    for (int w = 0; w < W; ++w) K[w] = ok ? Q[w * 32 + lane] : 0u;
    if (ok) {
        ++checked;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            for (uint32_t x = K[w]; x && ok; x &= x - 1) {
                const uint16_t* fr = frm + (size_t)(w * 32 + __ffs(x) - 1) * fs;
                for (int q = 0; q < n; ++q) {
                    const int r = __ldg(fr + q);
                    const uint32_t bit = 1u << (r & 31);
                    uint32_t* a1 = seen1 + (size_t)(r >> 5) * 32;
                    const uint32_t s1 = *a1;
                    if (!(s1 & bit)) {
                        *a1 = s1 | bit;
                        continue;
                    }
                    uint32_t* a2 = seen2 + (size_t)(r >> 5) * 32;
                    const uint32_t s2 = *a2;
                    if (s2 & bit) {
                        ok = false;
                        break;
                    }
                    *a2 = s2 | bit;
                }
            }
        }
        for (int i = 0; i < 2 * nw; ++i) seen1[(size_t)i * 32] = 0u;
    }
    __syncwarp();
    const unsigned acc = __ballot_sync(FULL, ok);
    if (!acc) return;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(p.out_ctl, (unsigned long long)__popc(acc));
    base = __shfl_sync(FULL, base, 0);
    if (ok) {
        const unsigned long long slot = base + __popc(acc & ((1u << lane) - 1u));
        if (slot < p.out_cap) {
            uint32_t* row = p.out_keys + slot * (unsigned long long)p.rw;
#pragma unroll
            for (int w = 0; w < W; ++w)
                if (w < p.rw - 1) row[w] = K[w];  // (words past the plan's mw are zero)
            for (int w = W; w < p.rw - 1; ++w) row[w] = 0u;
            row[p.rw - 1] = (uint32_t)map;
        }
    }
}

template <int W>
__global__ void __launch_bounds__(32 * ODO_WARPS) odometer(const __grid_constant__ OdoParams p) {
    extern __shared__ __align__(16) uint32_t odo_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // per lane: two "seen" bitsets over the ridges (seen once / seen twice),
    // word i of lane l at [i * 32 + l]: any per-lane access pattern is
    // bank-conflict free
    const int nw = p.cnt_words;  // ridge words
    uint32_t* wbase = odo_smem + (size_t)wib * (2 * nw * 32 + W * 32);
    uint32_t* Q = wbase + 2 * nw * 32;  // candidate queue: word w of entry e at Q[w * 32 + e]
    uint32_t* seen1 = wbase + lane;
    uint32_t* seen2 = seen1 + (size_t)nw * 32;
    for (int i = 0; i < 2 * nw; ++i) seen1[(size_t)i * 32] = 0u;
    int dig[MAX_INNER];
    unsigned long long leaves = 0, checked = 0;

    for (;;) {
        long long task = 0;
        if (lane == 0) task = (long long)atomicAdd(p.task_ctr, 1ull);
        task = __shfl_sync(FULL, task, 0);
        if (task >= p.total_tasks) break;
        // the map owning this task (maps ordered by first task)
        int lo = 0, hi = p.num_maps - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (p.maps[mid].task0 <= task) lo = mid;
            else hi = mid - 1;
        }
        const OdoMap om = p.maps[lo];
        const long long pre = (task - om.task0) * 32 + lane;
        const bool act = pre < om.outer;
        const int* ncand = p.blk_ncand + om.blk;
        const uint32_t* bdelta = p.words + om.delta_off;  // candidate c of block b at (blk_first[b] + c) * W
        const int* bfirst = p.blk_first + om.blk;
        const uint16_t* frm = p.fr + om.fr_off;
        uint32_t K[W];
#pragma unroll
        for (int w = 0; w < W; ++w) K[w] = __ldg(p.words + om.base_off + w);
        if (act) {
            long long rem = pre;
            for (int b = om.nb - om.r - 1; b >= 0; --b) {
                const int c = ncand[b];
                const int d = (int)(rem % c);
                rem /= c;
                if (d) xor_words<W>(K, bdelta + (size_t)(bfirst[b] + d) * W);
            }
        }
        const int b0 = om.nb - om.r;  // first inner block
        for (int i = 0; i < om.r; ++i) dig[i] = 0;
        const uint32_t* bstep = p.words + om.step_off;  // step c of block b at (blk_first[b] + c) * W
        // the innermost block's digit / size / steps stay in registers
        const int bl = om.nb - 1;
        const int nc_in = om.r > 0 ? ncand[bl] : 1;
        const uint32_t* step_in = bstep + (size_t)(om.r > 0 ? bfirst[bl] : 0) * W;
        int d_in = 0;
        int qn = 0;  // queued candidates (warp-uniform)
        // a binary innermost block {0, g} (the usual case: free generators
        // sort last) steps by g both ways: keep g in registers
        const bool bin_in = om.r > 0 && nc_in == 2;
        uint32_t g_in[W];
#pragma unroll
        for (int w = 0; w < W; ++w) g_in[w] = bin_in ? __ldg(step_in + w) : 0u;
        for (long long leaf = 0; leaf < om.inner; ++leaf) {
            int pc = 0;
#pragma unroll
            for (int w = 0; w < W; ++w) pc += __popc(K[w]);
            const bool cand = act && pc >= 1 && pc <= om.cap;
            leaves += act ? 1 : 0;
            unsigned cm = __ballot_sync(FULL, cand);
            while (cm) {  // enqueue (warp-uniform); a full queue is checked 32 at a time
                const int rank = __popc(cm & ((1u << lane) - 1u));
                const bool take = ((cm >> lane) & 1u) && rank < 32 - qn;
                if (take) {
#pragma unroll
                    for (int w = 0; w < W; ++w) Q[w * 32 + qn + rank] = K[w];
                }
                const unsigned tk = __ballot_sync(FULL, take);
                qn += __popc(tk);
                cm &= ~tk;
                if (qn == 32) {
                    __syncwarp();
                    flush_queue<W>(p, Q, qn, seen1, seen2, nw, frm, om.fs, om.n, om.map, lane, checked);
                    qn = 0;
                    __syncwarp();
                }
            }
            // advance the inner odometer (warp-uniform)
            if (om.r > 0) {
                if (bin_in) {
#pragma unroll
                    for (int w = 0; w < W; ++w) K[w] ^= g_in[w];
                } else {
                    xor_words<W>(K, step_in + (size_t)d_in * W);
                }
                if (++d_in == nc_in) {  // wrapped: the step back to candidate 0 is applied; carry
                    d_in = 0;
                    for (int i = om.r - 2; i >= 0; --i) {
                        const int b = b0 + i;
                        const int d = dig[i];
                        xor_words<W>(K, bstep + (size_t)(bfirst[b] + d) * W);
                        if (d + 1 < ncand[b]) {
                            dig[i] = d + 1;
                            break;
                        }
                        dig[i] = 0;
                    }
                }
            }
        }
        if (qn) {
            __syncwarp();
            flush_queue<W>(p, Q, qn, seen1, seen2, nw, frm, om.fs, om.n, om.map, lane, checked);
            __syncwarp();
        }
    }
    atomicAdd(p.leaf_ctr, leaves);
    atomicAdd(p.leaf_ctr + 1, checked);
}

template <int W>
int launch_w(const OdoParams& p, int num_sms, cudaStream_t st) {
    const size_t smem = (size_t)ODO_WARPS * (2 * p.cnt_words + W) * 32 * 4;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(odometer<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, odometer<W>, 32 * ODO_WARPS, smem) != cudaSuccess ||
        per_sm < 1)
        return 1;
    odometer<W><<<(unsigned)(num_sms * per_sm), 32 * ODO_WARPS, smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace

int odo_max_inner() { return MAX_INNER; }

int launch_odometer(const OdoParams& p, int W, int num_sms, cudaStream_t st) {
    switch (W) {
#define WPM_ODO_W(X) \
    case X: return launch_w<X>(p, num_sms, st);
        WPM_ODO_W(1) WPM_ODO_W(2) WPM_ODO_W(3) WPM_ODO_W(4) WPM_ODO_W(5) WPM_ODO_W(6) WPM_ODO_W(7) WPM_ODO_W(8)
        WPM_ODO_W(9) WPM_ODO_W(10) WPM_ODO_W(11) WPM_ODO_W(12) WPM_ODO_W(13) WPM_ODO_W(14) WPM_ODO_W(15)
        WPM_ODO_W(16) WPM_ODO_W(20) WPM_ODO_W(24) WPM_ODO_W(28) WPM_ODO_W(32)
#undef WPM_ODO_W
        default: return 1;
    }
}

int odo_words_bucket(int W) {
    if (W <= 16) return W < 1 ? 1 : W;
    if (W <= 20) return 20;
    if (W <= 24) return 24;
    if (W <= 28) return 28;
    if (W <= 32) return 32;
    return -1;
}

}  // namespace wpm
