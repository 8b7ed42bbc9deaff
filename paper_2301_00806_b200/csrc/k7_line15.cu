// k7_line15.cu -- Algorithm 2 line 15 on the device: canonical forms.
//
// Replaces, in the reference pipeline (pipeline.hpp:91-103), the per-complex
// `canonical_form(K)` (isomorphism.hpp:228-303) and the first-appearance
// dedupe of the canonical facet lists.  One warp per complex (a dynamic
// ticket counter hands complexes to warps: the cost varies by orders of
// magnitude with the complex's symmetry), everything in shared memory:
//
//  1. face poset as a bitmap over all 2^m vertex masks (m <= 15: <= 4 KB):
//     the facets' bits, then the down-closure one coordinate at a time
//     (in-word shifts for the 5 low mask bits, word pairs for the others);
//  2. minimal non-faces (complex.hpp:192-221) as a second bitmap:
//     S is one iff S is not a face and every S \ {b} is -- the same
//     shift / word-pair pattern, AND-reduced; listed in ascending order;
//  3. the refined vertex classes of detail::refine_classes
//     (isomorphism.hpp:162-218), with the reference's class ORDER (it fixes
//     which labels each class gets, hence the canonical form).  A vertex key
//     is [rank, -1, e, -1, e, ...] over its sorted env entries e =
//     [0, |S|, sorted ranks] (minimal non-face S) or [1, sorted ranks]
//     (facet).  No entry is a proper prefix of a different one, so entries
//     compare as fixed-width codes: type bit, |S| nibble, ranks as nibbles,
//     left aligned -- order preserving (ranks < 16, |S| <= n + 1 <= 12).
//     The item index rides in the low 11 bits, so one bitonic sort of
//     64-bit keys orders all entries of all vertices at once; a vertex's
//     sorted env is the subsequence of the items that contain it, stored as
//     ids (first sorted position of the code).  Keys of two vertices then
//     compare as (old rank, id sequence) -- 32 positions per step, ballot
//     for the first difference.  The initial key (the color sequence,
//     :17-24) is the same machinery with items = minimal non-faces, code =
//     |S|.  Rounds stop when the class count stops growing, as :209-214;
//  4. the lexicographically least relabeled facet list over all relabelings
//     that give class c the c-th consecutive label range (:259-288).  The
//     reference prunes at class boundaries; this is a DFS over single
//     placements that prunes at every one, still exactly: after labels
//     0..t are placed, the facets that are complete are exactly the final
//     list's masks below 2^(t+1), so comparing the masks that complete at
//     step t (all in [2^t, 2^(t+1))) with the best list's masks in that
//     range decides the branch against the best (the lists have the same
//     length, so the lowest mask in their symmetric difference decides,
//     with no prefix case).  The best list lives as a bitmap + a sorted
//     list; the current one as a bitmap + per-facet partial masks.
//
// Output: the canonical facet list as a row over all C(m, n) n-subsets in
// colex order (the line-13 row format), so the rows sort and dedupe with
// the same machinery (api.cu: first appearance = lowest survivor index).
// Parity: oracle/line15_port.c restates refine_classes / canonical_form
// literally; the tests check the device against it and against the
// reference itself (oracle/_ref plseeds_ref classes / line15).

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "wpm_internal.h"

namespace wpm {

namespace {

constexpr uint32_t FULL = 0xFFFFFFFFu;
constexpr int L15_WARPS = 4;
constexpr unsigned long long INF64 = ~0ull;
constexpr uint32_t INF32 = 0xFFFFFFFFu;

// positions p of a 32-bit word with bit b of p clear, b = 0..4
__device__ __forceinline__ uint32_t low_half_mask(int b) {
    return b == 0 ? 0x55555555u : b == 1 ? 0x33333333u : b == 2 ? 0x0F0F0F0Fu : b == 3 ? 0x00FF00FFu : 0x0000FFFFu;
}

__device__ __forceinline__ uint32_t colex_rank(uint32_t mask, const Binom& B) {
    uint32_t r = 0;
    int i = 1;
    for (uint32_t x = mask; x; x &= x - 1, ++i) r += B.c[__ffs(x) - 1][i];
    return r;
}

__device__ __forceinline__ int warp_incl_scan(int x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += t;
    }
    return x;
}

// bitonic sort of P (power of two) uint64 keys in shared memory, one warp
__device__ void warp_bitonic(unsigned long long* a, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int l = i ^ j;
                if (l > i) {
                    const unsigned long long x = a[i], y = a[l];
                    const bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[l] = x;
                    }
                }
            }
            __syncwarp();
        }
    }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {  // splitmix64 finalizer
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// sorted ranks of the vertices of `s` as nibbles from bit `top` downward
__device__ __forceinline__ unsigned long long rank_nibbles(uint32_t s, const uint16_t* clsmask, int ncls, int top) {
    unsigned long long code = 0;
    int pos = top;
    for (int r = 0; r < ncls && s; ++r) {
        const uint32_t hit = s & clsmask[r];
        s &= ~hit;
        for (int c = __popc(hit); c > 0; --c, pos -= 4) code |= (unsigned long long)r << pos;
    }
    return code;
}

}  // namespace

struct L15Src {
    // row mode: complex i = rows[idx ? idx[i] : i] (gw words over colex n-subsets)
    const uint32_t* rows;
    const uint32_t* idx;
    const int* num;  // device count (row mode, may be null)
    const uint16_t* unrank;
    // csr mode (rows == null): 0-based masks, ascending per complex
    const uint16_t* masks;
    const long long* off;
    long long count;
};

struct L15Out {
    uint32_t* rows;             // row mode: gw words per complex
    uint16_t* masks;            // csr mode: canonical masks at the input offsets
    int8_t* cls;                // optional: refined class per vertex (16 per complex)
    unsigned long long* cost;   // optional: single-vertex placements per complex
    unsigned long long* ctl;    // [0] ticket, [1] overflow, [2] labelings completed, [3] placements,
                                // [4] cache hits (canonical form confirmed from a cached one)
    // canonical-form cache (optional): write-once slots keyed by an
    // isomorphism-invariant hash; slot data = k, then the canonical facets
    unsigned long long* cache_key;
    uint16_t* cache_data;
    int cache_slots;            // power of two
    int cache_stride;           // uint16 per slot (>= kmax + 1)
};

namespace {

__global__ void __launch_bounds__(32 * L15_WARPS, 8) l15_canon(L15Src src, L15Out out, L15Layout L, Binom B) {
    extern __shared__ __align__(16) unsigned char l15_smem[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = l15_smem + (size_t)wib * L.bytes;
    uint16_t* fl = reinterpret_cast<uint16_t*>(base + L.o_fl);
    uint16_t* rm = reinterpret_cast<uint16_t*>(base + L.o_rm);
    uint32_t* fb = reinterpret_cast<uint32_t*>(base + L.o_fb);
    uint32_t* mb = reinterpret_cast<uint32_t*>(base + L.o_mb);
    uint16_t* mnf = reinterpret_cast<uint16_t*>(base + L.o_mnf);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(base + L.o_keys);
    uint16_t* ids = reinterpret_cast<uint16_t*>(base + L.o_ids);
    uint16_t* seq = reinterpret_cast<uint16_t*>(base + L.o_seq);
    uint16_t* best = reinterpret_cast<uint16_t*>(base + L.o_best);
    int* misc = reinterpret_cast<int*>(base + L.o_misc);
    int* seqoff = misc;                                        // [17]
    uint16_t* clsmask = reinterpret_cast<uint16_t*>(misc + 20);  // [16]
    uint8_t* clsrange = reinterpret_cast<uint8_t*>(misc + 28);  // [2 * 16] first / last label per class
    uint32_t* rowbuf = reinterpret_cast<uint32_t*>(misc + 48);  // [gw]

    const int m = L.m;
    const uint32_t vall = (1u << m) - 1u;
    const int W = L.bmw;
    const long long count = src.rows ? (src.num ? (long long)*src.num : src.count) : src.count;
    unsigned long long n_leaves = 0, n_steps = 0;

    for (;;) {
        long long ci = 0;
        if (lane == 0) ci = (long long)atomicAdd(out.ctl, 1ull);
        ci = __shfl_sync(FULL, ci, 0);
        if (ci >= count) break;

        // ---- 0. the facet list (0-based masks, ascending)
        unsigned long long c_steps = 0;
        int k = 0;
        if (src.rows) {
            const uint32_t* row = src.rows + (size_t)(src.idx ? src.idx[ci] : ci) * L.gw;
            for (int b0 = 0; b0 < L.gw; b0 += 32) {
                const int w = b0 + lane;
                uint32_t x = w < L.gw ? row[w] : 0u;
                const int c = __popc(x);
                const int inc = warp_incl_scan(c, lane);
                int pos = k + inc - c;
                for (; x; x &= x - 1) fl[pos++] = src.unrank[w * 32 + __ffs(x) - 1];
                k += __shfl_sync(FULL, inc, 31);
            }
        } else {
            const long long a = src.off[ci];
            k = (int)(src.off[ci + 1] - a);
            for (int j = lane; j < k; j += 32) fl[j] = src.masks[a + j];
        }
        if (k > L.kmax) {  // host bug: sized below the batch
            if (lane == 0) atomicAdd(out.ctl + 1, 1ull);
            continue;
        }
        __syncwarp();
        if (k == 0) {  // isomorphism.hpp:229
            if (src.rows)
                for (int w = lane; w < L.gw; w += 32) out.rows[(size_t)ci * L.gw + w] = 0u;
            continue;
        }

        // ---- 1. face bitmap: facets, then the down-closure
        for (int w = lane; w < W; w += 32) fb[w] = 0u;
        __syncwarp();
        for (int j = lane; j < k; j += 32) atomicOr(&fb[fl[j] >> 5], 1u << (fl[j] & 31));
        __syncwarp();
        const int lowb = m < 5 ? m : 5;
        for (int w = lane; w < W; w += 32) {
            uint32_t x = fb[w];
            for (int b = 0; b < lowb; ++b) x |= (x >> (1 << b)) & low_half_mask(b);
            fb[w] = x;
        }
        __syncwarp();
        for (int b = 5; b < m; ++b) {
            const int bit = 1 << (b - 5);
            for (int w = lane; w < W; w += 32)
                if (!(w & bit)) fb[w] |= fb[w | bit];
            __syncwarp();
        }

        // ---- 2. minimal non-faces: not a face, every one-smaller subset a face.
        // The reference's face set has no empty face (faces_by_card erases it,
        // complex.hpp:185), so no singleton is ever minimal -- not even a
        // ghost vertex's (complex.hpp:199-202 candidates fail :210-217)
        if (lane == 0) fb[0] &= ~1u;
        __syncwarp();
        const uint32_t valid = m >= 5 ? FULL : ((1u << (1 << m)) - 1u);
        for (int w = lane; w < W; w += 32) {
            const uint32_t f = fb[w];
            uint32_t x = ~f & valid & (w == 0 ? ~1u : FULL);
            for (int b = 0; b < lowb; ++b) x &= (f << (1 << b)) | low_half_mask(b);
            for (int b = 5; b < m; ++b) {
                const int bit = 1 << (b - 5);
                if (w & bit) x &= fb[w ^ bit];
            }
            mb[w] = x;
        }
        __syncwarp();
        int nm = 0;
        for (int b0 = 0; b0 < W; b0 += 32) {
            const int w = b0 + lane;
            uint32_t x = w < W ? mb[w] : 0u;
            const int c = __popc(x);
            const int inc = warp_incl_scan(c, lane);
            int pos = nm + inc - c;
            for (; x; x &= x - 1, ++pos)
                if (pos < L.mnfcap) mnf[pos] = (uint16_t)(w * 32 + __ffs(x) - 1);
            nm += __shfl_sync(FULL, inc, 31);
        }
        const int ni = nm + k;
        if (nm > L.mnfcap || ni > L.P) {
            if (lane == 0) atomicAdd(out.ctl + 1, 1ull);
            continue;
        }
        __syncwarp();

        // vertex degrees over the minimal non-faces and over the facets
        int degm = 0, degf = 0;
        for (int b0 = 0; b0 < ni; b0 += 32) {
            const int j = b0 + lane;
            const uint32_t s = j < nm ? mnf[j] : (j < ni ? fl[j - nm] : 0u);
            for (int v = 0; v < m; ++v) {
                const uint32_t bal = __ballot_sync(FULL, (s >> v) & 1u);
                const int cm = __popc(bal & (b0 + 32 <= nm ? FULL : (nm <= b0 ? 0u : ((1u << (nm - b0)) - 1u))));
                if (lane == v) {
                    degm += cm;
                    degf += __popc(bal) - cm;
                }
            }
        }

        // ---- 3. refine_classes
        int rank = 0, ncls = 1;
        if (lane < 16) clsmask[lane] = lane == 0 ? (uint16_t)vall : 0;
        __syncwarp();
        for (int round = -1; round < m; ++round) {
            const bool init = round < 0;
            const int items = init ? nm : ni;
            int P = 32;
            while (P < items) P <<= 1;
            // codes (isomorphism.hpp:166-169 color sequences / :184-203 env entries)
            for (int j = lane; j < P; j += 32) {
                unsigned long long key = INF64;
                if (j < items) {
                    if (j < nm) {
                        const uint32_t s = mnf[j];
                        key = (unsigned long long)__popc(s) << 59;
                        if (!init) key |= rank_nibbles(s, clsmask, ncls, 55);
                    } else {
                        key = (1ull << 63) | rank_nibbles(fl[j - nm], clsmask, ncls, 59);
                    }
                    key |= (unsigned long long)j;
                }
                keys[j] = key;
            }
            __syncwarp();
            warp_bitonic(keys, P, lane);
            // ids: first sorted position of each code
            int carry = 0;
            for (int b0 = 0; b0 < items; b0 += 32) {
                const int p = b0 + lane;
                int id = 0;
                if (p < items) {
                    const bool head = p == 0 || (keys[p] >> 11) != (keys[p - 1] >> 11);
                    id = head ? p : 0;
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(FULL, id, o);
                    if (lane >= o) id = max(id, t);
                }
                id = max(id, carry);
                if (p < items) ids[p] = (uint16_t)id;
                carry = __shfl_sync(FULL, id, 31);
            }
            // per-vertex sorted env sequences
            const int deg = init ? degm : degm + degf;
            {
                const int inc = warp_incl_scan(lane < m ? deg : 0, lane);
                if (lane < 16) seqoff[lane] = inc - (lane < m ? deg : 0);
            }
            __syncwarp();
            int fill = 0;  // lane v: entries written for vertex v
            for (int b0 = 0; b0 < items; b0 += 32) {
                const int p = b0 + lane;
                uint32_t s = 0;
                int id = 0;
                if (p < items) {
                    const int it = (int)(keys[p] & 0x7FFull);
                    s = it < nm ? mnf[it] : fl[it - nm];
                    id = ids[p];
                }
                for (int v = 0; v < m; ++v) {
                    const uint32_t bal = __ballot_sync(FULL, (s >> v) & 1u);
                    const int f = __shfl_sync(FULL, fill, v);
                    if ((s >> v) & 1u) seq[seqoff[v] + f + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)id;
                    if (lane == v) fill += __popc(bal);
                }
            }
            __syncwarp();
            // pairwise order of the keys (rank, sequence)
            uint32_t ltm = 0, eqm = 0;  // lane v: vertices u with key(u) < / == key(v)
            for (int u = 0; u < m; ++u) {
                const int ru = __shfl_sync(FULL, rank, u);
                if (lane < m && lane != u) {
                    if (ru < rank) ltm |= 1u << u;
                }
            }
            for (int u = 0; u < m; ++u) {
                const int ru = __shfl_sync(FULL, rank, u);
                const int du = __shfl_sync(FULL, deg, u);
                for (int v = u + 1; v < m; ++v) {
                    const int rv = __shfl_sync(FULL, rank, v);
                    if (rv != ru) continue;
                    const int dv = __shfl_sync(FULL, deg, v);
                    const uint16_t* su = seq + seqoff[u];
                    const uint16_t* sv = seq + seqoff[v];
                    const int len = min(du, dv);
                    int c = (du > dv) - (du < dv);
                    for (int b0 = 0; b0 < len; b0 += 32) {
                        const int p = b0 + lane;
                        const int a = p < len ? su[p] : 0, b = p < len ? sv[p] : 0;
                        const uint32_t diff = __ballot_sync(FULL, a != b);
                        if (diff) {
                            const int q = __ffs(diff) - 1;
                            const int aq = __shfl_sync(FULL, a, q), bq = __shfl_sync(FULL, b, q);
                            c = aq < bq ? -1 : 1;
                            break;
                        }
                    }
                    // c = cmp(key u, key v)
                    if (lane == v) {
                        if (c < 0) ltm |= 1u << u;
                        if (c == 0) eqm |= 1u << u;
                    }
                    if (lane == u) {
                        if (c > 0) ltm |= 1u << v;
                        if (c == 0) eqm |= 1u << v;
                    }
                }
            }
            const uint32_t firsts = __ballot_sync(FULL, lane < m && (eqm & ((1u << lane) - 1u)) == 0u);
            const int nrank = __popc(ltm & firsts);
            const int nc = __popc(firsts);
            if (!init && nc == ncls) break;  // :211-214
            rank = lane < m ? nrank : 0;
            ncls = nc;
            for (int r = 0; r < 16; ++r) {
                const uint32_t cm = __ballot_sync(FULL, lane < m && rank == r);
                if (lane == r) clsmask[r] = (uint16_t)cm;
            }
            __syncwarp();
        }
        if (out.cls && lane < 16) out.cls[ci * 16 + lane] = lane < m ? (int8_t)rank : (int8_t)-1;
        // isomorphism-invariant key: the last round's sorted entry codes
        // (ranks are class ids, item indices masked off) and the classes
        unsigned long long hkey = 0;
        if (out.cache_key) {
            for (int q = lane; q < ni; q += 32) hkey += mix64((keys[q] >> 11) ^ ((unsigned long long)q << 52));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) hkey += __shfl_xor_sync(FULL, hkey, o);
            hkey = mix64(hkey ^ ((unsigned long long)k << 32) ^ ((unsigned long long)ncls << 48) ^
                         (unsigned long long)m) | (1ull << 63);
        }

        bool no_seed = false;
    phase4:
        // ---- 4. least relabeled facet list over the class-respecting labelings
        // (class c owns the c-th consecutive label range, :232-288), by an
        // exact branch and bound over single placements.  Two placement
        // orders, both enumerating every such labeling:
        //  * facet mode: labels 0, 1, ... in turn.  Each facet's final mask
        //    is at least its placed labels plus, per class, the lowest labels
        //    that class still has free for the facet's unplaced vertices (a
        //    facet that is complete is exact).  The final ascending list then
        //    dominates the ascending list of these bounds elementwise, so if
        //    the bounds' list is above the best list at their first
        //    difference, every completion is: prune.  In counts: with x_B =
        //    the least best mask no bound hits and x_L = the least bound
        //    value hit more often than the best list has it, prune iff x_B <
        //    x_L;
        //  * co-facet mode: labels m-1, m-2, ... in turn, on the co-facets
        //    [m] \ F.  The facet list ascending is least iff the co-facet
        //    list descending is greatest (complement reverses the order);
        //    bounds from above (the highest free labels per class), mirror
        //    rule with maxima.
        // Co-facets of a Picard-4 complex have 4 vertices, so their bounds
        // tighten after 4 placements where facet bounds need ~n.
        const bool comode = L.mode == 2 || (L.mode == 0 && (m - L.n) <= L.n);
        int myslotcls = 0;  // lane s: class of the label placed at depth s
        {
            const int lab = comode ? m - 1 - lane : lane;
            int acc = 0;
            for (int r = 0; r < ncls; ++r) {
                const int sz = __popc(clsmask[r]);
                if (lab >= acc && lab < acc + sz) myslotcls = r;
                if (lane == r) {
                    clsrange[2 * r] = (uint8_t)acc;
                    clsrange[2 * r + 1] = (uint8_t)(acc + sz - 1);
                }
                acc += sz;
            }
        }
        unsigned long long rankpack = 0;  // 4-bit class of every vertex
        for (int v = 0; v < m; ++v) rankpack |= (unsigned long long)(__shfl_sync(FULL, rank, v) & 15) << (4 * v);
        for (int w = lane; w < W; w += 32) {
            fb[w] = 0u;  // scratch: bound values of the current node
            mb[w] = 0u;  // best list
        }
        for (int j = lane; j < k; j += 32) rm[j] = 0;
        __syncwarp();
        uint16_t* bnd = reinterpret_cast<uint16_t*>(base + L.o_bnd);  // per item: its bound at the current node
        bool have_best = false;
        uint32_t taken = 0;
        int t = 0;
        int my_v = 0;           // lane t: vertex placed at depth t
        uint32_t my_tried = 0;  // lane t: vertices tried at depth t
        int best_v = -1;        // lane t: vertex at depth t on the best leaf's path
        int ngen = 0;                 // automorphisms found (lane g holds number g)
        unsigned long long gen = 0;   // lane g: image of every vertex, 4 bits each
        uint32_t gen_fix = 0;         // lane g: the vertices it fixes
        auto item_of = [&](int j) -> uint32_t { return comode ? (vall & ~(uint32_t)fl[j]) : (uint32_t)fl[j]; };
        // a cached canonical form with the same invariant key seeds the
        // best.  A leaf equal to it proves K is isomorphic to the cached
        // complex (the leaf IS the cached list), so the search stops there:
        // its minimum is the cached one.  If the seed is not reachable
        // (not isomorphic), either a real leaf beats it or nothing survives
        // and the search reruns unseeded.
        const unsigned cslot = out.cache_key ? (unsigned)(hkey & (unsigned long long)(out.cache_slots - 1)) : 0u;
        bool seeded = false, found = false, real_best = false;
        // seed only where a fresh search is expensive: the labelings of the
        // class structure (prod of class-size factorials) exceed 7!; below
        // that the fresh search (with its automorphism pruning) measured
        // cheaper than confirming a cached form
        double labelings_bound = 1.0;
        for (int r = 0; r < ncls; ++r)
            for (int q = 2; q <= __popc(clsmask[r]); ++q) labelings_bound *= q;
        if (out.cache_key && !no_seed && labelings_bound > 5040.0) {
            unsigned long long ck = 0;
            if (lane == 0) ck = *(volatile unsigned long long*)(out.cache_key + cslot);
            ck = __shfl_sync(FULL, ck, 0);
            if (ck == hkey) {
                __threadfence();
                const uint16_t* cd = out.cache_data + (size_t)cslot * out.cache_stride;
                if ((int)__ldcg(cd) == k) {
                    for (int j = lane; j < k; j += 32) {
                        // facet list ascending -> item list ascending
                        const uint32_t f = __ldcg(cd + 1 + (comode ? k - 1 - j : j));
                        const uint32_t it = comode ? (vall & ~f) : f;
                        best[j] = (uint16_t)it;
                        atomicOr(&mb[it >> 5], 1u << (it & 31));
                    }
                    __syncwarp();
                    seeded = have_best = true;
                }
            }
        }
        auto undo = [&](int v, int tt) {
            const uint32_t vb = 1u << v;
            const int lab = comode ? m - 1 - tt : tt;
            for (int j = lane; j < k; j += 32)
                if (item_of(j) & vb) rm[j] = (uint16_t)(rm[j] & ~(1u << lab));
            taken &= ~vb;
            __syncwarp();
        };
        for (;;) {
            const int scls = __shfl_sync(FULL, myslotcls, t);
            const uint32_t tried = __shfl_sync(FULL, my_tried, t);
            uint32_t cand = clsmask[scls] & ~taken & ~tried;
            if (ngen && tried && cand) {
                // orbit pruning: a candidate in the orbit of a finished
                // sibling under the found automorphisms that fix this prefix
                // pointwise roots an image of that sibling's subtree
                const bool use = lane < ngen && (taken & ~gen_fix) == 0u;
                uint32_t orb = tried;
                for (;;) {
                    uint32_t img = 0;
                    if (use)
                        for (uint32_t x = orb; x; x &= x - 1)
                            img |= 1u << (uint32_t)((gen >> (4 * (__ffs(x) - 1))) & 15ull);
                    img = __reduce_or_sync(FULL, img) | orb;
                    if (img == orb) break;
                    orb = img;
                }
                cand &= ~orb;
            }
            if (!cand) {
                if (lane == t) my_tried = 0;
                if (t == 0) break;
                --t;
                undo(__shfl_sync(FULL, my_v, t), t);
                continue;
            }
            const int v = __ffs(cand) - 1;
            if (lane == t) {
                my_tried |= 1u << v;
                my_v = v;
            }
            ++n_steps;
            ++c_steps;
            const int lab = comode ? m - 1 - t : t;
            taken |= 1u << v;
            // place v; bound every item; mark the bound values (dups = hit twice)
            uint32_t xu = comode ? 0u : INF32;  // extreme bound value the best list lacks or has fewer of
            bool incomplete = false;
            for (int j = lane; j < k; j += 32) {
                const uint32_t f = item_of(j);
                uint32_t r = rm[j];
                if ((f >> v) & 1u) {
                    r |= 1u << lab;
                    rm[j] = (uint16_t)r;
                }
                uint32_t free_v = f & ~taken;
                incomplete |= free_v != 0u;
                unsigned long long used = 0;  // 4-bit per-class count of free labels taken
                for (; free_v; free_v &= free_v - 1) {
                    const int u = __ffs(free_v) - 1;
                    const int cl = (int)((rankpack >> (4 * u)) & 15ull);
                    const int c = (int)((used >> (4 * cl)) & 15ull);
                    used += 1ull << (4 * cl);
                    if (comode) r |= 1u << (min((int)clsrange[2 * cl + 1], lab - 1) - c);
                    else r |= 1u << (max((int)clsrange[2 * cl], t + 1) + c);
                }
                bnd[j] = (uint16_t)r;
                const uint32_t old = atomicOr(&fb[r >> 5], 1u << (r & 31));
                if (have_best) {
                    const bool dup = (old >> (r & 31)) & 1u;
                    const bool in_best = (mb[r >> 5] >> (r & 31)) & 1u;
                    if (dup || !in_best) xu = comode ? max(xu, r + 1u) : min(xu, r);
                }
            }
            __syncwarp();
            const bool leaf = t == m - 1 || (comode && !__any_sync(FULL, incomplete));
            int verdict = 1;  // -1 prune, 0 equal to the best (leaf), 1 continue / new best
            if (have_best) {
                uint32_t xb = comode ? 0u : INF32;  // extreme best value no bound hits
                for (int j = lane; j < k; j += 32) {
                    const uint32_t b = best[j];
                    if (!((fb[b >> 5] >> (b & 31)) & 1u)) xb = comode ? max(xb, b + 1u) : min(xb, b);
                }
                if (comode) {
                    xu = __reduce_max_sync(FULL, xu);
                    xb = __reduce_max_sync(FULL, xb);
                    verdict = xb > xu ? -1 : (xb == 0u && xu == 0u ? 0 : 1);
                } else {
                    xu = __reduce_min_sync(FULL, xu);
                    xb = __reduce_min_sync(FULL, xb);
                    verdict = xb < xu ? -1 : (xb == INF32 && xu == INF32 ? 0 : 1);
                }
            }
            int jump = -1;
            if (leaf && verdict == 0 && seeded && !real_best) {
                ++n_leaves;
                found = true;  // K is isomorphic to the cached complex
                break;
            }
            if (leaf) {
                // every bound is exact here: a new best iff the list is below the best
                ++n_leaves;
                if (verdict == 0) {
                    // a leaf equal to the best: best^-1 o current is an
                    // automorphism fixing the common prefix of the two paths
                    // and mapping this path's vertex at the first differing
                    // depth d onto the best path's -- so this depth-d branch
                    // is the image of the (finished) branch that holds the
                    // best, and nothing under it can be below the best
                    const uint32_t diff = __ballot_sync(FULL, lane <= t && my_v != best_v);
                    if (diff) jump = __ffs(diff) - 1;
                    if (diff && ngen < 32) {  // keep the automorphism: my_v[d] -> best_v[d], identity elsewhere
                        unsigned long long g = 0;
                        uint32_t moved = 0;
                        for (int d = 0; d <= t; ++d) {
                            const int a = __shfl_sync(FULL, my_v, d), b = __shfl_sync(FULL, best_v, d);
                            g |= (unsigned long long)b << (4 * a);
                            if (a != b) moved |= 1u << a;
                        }
                        for (uint32_t x = vall & ~taken; x; x &= x - 1) {
                            const int a = __ffs(x) - 1;
                            g |= (unsigned long long)a << (4 * a);
                        }
                        if (lane == ngen) {
                            gen = g;
                            gen_fix = vall & ~moved;
                        }
                        ++ngen;
                    }
                }
                if (verdict > 0) {
                    real_best = true;
                    best_v = lane <= t ? my_v : -1;
                    for (int w = lane; w < W; w += 32) mb[w] = fb[w];
                    __syncwarp();
                    int kk = 0;
                    for (int b0 = 0; b0 < W; b0 += 32) {
                        const int w = b0 + lane;
                        uint32_t y = w < W ? mb[w] : 0u;
                        const int c = __popc(y);
                        const int inc = warp_incl_scan(c, lane);
                        int pos = kk + inc - c;
                        for (; y; y &= y - 1) best[pos++] = (uint16_t)(w * 32 + __ffs(y) - 1);
                        kk += __shfl_sync(FULL, inc, 31);
                    }
                    have_best = true;
                }
            }
            for (int j = lane; j < k; j += 32) {
                const uint32_t r = bnd[j];
                atomicAnd(&fb[r >> 5], ~(1u << (r & 31)));
            }
            __syncwarp();
            if (leaf || verdict < 0) {
                undo(v, t);
                while (jump >= 0 && t > jump) {
                    if (lane == t) my_tried = 0;
                    --t;
                    undo(__shfl_sync(FULL, my_v, t), t);
                }
                continue;
            }
            ++t;
            if (lane == t) my_tried = 0;
        }
        if (seeded && !found && !real_best) {  // the seed was out of reach: search again, unseeded
            no_seed = true;
            goto phase4;
        }
        if (found && lane == 0) atomicAdd(out.ctl + 4, 1ull);
        // best[] holds the ascending list of facet masks (facet mode) or of
        // co-facet masks (co-facet mode: facet j is the complement of
        // best[k - 1 - j])
        if (comode) {
            __syncwarp();
            for (int j = lane; j < k; j += 32) rm[j] = (uint16_t)(vall & ~(uint32_t)best[k - 1 - j]);
            __syncwarp();
            for (int j = lane; j < k; j += 32) best[j] = rm[j];
            __syncwarp();
        }
        if (out.cache_key && !found && k + 1 <= out.cache_stride) {
            // publish this canonical form (write-once slot: claim, fill, release)
            int claimed = 0;
            if (lane == 0) claimed = atomicCAS(out.cache_key + cslot, 0ull, 1ull) == 0ull;
            if (__shfl_sync(FULL, claimed, 0)) {
                uint16_t* cd = out.cache_data + (size_t)cslot * out.cache_stride;
                for (int j = lane; j < k; j += 32) cd[1 + j] = best[j];
                if (lane == 0) cd[0] = (uint16_t)k;
                __threadfence();
                __syncwarp();
                if (lane == 0) atomicExch(out.cache_key + cslot, hkey);
            }
        }

        // ---- output
        if (out.cost && lane == 0) out.cost[ci] = c_steps;
        if (src.rows) {
            for (int w = lane; w < L.gw; w += 32) rowbuf[w] = 0u;
            __syncwarp();
            for (int j = lane; j < k; j += 32) {
                const uint32_t g = colex_rank(best[j], B);
                atomicOr(&rowbuf[g >> 5], 1u << (g & 31));
            }
            __syncwarp();
            for (int w = lane; w < L.gw; w += 32) out.rows[(size_t)ci * L.gw + w] = rowbuf[w];
        } else {
            const long long a = src.off[ci];
            for (int j = lane; j < k; j += 32) out.masks[a + j] = best[j];
        }
        __syncwarp();
    }
    if (lane == 0) {
        atomicAdd(out.ctl + 2, n_leaves);
        atomicAdd(out.ctl + 3, n_steps);
    }
}

// ---- first-appearance dedupe of the canonical rows (pipeline.hpp:97-100):
// kernel 4's record sort orders (row, survivor index) -- the index rides in
// the record as a payload word that breaks ties -- so the head of each run of
// equal rows carries the run's first appearance; heads mark is_rep[index];
// compacting is_rep over the survivor order gives the representatives in
// order of first appearance.  No library code.
__global__ void pack_rows_payload(const uint32_t* __restrict__ rows, int gw, long long n, int rw,
                                  uint32_t* __restrict__ recs) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * rw) return;
    const long long r = t / rw;
    const int w = (int)(t - r * rw);
    recs[t] = w < gw ? rows[(size_t)r * gw + w] : (w == gw ? (uint32_t)r : 0u);  // payload, padding, map 0
}

__global__ void iota_idx(uint32_t* idx, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) idx[i] = (uint32_t)i;
}

__global__ void mark_first(const uint32_t* __restrict__ sorted, int gw, const uint32_t* __restrict__ payload,
                           long long n, uint8_t* __restrict__ is_rep) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    bool head = p == 0;
    for (int w = 0; w < gw && !head; ++w) head = sorted[(size_t)p * gw + w] != sorted[(size_t)(p - 1) * gw + w];
    if (head) is_rep[payload[p]] = 1;
}

__global__ void gather_rows15(const uint32_t* __restrict__ rows, int gw, const uint32_t* __restrict__ idx,
                              long long n, uint32_t* __restrict__ out) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * gw) return;
    const long long r = t / gw;
    const int w = (int)(t - r * gw);
    out[t] = rows[(size_t)idx[r] * gw + w];
}

__global__ void max_facets(const uint32_t* __restrict__ rows, int gw, const uint32_t* __restrict__ idx,
                           long long n, int* __restrict__ out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int c = 0;
    if (i < n) {
        const uint32_t* r = rows + (size_t)(idx ? idx[i] : (uint32_t)i) * gw;
        for (int w = 0; w < gw; ++w) c += __popc(r[w]);
    }
    c = __reduce_max_sync(FULL, c);
    if ((threadIdx.x & 31) == 0 && c > 0) atomicMax(out, c);
}

}  // namespace

int l15_max_facets(const uint32_t* d_rows, int gw, const uint32_t* d_idx, long long count, int* d_out,
                   cudaStream_t st) {
    if (cudaMemsetAsync(d_out, 0, sizeof(int), st) != cudaSuccess) return 1;
    if (count <= 0) return 0;
    max_facets<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d_rows, gw, d_idx, count, d_out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

L15Layout l15_layout(int m, int n, int kmax, int mnfcap, int gw) {
    L15Layout L{};
    L.m = m;
    L.n = n;
    L.kmax = std::max(kmax, 1);
    L.mnfcap = std::max(mnfcap, 32);
    int P = 32;
    while (P < L.kmax + L.mnfcap) P <<= 1;
    L.P = P;
    L.seqcap = n * L.kmax + (n + 1) * L.mnfcap;
    L.bmw = m >= 5 ? (1 << (m - 5)) : 1;
    L.gw = gw;
    // placement order: 0 = by shape (co-facets when they are the smaller side),
    // 1 = facets, 2 = co-facets; WPM_L15_MODE overrides (experiments)
    L.mode = 0;
    if (const char* e = std::getenv("WPM_L15_MODE")) L.mode = std::atoi(e);
    auto al = [](int x) { return (x + 15) & ~15; };
    // phase-3 scratch (sort keys, ids, env sequences) overlays the two
    // bitmaps: the face / non-face bitmaps are dead once the minimal
    // non-faces are listed, the current / best bitmaps are born after the
    // classes are refined
    L.o_fb = 0;
    L.o_mb = al(L.bmw * 4);
    const int end4 = L.o_mb + al(L.bmw * 4);
    L.o_keys = 0;
    L.o_ids = al(P * 8);
    L.o_seq = L.o_ids + al(P * 2);
    const int end3 = L.o_seq + al(L.seqcap * 2);
    int o = std::max(end3, end4);
    L.o_misc = o;  o += al((48 + std::max(gw, 1)) * 4);
    L.o_fl = o;    o += al(L.kmax * 2);
    L.o_rm = o;    o += al(L.kmax * 2);
    L.o_best = o;  o += al(L.kmax * 2);
    L.o_bnd = o;   o += al(L.kmax * 2);
    L.o_mnf = o;   o += al(L.mnfcap * 2);
    L.bytes = o;
    return L;
}

size_t l15_smem_bytes(const L15Layout& L) { return (size_t)L.bytes * L15_WARPS; }

int l15_launch(const L15Layout& L, const uint32_t* d_rows, const uint32_t* d_idx, const int* d_num,
               const uint16_t* d_unrank, const uint16_t* d_masks, const long long* d_off, long long count,
               uint32_t* d_out_rows, uint16_t* d_out_masks, int8_t* d_cls, unsigned long long* d_cost,
               unsigned long long* d_ctl, unsigned long long* d_cache_key, uint16_t* d_cache_data, int cache_slots,
               int num_sms, cudaStream_t st) {
    if (count <= 0) return 0;
    const size_t smem = l15_smem_bytes(L);
    if (smem > 227 * 1024) return 1;
    if (cudaFuncSetAttribute(l15_canon, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, l15_canon, 32 * L15_WARPS, smem) != cudaSuccess ||
        per_sm < 1)
        return 1;
    const long long blocks = std::min<long long>((count + L15_WARPS - 1) / L15_WARPS, (long long)num_sms * per_sm);
    L15Src src{d_rows, d_idx, d_num, d_unrank, d_masks, d_off, count};
    L15Out out{d_out_rows, d_out_masks, d_cls, d_cost, d_ctl, d_cache_key, d_cache_data, cache_slots,
               L.kmax + 1};
    if (cudaMemsetAsync(d_ctl, 0, 5 * sizeof(unsigned long long), st) != cudaSuccess) return 1;
    if (d_cache_key &&
        cudaMemsetAsync(d_cache_key, 0, (size_t)cache_slots * sizeof(unsigned long long), st) != cudaSuccess)
        return 1;
    l15_canon<<<(unsigned)blocks, 32 * L15_WARPS, smem, st>>>(src, out, L, make_binom());
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// temp: the records, the sort's two record buffers, the sorted rows, the
// compaction's block counts
size_t l15_dedupe_temp_bytes(long long count, int gw) {
    const size_t rw = (size_t)rec_words(gw + 1);
    return (size_t)count * rw * 4 * 3 + (size_t)count * gw * 4 + compact_temp_bytes() + 1024;
}

// rows: count canonical rows; out: d_rep (indices of the first appearances,
// ascending), *d_nrep; scratch d_sidx (count: the sorted payloads), d_first
// (count: is_rep)
int l15_dedupe(const uint32_t* d_rows, long long count, int gw, uint32_t* d_sidx, uint32_t* d_iota, uint8_t* d_first,
               uint32_t* d_rep, int* d_nrep, void* d_temp, size_t temp_bytes, cudaStream_t st) {
    if (count <= 0) return cudaMemsetAsync(d_nrep, 0, sizeof(int), st) == cudaSuccess ? 0 : 1;
    iota_idx<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d_iota, count);  // the survivor order (fetch 14)
    if (temp_bytes < l15_dedupe_temp_bytes(count, gw)) return 1;
    const int rw = rec_words(gw + 1);
    uint32_t* recs = static_cast<uint32_t*>(d_temp);
    uint32_t* sort_tmp = recs + (size_t)count * rw;
    uint32_t* sorted = sort_tmp + (size_t)count * rw * 2;
    void* ctemp = sorted + (size_t)count * gw;
    const long long t = count * rw;
    pack_rows_payload<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(d_rows, gw, count, rw, recs);
    if (canon_sort_records(recs, count, gw, rw, gw, sorted, nullptr, d_sidx, sort_tmp,
                           (size_t)count * rw * 4 * 2, nullptr, nullptr, st))
        return 1;
    if (cudaMemsetAsync(d_first, 0, (size_t)count, st) != cudaSuccess) return 1;
    mark_first<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(sorted, gw, d_sidx, count, d_first);
    if (compact_flagged(nullptr, d_first, count, d_rep, d_nrep, ctemp, st)) return 1;
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int l15_gather(const uint32_t* d_rows, int gw, const uint32_t* d_idx, long long count, uint32_t* d_out,
               cudaStream_t st) {
    if (count <= 0) return 0;
    const long long t = count * gw;
    gather_rows15<<<(unsigned)((t + 255) / 256), 256, 0, st>>>(d_rows, gw, d_idx, count, d_out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace wpm
