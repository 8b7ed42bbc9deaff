// k3_search.cu -- kernel 3: the ridge-driven backtracking search.
//
// Replaces the body of enumerate_wpm (search.hpp:141-258): the kernel-basis
// odometer (:192-245) and its per-leaf ridge recount wpm_counts_ok
// (:114-131) become a depth-first search that only ever builds partial
// complexes whose ridge counts are <= 2:
//
//   include f : every ridge of f gains a count; a ridge reaching 2 excludes
//               its remaining candidate facets (a 3rd would break Prop. 2.1,
//               PAPER.md:206-208); the state is dead once an open ridge
//               (count 1) has no undecided candidate left.
//   open node : prune if |S| + ceil(open/n) > cap (the UBT count cap,
//               affine_property.hpp:49-54, search.hpp:181-187); branch on the
//               open ridge with the fewest undecided candidates (ties: lowest
//               ridge id) over "include u_i, exclude u_1..u_{i-1}".
//   closed    : (no open ridge) emit S if nonempty; if |S| + n + 1 <= cap,
//   node        branch "include f, exclude every undecided facet < f" (the
//               next ridge-disjoint component by its minimum facet).
//
// Branches partition the solution space, so every WPM is produced exactly
// once and the final sort/unique (search.hpp:254-256) finds no duplicate.
//
// 87-97 % of branch points have a single undecided candidate (measured on
// the CPU restatement, n = 5..11): those FORCED moves run as a chain inside
// one descent -- no frame, no sibling exclusion -- and unwind with one
// undo_to.  Frames exist only for real branch points.  The open ridges with
// exactly one undecided candidate are kept in a bitset, so the MRV choice is
// a first-set-bit lookup; the full (undecided, id) min-scan over the open
// bitset runs only when that bitset is empty.
//
// Execution model (B200): a persistent grid, one DFS per warp.  Lanes
// cooperate on each node: lane k < n updates the k-th ridge of the included
// facet; exclusions are flattened (facet, ridge) pairs over 32 lanes with
// shared-memory atomics; branch choices are __ballot_sync / __reduce_min_sync.
// The per-warp state lives in shared memory (ridge count + undecided count
// packed in one byte, facet status, an undo trail, the frame stack); every
// helper is inlined so the warp's scalars stay in registers and all state
// accesses are LDS/STS/ATOMS.  Per-map tables are read-only global memory
// (L1 resident).
//
// Work sharing replaces parallel_for_index (parallel.hpp:27-54): a global
// ticket queue of tasks (IN/OUT facet bitsets + the frame to resume).  Every
// few nodes a busy warp looks at a prefetched (head, tail) word; if warps are
// waiting it donates its shallowest frame that still has untried children
// (it marks the frame exhausted and keeps going).  The tree is the same
// whoever explores it, so node counts are deterministic.
#include <cstdint>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

#include "wpm_dev.cuh"
#include "wpm_internal.h"

namespace wpm {

namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint8_t FU = 0, FIN = 1, FOUT = 2;
constexpr uint16_t TR_INC = 0x8000;
constexpr uint32_t CLOSED_FRAME = 0xFFFFu;
constexpr uint32_t POS_DONE = 0xFFFFu;
constexpr uint32_t NO_CHILD = 0xFFFFu;
constexpr int FRAME_CAP = 64;    // frame stack of the fast layouts (measured depth <= 37)

enum TaskKind : uint32_t { T_SINGLE = 0, T_OPEN = 1, T_CLOSED = 2, T_ENTRY = 3 };

constexpr int a16(int x) { return (x + 15) & ~15; }

// Per-warp shared-memory layout of one size class: every offset is a
// compile-time constant, so each shared access is (warp base register +
// immediate + index) -- one register for the whole state, no address
// conversions in the PTX helpers.
// TSM: the per-map tables (fr, rp of every map of the plan) are copied into
// shared memory at kernel start and read with LDS (they are the L1-missing
// loads of the global-table layout: 20-27 % long-scoreboard stalls); the CTA
// then holds WPBV warps sharing one copy.  Used when every map's tables fit.
// MAV (map-affine, TSM layouts only): one work queue per map; a CTA works on
// one map at a time with only THAT map's tables in shared memory, and moves to
// the map with the most pending tasks per CTA once its map is finished -- the
// TS layout for plans whose maps' tables do not fit together (n = 7..10).
template <int NMAX, int MMAX, int DMAX, bool TSM = false, int WPBV = 4, int MINBV = 0, bool MAV = false>
struct LC {
    static constexpr int kN = NMAX, kM = MMAX, kDepth = DMAX;
    static constexpr bool TS = TSM;
    static constexpr bool MA = MAV;
    static_assert(!MAV || TSM, "map-affine layouts keep the tables in shared memory");
    static constexpr int WPB = WPBV;
    static constexpr int NP = a16(NMAX + 32), MP = a16(MMAX + 32);
    static constexpr int NW = (NMAX + 31) / 32, MW = (MMAX + 31) / 32;
    static constexpr int RS = 0;                           // uint8 per ridge: count | undecided << 2
    static constexpr int FST = RS + NP;                    // uint8 per facet: U / IN / OUT
    static constexpr int OPEN = FST + MP;                  // open ridges (count 1)
    static constexpr int B1 = OPEN + a16(4 * NW + 4);      // open ridges with one undecided candidate
    static constexpr int INB = B1 + a16(4 * NW + 4);       // IN facet bitset
    static constexpr int LATE = INB + a16(4 * MW + 4);     // donation scratch
    static constexpr int TRAIL = LATE + a16(4 * MW + 4);   // uint16 per decision (bit 15: include)
    static constexpr int FRAMES = TRAIL + a16(2 * MP);     // uint2 per branch frame
    static constexpr int NOPEN = FRAMES + a16(8 * (DMAX + 2));    // uint16 per frame: open ridges at its mark
    static constexpr int SCRATCH = NOPEN + a16(2 * (DMAX + 2));   // closing-ridge list
    static constexpr int META = SCRATCH + 64;                      // task scalars kept out of registers
    static constexpr int BYTES = META + 16;
    // CTAs per SM the register budget is cut for: 10 (48 registers, no
    // spills) up to the n = 8 shapes -- measured +1.5 / +5 / +6 % nodes/s
    // at n = 5 / 6 / 8 over 8 CTAs (64 registers) -- and 8 for the larger
    // shapes, whose shared state caps residency anyway (n = 11: -3 % at 10)
#ifdef K3_MIN_BLOCKS
    static constexpr int MIN_BLOCKS = TSM ? MINBV : K3_MIN_BLOCKS;
#else
    static constexpr int MIN_BLOCKS = TSM ? MINBV : (NMAX <= 720 ? 10 : 8);
#endif
};

// size classes (max ridges, max facets, frame capacity): the exact shapes of
// the Picard-4 universes per n (max N, max M over the maps), so the per-warp
// state is no larger than needed and L1 keeps room for the per-map tables,
// plus the general layouts
using C5 = LC<128, 128, FRAME_CAP>;       // n <= 5
using C6 = LC<232, 136, FRAME_CAP>;
using C7 = LC<420, 208, FRAME_CAP>;
using C8 = LC<720, 312, FRAME_CAP>;
using C9 = LC<1152, 440, FRAME_CAP>;
using C10 = LC<1792, 616, FRAME_CAP>;
using C11 = LC<2688, 840, FRAME_CAP>;
using CG = LC<4096, 2048, FRAME_CAP>;     // any universe within the device limits
// shared-memory-table variants (warps per CTA x CTAs per SM sized so the
// tables + per-warp state fit 227 KB and the registers 64 K)
using C5T = LC<128, 128, FRAME_CAP, true, 20, 2>;    // n <= 5: all 35 maps' tables ~70 KB per CTA
using C6T = LC<232, 136, FRAME_CAP, true, 32, 1>;    // n = 6: ~137 KB
using C10T = LC<1792, 616, FRAME_CAP, true, 24, 1>;  // n = 10: ~90 KB
// n = 11: ~45 KB of tables + 27 warps x 6.8 KB of state.  A 40-frame stack
// (measured depth <= 37 at n = 11; deeper runs redo with the full-depth
// class) frees 240 B per warp, so 27 warps fit instead of 24 (64 frames):
// n = 11 17.8 -> 17.2 ms (26 warps: 17.4; profiles/r02d_ab_c11.jsonl)
#ifndef K3_C11_WARPS
#define K3_C11_WARPS 27
#endif
#ifndef K3_C11_DEPTH
#define K3_C11_DEPTH 40
#endif
using C11T = LC<2688, 840, K3_C11_DEPTH, true, K3_C11_WARPS, 1>;
// any (m, n) = (15, 11) universe (the synthetic band, up to all 1365 11-subsets)
using C15 = LC<3008, 1368, FRAME_CAP>;
using C15T = LC<3008, 1368, FRAME_CAP, true, 18, 1>;
using C7M = LC<420, 208, FRAME_CAP, true, 20, 2, true>;   // n = 7: one map's tables (~8 KB) per CTA
using C8M = LC<720, 312, FRAME_CAP, true, 20, 2, true>;   // n = 8: ~14 KB
// n = 9: 18 warps x 2 CTAs with a 40-frame stack (measured 35.0 -> 34.3 ms;
// 20 x 2 at 48 registers spilled and lost); n = 10 keeps 16 x 2 (18 or 20
// warps measured 7-9 % slower there: 3 maps, longer per-map tails) --
// profiles/r02d_ab_mq.jsonl
#ifndef K3_C9M_WARPS
#define K3_C9M_WARPS 18
#endif
#ifndef K3_C9M_DEPTH
#define K3_C9M_DEPTH 40
#endif
#ifndef K3_C10M_WARPS
#define K3_C10M_WARPS 16
#endif
using C9M = LC<1152, 440, K3_C9M_DEPTH, true, K3_C9M_WARPS, 2, true>;  // n = 9: ~20 KB (41.9 -> 39.6 ms)
using C10M = LC<1792, 616, FRAME_CAP, true, K3_C10M_WARPS, 2, true>; // n = 10: ~30 KB, 32 warps per SM (32.5 -> 29.8 ms)
// (10 x 4 and 8 x 5 warps x CTAs measured within 1 % of 20 x 2 at n = 7, 8)
// (n = 9's seven maps need ~140 KB of tables: 16 warps per SM measured 34 %
// slower than the global-table layout at 32 -- no all-maps TS variant for n = 7..9)
using CGF = LC<4096, 2048, 2050>;         // full depth: the rerun after a frame overflow

struct MapView {
    int M, N, n, cap, map, nw;
    int capn;       // min(cap, 2^20): the open-ridge prune in 32-bit arithmetic
    int lpf_shift;  // lanes per facet in flattened passes: 1 << lpf_shift >= n
    unsigned nmag;  // ceil(2^20 / n): j / n = (j * nmag) >> 20 for every pair index j < 2^20 / n
    const uint16_t* fr;
    const uint16_t* rp;
    uint32_t frs, rps;  // the same tables in shared memory (TS layouts)
    int fs, ps;     // strides of fr (= n) and rp (<= 8, 0xFFFF padded)
};

// the warp's search state: its shared region + register scalars
template <class C>
struct WS {
    uint8_t* base;  // generic pointer to the warp's region (shared)
    uint32_t sb;    // the same as a 32-bit shared-window address
    int size, nopen, tl, depth;
    int ndead;  // nonzero iff some open ridge has no undecided candidate (a dead state is always abandoned)
    __device__ __forceinline__ uint8_t* rs() const { return base + C::RS; }
    __device__ __forceinline__ uint8_t* fst() const { return base + C::FST; }
    __device__ __forceinline__ uint32_t* open() const { return reinterpret_cast<uint32_t*>(base + C::OPEN); }
    __device__ __forceinline__ uint32_t* b1() const { return reinterpret_cast<uint32_t*>(base + C::B1); }
    __device__ __forceinline__ uint32_t* inb() const { return reinterpret_cast<uint32_t*>(base + C::INB); }
    __device__ __forceinline__ uint32_t* late() const { return reinterpret_cast<uint32_t*>(base + C::LATE); }
    __device__ __forceinline__ uint16_t* trail() const { return reinterpret_cast<uint16_t*>(base + C::TRAIL); }
    __device__ __forceinline__ uint2* frames() const { return reinterpret_cast<uint2*>(base + C::FRAMES); }
    __device__ __forceinline__ uint16_t* nopen_at() const { return reinterpret_cast<uint16_t*>(base + C::NOPEN); }
    __device__ __forceinline__ uint16_t* scratch() const { return reinterpret_cast<uint16_t*>(base + C::SCRATCH); }
    // [0] absolute branch depth of frames[0] (the root's closed frame is
    // depth 0), [1] root task id of the current task (progress accounting)
    __device__ __forceinline__ int dbase() const { return reinterpret_cast<const int*>(base + C::META)[0]; }
    __device__ __forceinline__ uint32_t root() const { return reinterpret_cast<const uint32_t*>(base + C::META)[1]; }
    // shared-window addresses for the PTX helpers
    __device__ __forceinline__ uint32_t a_rs_word(int r) const { return sb + C::RS + (r & ~3); }
    __device__ __forceinline__ uint32_t a_rs(int r) const { return sb + C::RS + r; }
    __device__ __forceinline__ uint32_t a_fst(int f) const { return sb + C::FST + f; }
    __device__ __forceinline__ uint32_t a_open(int r) const { return sb + C::OPEN + ((r >> 5) << 2); }
    __device__ __forceinline__ uint32_t a_b1(int r) const { return sb + C::B1 + ((r >> 5) << 2); }
    __device__ __forceinline__ uint32_t a_inb(int f) const { return sb + C::INB + ((f >> 5) << 2); }
    __device__ __forceinline__ uint32_t a_trail(int e) const { return sb + C::TRAIL + 2 * e; }
    __device__ __forceinline__ uint32_t a_scratch(int j) const { return sb + C::SCRATCH + 2 * j; }
};

__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// the work queue of map q: its control words ([0] tail << 32 | head, [1] CTAs
// on the map, [2] pending), ready flags and record ring.  Map-affine layouts
// keep one queue per map after the plan-wide counters (qctl[0..7]); the others
// one queue in qctl[0..7] itself
template <class C>
__device__ __forceinline__ unsigned long long* q_ctl(const SearchParams& p, int q) {
    return C::MA ? p.qctl + 8 * (q + 1) : p.qctl;
}
template <class C>
__device__ __forceinline__ unsigned long long* q_ready(const SearchParams& p, int q) {
    return C::MA ? p.qready + (size_t)q * p.qcap : p.qready;
}
template <class C>
__device__ __forceinline__ uint32_t* q_rec(const SearchParams& p, int q) {
    return C::MA ? p.qrec + (size_t)q * p.qcap * p.recw : p.qrec;
}

// per-map table reads: the k-th ridge of a facet (fr), the q-th candidate
// facet of a ridge (rp); LDS for the shared-memory layouts, LDG otherwise
template <class C>
__device__ __forceinline__ int ldfr(const MapView& mp, int i) {
    if constexpr (C::TS) {
        unsigned short v;
        // volatile: never speculated -- callers guard out-of-range indices
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(mp.frs + 2u * (unsigned)i));
        return v;
    } else {
        return __ldg(mp.fr + i);
    }
}
template <class C>
__device__ __forceinline__ int ldrp(const MapView& mp, int i) {
    if constexpr (C::TS) {
        unsigned short v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(mp.rps + 2u * (unsigned)i));
        return v;
    } else {
        return __ldg(mp.rp + i);
    }
}

// Predicated shared-memory updates: one instruction each, no branch, so the
// warp never diverges around them (a C++ `if (cond) atomicXor(...)` costs a
// BSSY/BSYNC pair plus BRA.DIV guards before the next warp intrinsic).
__device__ __forceinline__ void red_xor_if(uint32_t a, uint32_t v, bool pred) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q red.shared.xor.b32 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
__device__ __forceinline__ void red_and_if(uint32_t a, uint32_t v, bool pred) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q red.shared.and.b32 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
__device__ __forceinline__ void red_or_if(uint32_t a, uint32_t v, bool pred) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q red.shared.or.b32 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
__device__ __forceinline__ void st_u8_if(uint32_t a, uint32_t v, bool pred) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u8 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
__device__ __forceinline__ void st_u16_if(uint32_t a, uint32_t v, bool pred) {
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.shared.u16 [%0], %1; }" ::"r"(a), "r"(v),
                 "r"((uint32_t)pred)
                 : "memory");
}
// predicated shared atomic add returning the old word (0 when not executed)
__device__ __forceinline__ uint32_t atom_add_if(uint32_t a, uint32_t v, bool pred) {
    uint32_t old = 0;
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q atom.shared.add.u32 %0, [%1], %2; }"
                 : "+r"(old)
                 : "r"(a), "r"(v), "r"((uint32_t)pred)
                 : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

// ------------------------------------------------------------ state updates
// ridge byte = c | a << 2: c = IN candidates (0..2), a = undecided candidates.
// open: c == 1.  b1: c == 1 && a == 1.  dead: c == 1 && a == 0.

// Flattened (decision, ridge) pairs of trail[lo..hi): body(act, e, k) per
// lane, k = the ridge slot of trail entry e.  Up to n = 8 a facet takes a
// power-of-two lane group (n = 5: 4 facets x 8 lanes per pass); the n >= 9
// size classes pack the pairs n per facet over all 32 lanes (trail entry
// lo + j / n, slot j % n, j / n by a multiply-shift): n = 11 -5 % search time,
// n = 8 +4 % (the division costs more than it saves when 8 lanes fit a facet)
template <class C, class F>
__device__ __forceinline__ void for_pairs(const MapView& mp, int lo, int hi, int lane, F&& body) {
    if constexpr (C::kN > 720) {
        const int tot = (hi - lo) * mp.n;
        for (int j0 = lane; j0 < tot + lane; j0 += 32) {
            const int q = (int)(((unsigned)j0 * mp.nmag) >> 20), k = j0 - q * mp.n;
            body(j0 < tot, lo + q, k);
        }
    } else {
        const int sh_l = mp.lpf_shift, k = lane & ((1 << sh_l) - 1), per = 32 >> sh_l;
        for (int e0 = lo; e0 < hi; e0 += per) {
            const int e = e0 + (lane >> sh_l);
            body(e < hi && k < mp.n, e, k);
        }
    }
}

// a -= 1 on every ridge of the facets trail[lo..hi) (already marked OUT)
template <class C>
__device__ __forceinline__ void apply_exclusions(WS<C>& w, const MapView& mp, int lo, int hi, int lane) {
    for_pairs<C>(mp, lo, hi, lane, [&](bool act, int e, int k) {
        const int g = act ? (w.trail()[e] & 0x7FFF) : 0;
        const int r = act ? ldfr<C>(mp, g * mp.fs + k) : 0;
        const unsigned sh = (r & 3) * 8;
        const unsigned ob = (atom_add_if(w.a_rs_word(r), 0u - (4u << sh), act) >> sh) & 0xFFu;
        // (1,1) -> (1,0): dead and leaves the forced set; (1,2) -> (1,1): enters it
        red_xor_if(w.a_b1(r), 1u << (r & 31), act && (ob == 5u || ob == 9u));
        w.ndead |= (int)__any_sync(FULL, act && ob == 5u);
    });
}

// exclude one facet (a tried sibling)
template <class C>
__device__ __forceinline__ void exclude_one(WS<C>& w, const MapView& mp, int g, int lane) {
    st_u8_if(w.a_fst(g), FOUT, lane == 0);
    st_u16_if(w.a_trail(w.tl), (uint32_t)g, lane == 0);
    const bool act = lane < mp.n;
    const int r = act ? ldfr<C>(mp, g * mp.fs + lane) : 0;
    const unsigned sh = (r & 3) * 8;
    const unsigned ob = (atom_add_if(w.a_rs_word(r), 0u - (4u << sh), act) >> sh) & 0xFFu;
    red_xor_if(w.a_b1(r), 1u << (r & 31), act && (ob == 5u || ob == 9u));
    w.ndead |= (int)__any_sync(FULL, act && ob == 5u);
    w.tl += 1;
    __syncwarp();
}

// The facet's ridges and their current bytes (lane k < n: k-th ridge), and
// whether including it is dead on arrival: one of its ridges has it as the
// sole undecided candidate (c = 0, a = 1) and would open with a = 0.  On the
// CPU restatement 92-97 % of dead includes are of this kind; they are counted
// as nodes but never applied (no include, no undo).
struct Probe {
    int r;
    unsigned b;
    bool dead;
};

template <class C>
__device__ __forceinline__ Probe probe_facet(const WS<C>& w, const MapView& mp, int f, int lane) {
    Probe pr{0, 4u, false};
    if (lane < mp.n) {
        pr.r = ldfr<C>(mp, f * mp.fs + lane);
        pr.b = w.rs()[pr.r];
    }
    pr.dead = __any_sync(FULL, pr.b == (1u << 2) && lane < mp.n);
    return pr;
}

template <class C>
__device__ __forceinline__ void include_facet(WS<C>& w, const MapView& mp, int f, const Probe& pr, int lane) {
    const bool act = lane < mp.n;
    const int r = pr.r;
    const unsigned b = pr.b;
    const unsigned c = b & 3u;               // c in {0,1}, a >= 1 (f is undecided)
    const bool closed = act && c == 1u;
    // branch-free: every lane k < n updates its ridge (c + 1, a - 1); the open
    // bit always flips (0 -> 1 opens, 1 -> 2 closes); the forced bit flips on
    // (1,1) -> (2,0) and (0,2) -> (1,1).  Opening with a = 0 cannot happen:
    // probe_facet filtered those includes.
    const unsigned bit = 1u << (r & 31);
    st_u8_if(w.a_rs(r), b + 1u - 4u, act);
    red_xor_if(w.a_open(r), bit, act);
    red_xor_if(w.a_b1(r), bit, act && (b == 5u || b == 8u));
    const unsigned bc = __ballot_sync(FULL, closed);
    w.nopen += mp.n - 2 * __popc(bc);
    st_u16_if(w.a_scratch(__popc(bc & lanemask_lt(lane))), (uint32_t)r, closed);
    st_u8_if(w.a_fst(f), FIN, lane == 0);
    red_or_if(w.a_inb(f), 1u << (f & 31), lane == 0);
    st_u16_if(w.a_trail(w.tl), (uint32_t)(f | TR_INC), lane == 0);
    w.tl += 1;
    w.size += 1;
    __syncwarp();
    if (!bc) return;
    // propagation: closing ridges exclude their other undecided candidates.
    // Two ridges of f share no candidate besides f, so the list has no repeats.
    const int ncl = __popc(bc);
    const int base = w.tl;
    int E = 0;
    for (int j0 = 0; j0 < ncl; j0 += 4) {
        const int j = j0 + (lane >> 3), q = lane & 7;
        const bool slot = j < ncl && q < mp.ps;
        const int rr = w.scratch()[j & 31];
        const int g0 = slot ? ldrp<C>(mp, rr * mp.ps + q) : (int)NONE16;
        const int g = g0 == NONE16 ? 0 : g0;
        const bool v = g0 != NONE16 && w.fst()[g] == FU;
        const unsigned bv = __ballot_sync(FULL, v);
        st_u16_if(w.a_trail(base + E + __popc(bv & lanemask_lt(lane))), (uint32_t)g, v);
        st_u8_if(w.a_fst(g), FOUT, v);
        E += __popc(bv);
    }
    if (E) {
        __syncwarp();
        apply_exclusions(w, mp, base, base + E, lane);
        w.tl += E;
    }
    __syncwarp();
}

// Undo every decision on trail[mark..tl) at once.  Each decision is an
// additive delta on the packed ridge bytes (include: c+1, a-1; exclusion:
// a-1), so the final bytes do not depend on the order the inverse deltas are
// applied in.  All (decision, ridge) pairs are flattened over the 32 lanes and
// applied with shared atomics; each atomic returns the exact old byte, so the
// open / forced bit flips it reports are exact whatever the interleaving.
// The tallies need no per-pair vote: every mark is taken at a live node
// (ndead == 0; a frame is pushed only when nothing is dead and a sibling
// exclusion that kills a ridge retires its open frame), so the state after
// the undo has ndead = 0 and the open count the caller saved at the mark.
template <class C>
__device__ __forceinline__ void undo_to(WS<C>& w, const MapView& mp, int mark, int nopen_mark, int lane) {
    const int lo = mark, hi = w.tl;
    if (hi <= lo) return;
    for (int e0 = lo; e0 < hi; e0 += 32) {
        const int e = e0 + lane;
        const bool act = e < hi;
        const unsigned t = act ? (unsigned)w.trail()[e] : 0u;
        const int g = (int)(t & 0x7FFFu);
        const bool inc = act && (t & TR_INC);
        st_u8_if(w.a_fst(g), FU, act);
        red_and_if(w.a_inb(g), ~(1u << (g & 31)), inc);
        w.size -= __popc(__ballot_sync(FULL, inc));
    }
    for_pairs<C>(mp, lo, hi, lane, [&](bool act, int e, int k) {
        const unsigned t = act ? (unsigned)w.trail()[e] : 0u;
        const int g = (int)(t & 0x7FFFu);
        const int r = act ? ldfr<C>(mp, g * mp.fs + k) : 0;
        const unsigned delta = (t & TR_INC) ? 3u : 4u;  // (c-1, a+1) or (a+1)
        const unsigned sh = (r & 3) * 8;
        const unsigned ob = (atom_add_if(w.a_rs_word(r), delta << sh, act) >> sh) & 0xFFu;
        const unsigned nb = ob + delta;
        const unsigned bit = 1u << (r & 31);
        red_xor_if(w.a_open(r), bit, act && (((ob & 3u) == 1u) != ((nb & 3u) == 1u)));
        red_xor_if(w.a_b1(r), bit, act && ((ob == 5u) != (nb == 5u)));
    });
    w.nopen = nopen_mark;
    w.ndead = 0;
    w.tl = mark;
    __syncwarp();
}

#ifdef WPM_DEBUG
// Debug builds: recompute every derived quantity from the facet statuses and
// trap on the first mismatch (counts, open / forced bitsets, open / dead
// tallies, IN bitset, size).
template <class C>
__device__ void debug_check(const WS<C>& w, const MapView& mp, int lane, int where) {
    __syncwarp();
    int bad = 0, nopen = 0, ndead = 0, size = 0;
    for (int r = lane; r < mp.N; r += 32) {
        unsigned c = 0, a = 0;
        for (int q = 0; q < mp.ps; ++q) {
            const int g = ldrp<C>(mp, r * mp.ps + q);
            if (g == NONE16) continue;
            c += w.fst()[g] == FIN;
            a += w.fst()[g] == FU;
        }
        const unsigned b = w.rs()[r];
        if (b != (c | (a << 2))) bad |= 1;
        const bool op = c == 1, f1 = c == 1 && a == 1;
        if (((w.open()[r >> 5] >> (r & 31)) & 1u) != (unsigned)op) bad |= 2;
        if (((w.b1()[r >> 5] >> (r & 31)) & 1u) != (unsigned)f1) bad |= 4;
        nopen += op;
        ndead += op && a == 0;
    }
    for (int f = lane; f < mp.M; f += 32) {
        size += w.fst()[f] == FIN;
        if (((w.inb()[f >> 5] >> (f & 31)) & 1u) != (unsigned)(w.fst()[f] == FIN)) bad |= 8;
    }
    __syncwarp();
    nopen = (int)__reduce_add_sync(FULL, (unsigned)nopen);
    ndead = (int)__reduce_add_sync(FULL, (unsigned)ndead);
    size = (int)__reduce_add_sync(FULL, (unsigned)size);
    bad = (int)__reduce_or_sync(FULL, (unsigned)bad);
    if (nopen != w.nopen) bad |= 16;
    if ((ndead != 0) != (w.ndead != 0)) bad |= 32;
    if (size != w.size) bad |= 64;
    if (bad) {
        if (lane == 0)
            printf("WPM_DEBUG mismatch %d at site %d: nopen %d/%d ndead %d/%d size %d/%d tl %d depth %d\n", bad, where,
                   w.nopen, nopen, w.ndead, ndead, w.size, size, w.tl, w.depth);
        __trap();
    }
}
#define DEBUG_CHECK(w, mp, lane, where) debug_check(w, mp, lane, where)
#else
#define DEBUG_CHECK(w, mp, lane, where) ((void)0)
#endif

// MRV branch ridge: the lowest open ridge with one undecided candidate, else
// the open ridge with the fewest (ties: lowest id).  Returns ridge | a << 16.
template <class C>
__device__ __forceinline__ unsigned select_ridge(const WS<C>& w, int nw, int lane) {
    for (int i0 = 0; i0 < nw; i0 += 32) {
        const unsigned word = (i0 + lane < nw) ? w.b1()[i0 + lane] : 0u;
        const unsigned bw = __ballot_sync(FULL, word != 0u);
        if (bw) {
            const int l = __ffs(bw) - 1;
            const unsigned x = __shfl_sync(FULL, word, l);
            return (unsigned)((i0 + l) * 32 + __ffs(x) - 1) | (1u << 16);
        }
    }
    unsigned best = 0xFFFFFFFFu;
    for (int i = lane; i < nw; i += 32) {
        unsigned bits = w.open()[i];
        while (bits) {
            const int r = i * 32 + __ffs(bits) - 1;
            bits &= bits - 1u;
            best = min(best, ((unsigned)(w.rs()[r] >> 2) << 16) | (unsigned)r);
        }
    }
    __syncwarp();  // reconverge after the divergent scan before the CREDUX
    return __reduce_min_sync(FULL, best);
}

// the undecided candidates of an OPEN frame's ridge from slot pos: first one
template <class C>
__device__ __forceinline__ int first_candidate(const WS<C>& w, const MapView& mp, int ridge, int pos, int* slot,
                                               int lane) {
    const bool in_range = lane >= pos && lane < mp.ps;
    const int g0 = in_range ? ldrp<C>(mp, ridge * mp.ps + lane) : (int)NONE16;
    const int g = g0 == NONE16 ? 0 : g0;
    const bool ok = g0 != NONE16 && w.fst()[g] == FU;
    const unsigned b = __ballot_sync(FULL, ok);
    if (!b) return -1;
    const int q = __ffs(b) - 1;
    *slot = q;
    return __shfl_sync(FULL, g, q);
}

// next undecided child of a frame from its pos; -1 if none
template <class C>
__device__ __forceinline__ int next_child(const WS<C>& w, const MapView& mp, uint2 fr, int* new_pos, int lane) {
    const uint32_t ridge = fr.x & 0xFFFFu, pos = fr.x >> 16;
    if (pos == POS_DONE) return -1;
    if (ridge == CLOSED_FRAME) {
        for (int p0 = (int)pos; p0 < mp.M; p0 += 32) {
            const int f = p0 + lane;
            const unsigned b = __ballot_sync(FULL, f < mp.M && w.fst()[f] == FU);
            if (b) {
                const int c = p0 + __ffs(b) - 1;
                *new_pos = c + 1;
                return c;
            }
        }
        return -1;
    }
    int q = 0;
    const int g = first_candidate(w, mp, (int)ridge, (int)pos, &q, lane);
    *new_pos = q + 1;
    return g;
}

// --------------------------------------------------------------- the search

template <class C>
__device__ __forceinline__ void emit(const WS<C>& w, const MapView& mp, const SearchParams& p, int lane) {
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(&p.out_ctl[0], 1ull);
    slot = __shfl_sync(FULL, slot, 0);
    if (slot < p.out_cap) {  // key row: bitset words, zero padded, then the map id
        uint32_t* o = p.out_keys + slot * (unsigned long long)p.rw;
        const int mw = (mp.M + 31) >> 5, last = p.rw - 1;
        #pragma unroll 1
        for (int i = lane; i < p.rw; i += 32) o[i] = i < mw ? w.inb()[i] : (i == last ? (uint32_t)mp.map : 0u);
    }
}

// the current state as a task record "resume branch frame `ridge` from its
// first child" (frontier expansion: the frame at the cutoff depth)
template <class C>
__device__ __forceinline__ void write_frontier(const WS<C>& w, const MapView& mp, const SearchParams& p, uint32_t ridge,
                                               int lane) {
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(&p.front_ctl[0], 1ull);
    slot = __shfl_sync(FULL, slot, 0);
    if (slot >= p.front_cap) return;  // counted: the host reruns with room
    uint32_t* rec = p.front_out + slot * (unsigned long long)p.recw;
    if (lane == 0) {
        rec[0] = (uint32_t)mp.map | ((ridge == CLOSED_FRAME ? (uint32_t)T_CLOSED : (uint32_t)T_OPEN) << 24);
        rec[1] = ridge;
        rec[2] = (uint32_t)(w.dbase() + w.depth) << 16;
        rec[3] = w.root();
    }
    const int mw = (mp.M + 31) >> 5;
    #pragma unroll 1
    for (int f0 = 0; f0 < mw * 32; f0 += 32) {
        const int f = f0 + lane;
        const uint8_t st = f < mp.M ? w.fst()[f] : (uint8_t)FU;
        const unsigned bi = __ballot_sync(FULL, st == FIN), bo = __ballot_sync(FULL, st == FOUT);
        if (lane == 0) {
            rec[4 + (f0 >> 5)] = bi;
            rec[4 + p.mw + (f0 >> 5)] = bo;
        }
    }
}

// The descent below a node just entered (after an include, or at a task
// entry): emit / prune, follow forced moves as a chain of includes, stop at
// the next real branch point by pushing its frame.  Returns true if a frame
// was pushed; false if the descent ended (dead, pruned, or a leaf).
template <class C>
__device__ __forceinline__ bool descend(WS<C>& w, const MapView& mp, const SearchParams& p, unsigned& nodes,
                                        int lane) {
    for (;;) {
        if (w.ndead) return false;
        uint32_t ridge;
        if (w.nopen == 0) {
            if (w.size > 0 && w.size <= mp.cap) emit(w, mp, p, lane);  // count_cap at the leaf, search.hpp:218-220
            if (w.size + mp.n + 1 > mp.cap) return false;
            ridge = CLOSED_FRAME;
        } else {
            // |S| + ceil(open / n) > cap  <=>  open > (cap - |S|) * n
            // (32-bit: capn = min(cap, 2^20) never prunes where cap would not -- open <= N < 2^12)
            if ((mp.capn - w.size) * mp.n < w.nopen) return false;
            const unsigned sel = select_ridge(w, mp.nw, lane);
            ridge = sel & 0xFFFFu;
            if ((sel >> 16) == 1u) {  // forced: the only undecided candidate
                int q;
                const int u = first_candidate(w, mp, (int)ridge, 0, &q, lane);
                const Probe pr = probe_facet(w, mp, u, lane);
                ++nodes;
                if (pr.dead) return false;
                include_facet(w, mp, u, pr, lane);
                DEBUG_CHECK(w, mp, lane, 1);
                continue;
            }
        }
        if (p.cutoff && w.dbase() + w.depth >= p.cutoff) {  // split mode: hand the frame on
            write_frontier(w, mp, p, ridge, lane);
            return false;
        }
        if (w.depth >= C::kDepth) {
            // frame stack full (the fast layouts hold FRAME_CAP frames): flag the
            // run as incomplete; the host discards it and reruns with the
            // full-depth layout
            if (lane == 0) atomicExch(&p.out_ctl[2], 1ull);
            return false;
        }
        if (lane == 0) w.frames()[w.depth] = make_uint2(ridge, NO_CHILD);
        w.depth += 1;
        __syncwarp();
        return true;
    }
}

// rebuild the warp state from an IN/OUT record (+ closure: a ridge with two
// IN candidates excludes the rest).  Returns false if infeasible.
template <class C>
__device__ __forceinline__ bool load_state(WS<C>& w, const MapView& mp, const uint32_t* rec_in,
                                           const uint32_t* rec_out, bool closure, int lane) {
    const int M = mp.M, N = mp.N, mw = (M + 31) >> 5, nw = mp.nw;
    uint8_t* rs = w.rs();
    uint8_t* fst = w.fst();
    int size = 0;
    #pragma unroll 1
    for (int i = lane; i < mw; i += 32) {
        const uint32_t iv = __ldcg(rec_in + i);
        w.inb()[i] = iv;
        size += __popc(iv);
    }
    #pragma unroll 1
    for (int f0 = 0; f0 < M; f0 += 32) {
        const int f = f0 + lane;
        const uint32_t iv = __ldcg(rec_in + (f0 >> 5)), ov = __ldcg(rec_out + (f0 >> 5));
        const uint32_t bit = 1u << lane;
        if (f < M) fst[f] = (iv & bit) ? FIN : ((ov & bit) ? FOUT : FU);
    }
    __syncwarp();  // reconverge after the divergent loops before the CREDUX
    w.size = (int)__reduce_add_sync(FULL, (unsigned)size);
    __syncwarp();
    if (closure) {
        // pass 1: IN counts; a count >= 3 is infeasible
        bool bad = false;
        #pragma unroll 1
        for (int r = lane; r < N; r += 32) {
            unsigned c = 0;
            #pragma unroll 1
            for (int q = 0; q < mp.ps; ++q) {
                const int g = ldrp<C>(mp, r * mp.ps + q);
                c += g != NONE16 && fst[g] == FIN;
            }
            bad |= c > 2u;
            rs[r] = (uint8_t)min(c, 2u);
        }
        if (__any_sync(FULL, bad)) return false;
        __syncwarp();
        // closure: undecided facets on a closed ridge are excluded
        #pragma unroll 1
        for (int f = lane; f < M; f += 32) {
            if (fst[f] != FU) continue;
            bool on_closed = false;
            #pragma unroll 1
            for (int k = 0; k < mp.n; ++k) on_closed |= rs[ldfr<C>(mp, f * mp.fs + k)] == 2u;
            if (on_closed) fst[f] = FOUT;
        }
        __syncwarp();
    }
    // pass 2 (the only pass for states produced by the search itself, which
    // are closed already): counts, open / b1 bitsets, open / dead tallies
    int nopen = 0, ndead = 0;
    #pragma unroll 1
    for (int r0 = 0; r0 < nw * 32; r0 += 32) {
        const int r = r0 + lane;
        bool op = false, dd = false, one = false;
        if (r < N) {
            unsigned a = 0, ci = 0;
            #pragma unroll 1
            for (int q = 0; q < mp.ps; ++q) {
                const int g0 = ldrp<C>(mp, r * mp.ps + q);
                const unsigned s = g0 != NONE16 ? fst[g0] : (unsigned)FOUT;
                a += s == FU;
                ci += s == FIN;
            }
            const unsigned c = closure ? (unsigned)rs[r] : ci;
            rs[r] = (uint8_t)(c | (a << 2));
            op = c == 1u;
            dd = op && a == 0u;
            one = op && a == 1u;
        }
        const unsigned bo = __ballot_sync(FULL, op), b1 = __ballot_sync(FULL, one);
        if (lane == 0) {
            w.open()[r0 >> 5] = bo;
            w.b1()[r0 >> 5] = b1;
        }
        nopen += __popc(bo);
        ndead += __popc(__ballot_sync(FULL, dd));
    }
    w.nopen = nopen;
    w.ndead = ndead;
    w.tl = 0;
    w.depth = 0;
    __syncwarp();
    return true;
}

// donate the shallowest frame that still has an untried child.  The
// frame's state = the current state minus every decision on the trail at or
// after mk (`late`), with its in-progress child excluded.
template <class C>
__device__ __forceinline__ bool try_donate(WS<C>& w, const MapView& mp, const SearchParams& p, int lane) {
    const int M = mp.M, mw = (M + 31) >> 5;
    uint32_t* late = w.late();
    const uint8_t* fst = w.fst();
    #pragma unroll 1
    for (int d = 0; d < w.depth; ++d) {
        const uint2 fr = w.frames()[d];
        const uint32_t ridge = fr.x & 0xFFFFu, pos = fr.x >> 16;
        if (pos == POS_DONE) continue;
        const bool busy = (fr.y & 0xFFFFu) != NO_CHILD && d + 1 < w.depth;
        const int mk = busy ? (int)(fr.y >> 16) : w.tl;  // the frame's own state
        const int cur = busy ? (int)(fr.y & 0xFFFFu) : -1;
        #pragma unroll 1
        for (int i = lane; i < mw; i += 32) late[i] = 0u;
        __syncwarp();
        #pragma unroll 1
        for (int e = mk + lane; e < w.tl; e += 32) {
            const int g = w.trail()[e] & 0x7FFF;
            atomicOr(&late[g >> 5], 1u << (g & 31));
        }
        __syncwarp();
        bool any = false;
        if (ridge == CLOSED_FRAME) {
            #pragma unroll 1
            for (int f0 = (int)pos; f0 < M && !any; f0 += 32) {
                const int f = f0 + lane;
                any = __any_sync(FULL, f < M && f != cur && (fst[f] == FU || ((late[f >> 5] >> (f & 31)) & 1u)));
            }
        } else {
            bool ok = false;
            if (lane >= (int)pos && lane < mp.ps) {
                const int g = ldrp<C>(mp, ridge * mp.ps + lane);
                ok = g != NONE16 && g != cur && (fst[g] == FU || ((late[g >> 5] >> (g & 31)) & 1u));
            }
            any = __any_sync(FULL, ok);
        }
        if (!any) continue;
        // claim a push ticket (high half of the queue word)
        unsigned long long t = 0;
        unsigned long long* qc = q_ctl<C>(p, mp.map);
        if (lane == 0) {
            atomicAdd(&qc[2], 1ull);  // pending, before publishing
            if (p.root_pend) atomicAdd(&p.root_pend[w.root()], 1u);
            t = atomicAdd(&qc[0], 1ull << 32) >> 32;
        }
        t = __shfl_sync(FULL, t, 0);
        uint32_t* rec = q_rec<C>(p, mp.map) + (t % (unsigned long long)p.qcap) * (unsigned long long)p.recw;
        if (lane == 0) {
            rec[0] = (uint32_t)mp.map | ((ridge == CLOSED_FRAME ? (uint32_t)T_CLOSED : (uint32_t)T_OPEN) << 24);
            rec[1] = ridge;
            rec[2] = pos | ((uint32_t)(w.dbase() + d) << 16);
            rec[3] = w.root();
        }
        #pragma unroll 1
        for (int f0 = 0; f0 < mw * 32; f0 += 32) {
            const int f = f0 + lane;
            bool in = false, out = false;
            if (f < M) {
                const uint8_t s = fst[f];
                const bool before = !((late[f >> 5] >> (f & 31)) & 1u);
                in = s == FIN && before;
                out = (s == FOUT && before) || f == cur;
            }
            const unsigned bi = __ballot_sync(FULL, in), bo = __ballot_sync(FULL, out);
            if (lane == 0) {
                rec[4 + (f0 >> 5)] = bi;
                rec[4 + p.mw + (f0 >> 5)] = bo;
            }
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            atomicExch(&q_ready<C>(p, mp.map)[t % (unsigned long long)p.qcap], t + 1ull);
            w.frames()[d].x = ridge | (POS_DONE << 16);  // exhausted here
        }
        __syncwarp();
        return true;
    }
    return false;
}

// map-affine layouts: the CTA's next map, chosen by warp 0 while the CTA
// waits -- first the map whose seeds hold this CTA's share of all root tasks,
// later the unfinished map with the most pending tasks per CTA on it -- and
// its tables loaded into shared memory.  -1: no map has work left (or the
// node budget is spent).
template <class C>
__device__ int ma_next_map(const SearchParams& p, int prev, uint8_t* smem, int* s_map) {
    __syncthreads();  // every warp is done with the previous map's tables
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int pick = -1;
        if (prev < 0) {
            if (lane == 0) {
                const long long total = p.map_first[p.num_maps];
                const long long target = ((2LL * blockIdx.x + 1) * total) / (2LL * gridDim.x);
                int q = 0;
                while (q + 1 < p.num_maps && p.map_first[q + 1] <= target) ++q;
                pick = q;
            }
        } else {
            if (lane == 0) atomicAdd(&q_ctl<C>(p, prev)[1], (unsigned long long)-1ll);
            const bool stop = p.node_budget && ld_relaxed_u64(&p.out_ctl[3]);
            unsigned long long bp = 0, bo = 1;
            int bq = -1;
            #pragma unroll 1
            for (int q = lane; q < p.num_maps && !stop; q += 32) {
                const unsigned long long pend = ld_relaxed_u64(&q_ctl<C>(p, q)[2]);
                if (!pend) continue;
                const unsigned long long on = ld_relaxed_u64(&q_ctl<C>(p, q)[1]) + 1ull;
                if (bq < 0 || pend * bo > bp * on) {
                    bp = pend;
                    bo = on;
                    bq = q;
                }
            }
            #pragma unroll
            for (int o = 16; o; o >>= 1) {
                const unsigned long long op = __shfl_down_sync(FULL, bp, o), oo = __shfl_down_sync(FULL, bo, o);
                const int oq = __shfl_down_sync(FULL, bq, o);
                if (oq >= 0 && (bq < 0 || op * bo > bp * oo)) {
                    bp = op;
                    bo = oo;
                    bq = oq;
                }
            }
            pick = bq;
        }
        if (lane == 0) {
            if (pick >= 0) atomicAdd(&q_ctl<C>(p, pick)[1], 1ull);
            *s_map = pick;
        }
    }
    __syncthreads();
    const int q = *s_map;
    if (q >= 0) {
        const MapDesc md = p.maps[q];
        const int nf = md.M * md.fr_stride, nr = md.N * md.rp_stride;
        uint16_t* dfr = reinterpret_cast<uint16_t*>(smem);
        uint16_t* drp = reinterpret_cast<uint16_t*>(smem + a16(2 * nf));
        #pragma unroll 1
        for (int i = threadIdx.x; i < nf; i += blockDim.x) dfr[i] = __ldg(p.fr + md.fr_off + i);
        #pragma unroll 1
        for (int i = threadIdx.x; i < nr; i += blockDim.x) drp[i] = __ldg(p.rp + md.rp_off + i);
    }
    __syncthreads();
    return q;
}

template <class C>
__global__ void __launch_bounds__(32 * C::WPB, C::MIN_BLOCKS) k3_search(const __grid_constant__ SearchParams p) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // TS layouts: every map's fr then rp tables at the CTA's base, then the
    // warps; map-affine layouts: the current map's tables only
    const int tab_bytes = C::TS ? (C::MA ? p.ma_tab_bytes : 16 * (((p.fr_words + 7) >> 3) + ((p.rp_words + 7) >> 3))) : 0;
    if constexpr (C::TS && !C::MA) {
        const uint4* src_fr = reinterpret_cast<const uint4*>(p.fr);
        const uint4* src_rp = reinterpret_cast<const uint4*>(p.rp);
        uint4* dfr = reinterpret_cast<uint4*>(smem);
        const int nfr = (p.fr_words + 7) >> 3, nrp = (p.rp_words + 7) >> 3;
        uint4* drp = reinterpret_cast<uint4*>(smem + 16 * nfr);
        for (int i = threadIdx.x; i < nfr; i += blockDim.x) dfr[i] = __ldg(src_fr + i);
        for (int i = threadIdx.x; i < nrp; i += blockDim.x) drp[i] = __ldg(src_rp + i);
        __syncthreads();
    }
    const uint32_t tab_s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const uint32_t rp_s = tab_s + 16u * (uint32_t)((p.fr_words + 7) >> 3);
    WS<C> w;
    w.base = smem + tab_bytes + wid * C::BYTES;
    w.sb = static_cast<uint32_t>(__cvta_generic_to_shared(w.base));
    // search nodes: `nodes` (64-bit) takes the 32-bit running count `tn` at
    // every queue check and task end, so the per-node work is a 32-bit
    // increment and compare
    unsigned long long nodes = 0, tasks = 0;
    unsigned tn = 0;
#ifdef WPM_PROFILE
    // busy / waiting / final-wait clocks per warp (qctl[5..7]; WPM_PROFILE=1 prints them)
    unsigned long long prof_busy = 0, prof_wait = 0, prof_t = clock64();
#endif

    __shared__ int s_map;
    int cur = 0;  // the CTA's map (map-affine layouts); queue 0 otherwise
    if constexpr (C::MA) cur = ma_next_map<C>(p, -1, smem, &s_map);
    while (cur >= 0) {
    unsigned long long* const qc = q_ctl<C>(p, cur);
    unsigned long long* const qrdy = q_ready<C>(p, cur);
    uint32_t* const qrec = q_rec<C>(p, cur);
    for (;;) {
        // ---- pop: a ticket queue.  One atomicAdd on the low half of the
        // queue word claims ticket t; the warp waits on ITS slot until the
        // pusher holding push-ticket t publishes it (FIFO hand-off, no CAS
        // retries, no shared spin address).  pending == 0 means no task
        // exists anywhere and no warp can push again: every waiter leaves.
        // In claim mode a waiter also pulls shared frontier records into the
        // queue while this GPU runs low (pending < claim_low), and leaves only
        // once the shared frontier is exhausted too.
        unsigned long long tk = 0;
        if (lane == 0) tk = atomicAdd(&qc[0], 1ull) & 0xFFFFFFFFull;
        long long t = -1;
        bool exhausted = p.claim_recs == nullptr;
        for (;;) {
            long long claim = -1;
            if (lane == 0) {
                volatile unsigned long long* rdy = qrdy + (tk % (unsigned long long)p.qcap);
                volatile unsigned long long* pend = qc + 2;
                unsigned backoff = (unsigned)p.backoff_min;
                if (exhausted) {  // no shared frontier to claim from: the tight ticket wait
                    for (;;) {
                        if (*rdy == tk + 1ull) {
                            t = (long long)tk;
                            break;
                        }
                        if (*pend == 0ull || (p.node_budget && ld_relaxed_u64(&p.out_ctl[3]))) {
                            t = -2;  // no task left anywhere, or the node budget is spent
                            break;
                        }
                        __nanosleep(backoff);
                        backoff = min(backoff * 2u, (unsigned)p.backoff_max);
                    }
                }
                while (t == -1) {
                    if (*rdy == tk + 1ull) {
                        t = (long long)tk;
                        break;
                    }
                    if (!exhausted && *pend < (unsigned long long)p.claim_low) {
                        // (a plain read first: idle warps polling must not hammer the
                        // pending counter the busy warps update -- measured +30 % claim
                        // time at 12.7 k records without it)
                        if (atomicAdd(&qc[2], 1ull) < (unsigned long long)p.claim_low) {
                            const unsigned long long i = atomicAdd_system(p.claim_ctr, 1ull);
                            if (i < (unsigned long long)p.claim_count) {
                                claim = (long long)i;  // pending already counts it
                                break;
                            }
                            exhausted = true;
                        }
                        atomicAdd(&qc[2], (unsigned long long)-1ll);
                        if (!exhausted) {
                            unsigned long long c;
                            asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(c) : "l"(p.claim_ctr));
                            exhausted = c >= (unsigned long long)p.claim_count;
                        }
                        __threadfence();  // the shared counter before the pending count
                    }
                    if (exhausted && (*pend == 0ull || (p.node_budget && ld_relaxed_u64(&p.out_ctl[3])))) {
                        t = -2;  // no task left anywhere, or the node budget is spent
                        break;
                    }
                    __nanosleep(backoff);
                    backoff = min(backoff * 2u, (unsigned)p.backoff_max);
                }
            }
            claim = __shfl_sync(FULL, claim, 0);
            if (claim < 0) break;
            // push the claimed frontier record (root id = its frontier index)
            unsigned long long pt = 0;
            if (lane == 0) pt = atomicAdd(&qc[0], 1ull << 32) >> 32;
            pt = __shfl_sync(FULL, pt, 0);
            const uint32_t* src = p.claim_recs + (unsigned long long)claim * p.recw;
            uint32_t* dst = qrec + (pt % (unsigned long long)p.qcap) * (unsigned long long)p.recw;
            for (int i = lane; i < p.recw; i += 32) dst[i] = i == 3 ? (uint32_t)claim : __ldcg(src + i);
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicExch(&qrdy[pt % (unsigned long long)p.qcap], pt + 1ull);
        }
        t = __shfl_sync(FULL, t, 0);
#ifdef WPM_PROFILE
        {
            const unsigned long long now = clock64();
            if (t == -2) {
                if (lane == 0) atomicAdd(&p.qctl[7], now - prof_t);
            } else {
                prof_wait += now - prof_t;
            }
            prof_t = now;
        }
#endif
        if (t == -2) break;
        const unsigned long long slot = (unsigned long long)t % (unsigned long long)p.qcap;
        __syncwarp();
        __threadfence();
        if (p.node_budget) {  // budget spent: leave the queue as is (one read, warp-uniform)
            int spent = 0;
            if (lane == 0) spent = ld_relaxed_u64(&p.out_ctl[3]) != 0ull;
            if (__shfl_sync(FULL, spent, 0)) break;
        }
        const uint32_t* rec = qrec + slot * (unsigned long long)p.recw;
        const uint32_t h0 = __ldcg(rec), h1 = __ldcg(rec + 1), h2 = __ldcg(rec + 2), h3 = __ldcg(rec + 3);
        if (lane == 0) {
            reinterpret_cast<int*>(w.base + C::META)[0] = (int)(h2 >> 16);
            reinterpret_cast<uint32_t*>(w.base + C::META)[1] = h3;
            reinterpret_cast<unsigned long long*>(w.base + C::META)[1] = nodes;  // per-root node accounting
        }
        __syncwarp();
        const int map = (int)(h0 & 0xFFFFu);
        const uint32_t kind = h0 >> 24;
        const MapDesc md = p.maps[map];
        MapView mp;
        mp.M = md.M;
        mp.N = md.N;
        mp.n = md.n;
        mp.cap = md.cap;
        mp.capn = min(md.cap, 1 << 20);
        mp.map = map;
        mp.nw = (md.N + 31) >> 5;
        mp.lpf_shift = md.n <= 4 ? 2 : (md.n <= 8 ? 3 : 4);
        mp.nmag = ((1u << 20) + (unsigned)md.n - 1u) / (unsigned)md.n;
        mp.fr = p.fr + md.fr_off;
        mp.rp = p.rp + md.rp_off;
        if constexpr (C::MA) {  // map == cur: its tables alone, fr then rp
            mp.frs = tab_s;
            mp.rps = tab_s + (uint32_t)a16(2 * md.M * md.fr_stride);
        } else {
            mp.frs = tab_s + 2u * md.fr_off;
            mp.rps = rp_s + 2u * md.rp_off;
        }
        mp.fs = md.fr_stride;
        mp.ps = md.rp_stride;
        ++tasks;

        // only pinned ENTRY tasks need the closure pass; seeded roots (nothing
        // IN) and donated frames (a state of the search) are closed already
        if (load_state(w, mp, rec + 4, rec + 4 + p.mw, kind == T_ENTRY, lane)) {
            if (kind == T_SINGLE) {
                const Probe pr = probe_facet(w, mp, (int)h1, lane);
                ++tn;
                if (!pr.dead) {
                    include_facet(w, mp, (int)h1, pr, lane);
                    DEBUG_CHECK(w, mp, lane, 2);
                    descend(w, mp, p, tn, lane);
                }
            } else if (kind == T_ENTRY) {
                descend(w, mp, p, tn, lane);
            } else if (w.ndead == 0) {  // resume a donated frame
                if (lane == 0)
                    w.frames()[0] =
                        make_uint2((kind == T_CLOSED ? CLOSED_FRAME : h1) | ((h2 & 0xFFFFu) << 16), NO_CHILD);
                w.depth = 1;
                __syncwarp();
            }
        }
        // ---- the DFS over branch frames
        unsigned long long qword = ld_relaxed_u64(&qc[0]);  // prefetched queue state
        unsigned long long flushed = nodes;  // node-budget mode: count already in qctl[1]
        unsigned chk = (unsigned)p.first_check;  // nodes before the next look at the queue
        while (w.depth > 0) {
            const uint2 fr = w.frames()[w.depth - 1];
            int npos = 0;
            const int c = next_child(w, mp, fr, &npos, lane);
            if (c < 0) {
                // frame exhausted: back to the parent frame's state before its
                // current child, then exclude that child there
                w.depth -= 1;
                if (w.depth > 0) {
                    const uint2 pf = w.frames()[w.depth - 1];
                    undo_to(w, mp, (int)(pf.y >> 16), (int)w.nopen_at()[w.depth - 1], lane);
                    DEBUG_CHECK(w, mp, lane, 3);
                    exclude_one(w, mp, (int)(pf.y & 0xFFFFu), lane);
                    DEBUG_CHECK(w, mp, lane, 4);
                    if ((pf.x & 0xFFFFu) != CLOSED_FRAME && w.ndead) {
                        if (lane == 0) w.frames()[w.depth - 1].x = (pf.x & 0xFFFFu) | (POS_DONE << 16);
                        __syncwarp();
                    }
                }
                continue;
            }
            const int cm = w.tl, om = w.nopen;
            if (lane == 0) {
                w.frames()[w.depth - 1] =
                    make_uint2((fr.x & 0xFFFFu) | ((uint32_t)npos << 16), (uint32_t)c | ((uint32_t)cm << 16));
                w.nopen_at()[w.depth - 1] = (uint16_t)om;
            }
            __syncwarp();
            const Probe pr = probe_facet(w, mp, c, lane);
            ++tn;
            bool pushed = false;
            if (!pr.dead) {
                include_facet(w, mp, c, pr, lane);
                DEBUG_CHECK(w, mp, lane, 5);
                pushed = descend(w, mp, p, tn, lane);
            }
            if (!pushed) {
                undo_to(w, mp, cm, om, lane);
                DEBUG_CHECK(w, mp, lane, 6);
                exclude_one(w, mp, c, lane);
                DEBUG_CHECK(w, mp, lane, 7);
                if ((fr.x & 0xFFFFu) != CLOSED_FRAME && w.ndead) {
                    if (lane == 0) w.frames()[w.depth - 1].x = (fr.x & 0xFFFFu) | (POS_DONE << 16);
                    __syncwarp();
                }
            }
            if (tn >= chk) {
                nodes += tn;
                tn = 0;
                // waiting warps <=> the head ticket ran ahead of the tail
                const long long queued = (long long)(qword >> 32) - (long long)(qword & 0xFFFFFFFFull);
                // many warps waiting (a ramp, a tail, a GPU holding few
                // frontier records): look again sooner
                chk = queued < -(long long)p.starve_at ? (unsigned)p.starve_check : (unsigned)p.check_every;
                if (queued < (long long)p.hungry) {
                    // warps are waiting (head ran past tail): hand out up to
                    // donate_max frames at once, shallowest first
                    const int k = queued < 0 ? p.donate_max : 1;
                    for (int i = 0; i < k; ++i)
                        if (!try_donate(w, mp, p, lane)) break;
                }
                qword = ld_relaxed_u64(&qc[0]);  // consumed at the next check
                if (p.node_budget) {
                    int stop = 0;
                    if (lane == 0) {
                        const unsigned long long d = nodes - flushed;
                        if (atomicAdd(&p.qctl[1], d) + d >= p.node_budget) atomicExch(&p.out_ctl[3], 1ull);
                        stop = ld_relaxed_u64(&p.out_ctl[3]) != 0ull;
                    }
                    flushed = nodes;
                    if (__shfl_sync(FULL, stop, 0)) break;  // abandon the task (a truncated run)
                }
            }
        }
        // task finished
        nodes += tn;
        tn = 0;
        if (lane == 0) {
            if (p.root_nodes)
                atomicAdd(&p.root_nodes[w.root()], nodes - reinterpret_cast<unsigned long long*>(w.base + C::META)[1]);
            if (p.root_pend && atomicSub(&p.root_pend[w.root()], 1u) == 1u) {
                const unsigned long long d = atomicAdd(p.roots_done, 1ull) + 1ull;
                if (p.progress_host)  // host takes the max of what it sees
                    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p.progress_host), "l"(d) : "memory");
            }
            atomicAdd(&qc[2], (unsigned long long)-1ll);
        }
#ifdef WPM_PROFILE
        {
            const unsigned long long now = clock64();
            prof_busy += now - prof_t;
            prof_t = now;
        }
#endif
    }
    if constexpr (C::MA) cur = ma_next_map<C>(p, cur, smem, &s_map);
    else break;
    }
    if (lane == 0) {
        atomicAdd(&p.qctl[3], tasks);
        atomicAdd(&p.qctl[4], nodes);
#ifdef WPM_PROFILE
        atomicAdd(&p.qctl[5], prof_busy);
        atomicAdd(&p.qctl[6], prof_wait);
#endif
    }
}

__global__ void seed_tasks(SearchParams p, int ntasks, const int32_t* __restrict__ task_map,
                           const int32_t* __restrict__ task_f, const int32_t* __restrict__ task_kind,
                           const uint32_t* __restrict__ pin_in, const uint32_t* __restrict__ pin_out) {
    // one warp per task: IN = pinned-in, OUT = pinned-out + (SINGLE f) every facet < f
    const int lane = threadIdx.x & 31;
    const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (t >= ntasks) return;
    const int map = task_map[t], f = task_f[t], kind = task_kind[t];
    // map queues: task t is slot t - map_first[map] of its map's queue
    const size_t slot = p.map_queues ? (size_t)map * p.qcap + (size_t)(t - p.map_first[map]) : (size_t)t;
    uint32_t* rec = p.qrec + slot * p.recw;
    if (lane == 0) {
        rec[0] = (uint32_t)map | ((uint32_t)kind << 24);
        rec[1] = (uint32_t)f;
        rec[2] = (kind == T_SINGLE ? 1u : 0u) << 16;  // a root task includes a child of the depth-0 frame
        rec[3] = (uint32_t)t;
        if (p.root_pend) p.root_pend[t] = 1u;
    }
    for (int i = lane; i < p.mw; i += 32) {
        uint32_t in = 0, out = 0;
        if (kind == T_SINGLE) {
            const int lo = i * 32;
            if (f >= lo + 32) out = 0xFFFFFFFFu;
            else if (f > lo) out = (1u << (f - lo)) - 1u;
        }
        if (pin_in) in = pin_in[(size_t)map * p.mw + i];
        if (pin_out) out |= pin_out[(size_t)map * p.mw + i];
        rec[4 + i] = in;
        rec[4 + p.mw + i] = out;
    }
    if (lane == 0) p.qready[slot] = (unsigned long long)(p.map_queues ? t - p.map_first[map] : t) + 1ull;
}

// seed the queue with task records (a frontier): record i -> ticket i, root id i
__global__ void seed_records(SearchParams p, const uint32_t* __restrict__ recs, long long count) {
    const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= count) return;
    const uint32_t* src = recs + (size_t)i * p.recw;
    uint32_t* dst = p.qrec + (size_t)i * p.recw;
    for (int k = lane; k < p.recw; k += 32) dst[k] = k == 3 ? (uint32_t)i : src[k];
    if (lane == 0) {
        if (p.root_pend) p.root_pend[i] = 1u;
        p.qready[i] = (unsigned long long)i + 1ull;
    }
}

template <class C>
int launch_class(const SearchParams& p, int num_sms, cudaStream_t st, int* warps_out) {
    const int wpb = C::WPB;  // warps per CTA
    // fr and rp each padded to 16 bytes (the kernel's layout)
    const size_t tab = !C::TS ? 0 : C::MA ? (size_t)p.ma_tab_bytes : (size_t)16 * (((p.fr_words + 7) >> 3) + ((p.rp_words + 7) >> 3));
    const size_t smem = tab + (size_t)C::BYTES * wpb;
    // experiment knob: the L1 / shared split (percent of the max shared carveout)
    if (const char* e = std::getenv("WPM_CARVEOUT"))
        cudaFuncSetAttribute(k3_search<C>, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(e));
    int per_sm = occupancy_cached(reinterpret_cast<const void*>(k3_search<C>), 32 * wpb, smem);
    if (per_sm < 1) return 0;
    if (const char* e = std::getenv("WPM_BLOCKS_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    const int grid = per_sm * num_sms;
    k3_search<C><<<grid, 32 * wpb, smem, st>>>(p);
    if (cudaGetLastError() != cudaSuccess) return 0;
    if (warps_out) *warps_out = grid * wpb;
    return grid;
}

}  // namespace

int launch_seed_tasks(const SearchParams& p, int ntasks, const int32_t* d_task_map, const int32_t* d_task_f,
                      const int32_t* d_task_kind, const uint32_t* d_pin_in, const uint32_t* d_pin_out,
                      cudaStream_t st) {
    if (ntasks <= 0) return 0;
    const int threads = 128, blocks = (ntasks * 32 + threads - 1) / threads;
    seed_tasks<<<blocks, threads, 0, st>>>(p, ntasks, d_task_map, d_task_f, d_task_kind, d_pin_in, d_pin_out);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

__global__ void fill_u32(unsigned int* d, unsigned int v, long long count) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) d[i] = v;
}

int launch_fill_u32(unsigned int* d, unsigned int v, long long count, cudaStream_t st) {
    if (count <= 0) return 0;
    fill_u32<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d, v, count);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int launch_seed_records(const SearchParams& p, const uint32_t* d_recs, long long count, cudaStream_t st) {
    if (count <= 0) return 0;
    const long long threads = count * 32;
    seed_records<<<(unsigned)((threads + 127) / 128), 128, 0, st>>>(p, d_recs, count);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

// a TS layout fits if its CTAs (tables + warps) fit the SM's shared memory
template <class C>
bool ts_fits(const SearchParams& p) {
    const size_t tab = C::MA ? (size_t)p.ma_tab_bytes : (size_t)16 * (((p.fr_words + 7) >> 3) + ((p.rp_words + 7) >> 3));
    return (size_t)C::MIN_BLOCKS * (tab + (size_t)C::BYTES * C::WPB + 64) <= 227u * 1024u;
}

// the layout the plan's kernel 3 would use takes one queue per map (the host
// then seeds the map queues: SearchParams::map_queues)
bool k3_map_queues(const SearchParams& p) {
    const char* e = std::getenv("WPM_MAPQ");
    if (e && std::atoi(e) == 0) return false;
    const char* ts_env = std::getenv("WPM_TS");
    if (ts_env && std::atoi(ts_env) == 0) return false;
    if (p.max_depth > FRAME_CAP || p.cutoff > 0 || p.claim_recs) return false;
    const int N = p.max_N, M = p.max_M;
    if (N > C6::kN && N <= C7M::kN && M <= C7M::kM) return ts_fits<C7M>(p);
    if (N > C7::kN && N <= C8M::kN && M <= C8M::kM) return ts_fits<C8M>(p);
    if (N > C8::kN && N <= C9M::kN && M <= C9M::kM) return ts_fits<C9M>(p);
    if (N > C9::kN && N <= C10M::kN && M <= C10M::kM) return ts_fits<C10M>(p);
    return false;
}

// the smallest size class that holds the plan (max_depth > FRAME_CAP asks for
// the full-depth layout); the shared-memory-table variant when it fits
// (WPM_TS=0 disables it)
int launch_k3_search(const SearchParams& p, int num_sms, cudaStream_t st, int* warps_out) {
    const int N = p.max_N, M = p.max_M;
    if (p.max_depth > FRAME_CAP) return launch_class<CGF>(p, num_sms, st, warps_out);
    const char* ts_env = std::getenv("WPM_TS");
    const bool ts_on = !ts_env || std::atoi(ts_env) != 0;
    if (ts_on) {
        if (N <= C5T::kN && M <= C5T::kM && ts_fits<C5T>(p)) return launch_class<C5T>(p, num_sms, st, warps_out);
        if (p.map_queues) {
            if (N <= C7M::kN && M <= C7M::kM) return launch_class<C7M>(p, num_sms, st, warps_out);
            if (N <= C8M::kN && M <= C8M::kM) return launch_class<C8M>(p, num_sms, st, warps_out);
            if (N <= C9M::kN && M <= C9M::kM) return launch_class<C9M>(p, num_sms, st, warps_out);
            return launch_class<C10M>(p, num_sms, st, warps_out);
        }
        if (N <= C6T::kN && M <= C6T::kM && N > C5T::kN && ts_fits<C6T>(p))
            return launch_class<C6T>(p, num_sms, st, warps_out);
        if (N <= C10T::kN && M <= C10T::kM && N > C9::kN && ts_fits<C10T>(p))
            return launch_class<C10T>(p, num_sms, st, warps_out);
        if (N <= C11T::kN && M <= C11T::kM && N > C10::kN && ts_fits<C11T>(p))
            return launch_class<C11T>(p, num_sms, st, warps_out);
        if (N <= C15T::kN && M <= C15T::kM && (N > C11::kN || M > C11::kM) && ts_fits<C15T>(p))
            return launch_class<C15T>(p, num_sms, st, warps_out);
    }
    if (N <= C5::kN && M <= C5::kM) return launch_class<C5>(p, num_sms, st, warps_out);
    if (N <= C6::kN && M <= C6::kM) return launch_class<C6>(p, num_sms, st, warps_out);
    if (N <= C7::kN && M <= C7::kM) return launch_class<C7>(p, num_sms, st, warps_out);
    if (N <= C8::kN && M <= C8::kM) return launch_class<C8>(p, num_sms, st, warps_out);
    if (N <= C9::kN && M <= C9::kM) return launch_class<C9>(p, num_sms, st, warps_out);
    if (N <= C10::kN && M <= C10::kM) return launch_class<C10>(p, num_sms, st, warps_out);
    if (N <= C11::kN && M <= C11::kM) return launch_class<C11>(p, num_sms, st, warps_out);
    if (N <= C15::kN && M <= C15::kM) return launch_class<C15>(p, num_sms, st, warps_out);
    return launch_class<CG>(p, num_sms, st, warps_out);
}

}  // namespace wpm
