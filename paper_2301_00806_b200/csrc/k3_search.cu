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
// Execution model (B200): a persistent grid, one DFS per warp.  Lanes
// cooperate on each node: lane k < n updates the k-th ridge of the included
// facet; exclusions are flattened (facet, ridge) pairs over 32 lanes with
// shared-memory atomics; the branch ridge is a warp min-reduction over the
// open-ridge bitset; the next candidate is a __ballot_sync over the ridge's
// <= 8 candidate slots (or over 32 facets at a closed node).  The per-warp
// search state lives in shared memory (ridge counts + undecided counts packed
// in one byte, facet status, an undo trail and the frame stack); the per-map
// tables are read-only global memory (L1 resident).
//
// Work sharing replaces parallel_for_index (parallel.hpp:27-54): a global
// queue of tasks (IN/OUT facet bitsets + the frame to resume).  Warps pop
// tasks; every few nodes a busy warp checks whether the queue runs short and,
// if so, donates its shallowest frame that still has untried children (it
// marks the frame exhausted and keeps going).  The tree explored is the same
// whoever explores it, so node counts are deterministic.
#include <cstdint>
#include <climits>

#include "wpm_dev.cuh"
#include "wpm_internal.h"

namespace wpm {

namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint8_t FU = 0, FIN = 1, FOUT = 2;
constexpr uint16_t TR_INC = 0x8000;
constexpr uint16_t CLOSED_FRAME = 0xFFFF;

enum TaskKind : uint32_t { T_SINGLE = 0, T_OPEN = 1, T_CLOSED = 2, T_ENTRY = 3 };

// per-warp shared-memory layout, byte offsets
struct Layout {
    int rs, fst, dpos, open, inb, trail, frames, bytes;
    int nw, mw;
};

__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline Layout make_layout(int maxM, int maxN, int maxDepth) {
    Layout L;
    const int MP = align16(maxM + 32), NP = align16(maxN + 32);
    L.nw = (maxN + 31) / 32;
    L.mw = (maxM + 31) / 32;
    int o = 0;
    L.rs = o;     o += NP;                  // uint8 per ridge: count | undecided << 2
    L.fst = o;    o += MP;                  // uint8 per facet
    L.dpos = o;   o += align16(2 * MP);     // uint16 per facet: trail index + 1 of its decision
    L.open = o;   o += align16(4 * L.nw + 4);   // open-ridge bitset
    L.inb = o;    o += align16(4 * L.mw + 4);   // IN facet bitset
    L.trail = o;  o += align16(2 * MP);     // uint16 per decision
    L.frames = o; o += align16(8 * (maxDepth + 2));
    L.bytes = o;
    return L;
}

struct Frame {  // two words
    uint32_t a;  // mark (low 16) | ridge or CLOSED_FRAME (high 16)
    uint32_t b;  // pos (low 16) | cur (high 16)
};

struct Warp {
    uint8_t* rs;
    uint32_t* rsw;
    uint8_t* fst;
    uint16_t* dpos;
    uint32_t* open;
    uint32_t* inb;
    uint16_t* trail;
    Frame* frames;
    int size, nopen, ndead, tl, depth;
};

struct MapView {
    int M, N, n, cap, map;
    const uint16_t* fr;
    const uint16_t* rp;
    const uint8_t* npar;
};

__device__ __forceinline__ unsigned lanemask_lt(int lane) { return (1u << lane) - 1u; }

// ------------------------------------------------------------ state updates

// av -= 1 on every ridge of the facets trail[lo..hi) (already marked OUT)
__device__ __forceinline__ void apply_exclusions(Warp& w, const MapView& mp, int lo, int hi, int lane) {
    const int n = mp.n;
    for (int e0 = lo; e0 < hi; e0 += 2) {
        const int e = e0 + (lane >> 4), k = lane & 15;
        bool dead = false;
        if (e < hi && k < n) {
            const int g = w.trail[e] & 0x7FFF;
            const int r = __ldg(mp.fr + g * FR + k);
            const unsigned sh = (r & 3) * 8;
            const unsigned old = atomicSub(&w.rsw[r >> 2], 4u << sh);
            const unsigned ob = (old >> sh) & 0xFFu;
            dead = (ob & 3u) == 1u && (ob >> 2) == 1u;
        }
        w.ndead += __popc(__ballot_sync(FULL, dead));
    }
}

__device__ __forceinline__ void undo_exclusions(Warp& w, const MapView& mp, int lo, int hi, int lane) {
    const int n = mp.n;
    for (int e = lo + lane; e < hi; e += 32) w.fst[w.trail[e] & 0x7FFF] = FU;
    for (int e0 = lo; e0 < hi; e0 += 2) {
        const int e = e0 + (lane >> 4), k = lane & 15;
        bool undead = false;
        if (e < hi && k < n) {
            const int g = w.trail[e] & 0x7FFF;
            const int r = __ldg(mp.fr + g * FR + k);
            const unsigned sh = (r & 3) * 8;
            const unsigned old = atomicAdd(&w.rsw[r >> 2], 4u << sh);
            const unsigned ob = (old >> sh) & 0xFFu;
            undead = (ob & 3u) == 1u && (ob >> 2) == 0u;
        }
        w.ndead -= __popc(__ballot_sync(FULL, undead));
    }
    __syncwarp();
}

// exclude one facet (a tried sibling)
__device__ __forceinline__ void exclude_one(Warp& w, const MapView& mp, int g, int lane) {
    if (lane == 0) {
        w.fst[g] = FOUT;
        w.trail[w.tl] = (uint16_t)g;
        w.dpos[g] = (uint16_t)(w.tl + 1);
    }
    __syncwarp();
    apply_exclusions(w, mp, w.tl, w.tl + 1, lane);
    w.tl += 1;
    __syncwarp();
}

__device__ __forceinline__ void include_facet(Warp& w, const MapView& mp, int f, int lane) {
    const int n = mp.n;
    const bool act = lane < n;
    int r = 0;
    unsigned b = 0;
    if (act) {
        r = __ldg(mp.fr + f * FR + lane);
        b = w.rs[r];
    }
    const unsigned c = b & 3u, a = b >> 2;
    const unsigned nc = c + 1u, na = a - 1u;
    const bool opened = act && nc == 1u, closed = act && nc == 2u;
    if (act) w.rs[r] = (uint8_t)(nc | (na << 2));
    if (opened || closed) atomicXor(&w.open[r >> 5], 1u << (r & 31));
    const unsigned bo = __ballot_sync(FULL, opened), bc = __ballot_sync(FULL, closed);
    const unsigned bd = __ballot_sync(FULL, opened && na == 0u);
    w.nopen += __popc(bo) - __popc(bc);
    w.ndead += __popc(bd);
    if (lane == 0) {
        w.fst[f] = FIN;
        w.inb[f >> 5] |= 1u << (f & 31);
        w.trail[w.tl] = (uint16_t)(f | TR_INC);
        w.dpos[f] = (uint16_t)(w.tl + 1);
    }
    w.tl += 1;
    w.size += 1;
    __syncwarp();
    if (!bc) return;
    // propagation: closing ridges exclude their other undecided candidates.
    // Two ridges of f share no candidate besides f, so the list has no repeats.
    const int base = w.tl;
    int E = 0;
    unsigned rem = bc;
    while (rem) {
        const int jj = lane >> 3, q = lane & 7;
        const unsigned src = __fns(rem, 0, jj + 1);  // lane holding the (jj+1)-th closing ridge
        const int rr = __shfl_sync(FULL, r, (int)(src & 31u));
        bool v = false;
        int g = 0;
        if (src < 32u && q < (int)__ldg(mp.npar + rr)) {
            g = __ldg(mp.rp + rr * RP + q);
            v = w.fst[g] == FU;
        }
        const unsigned bv = __ballot_sync(FULL, v);
        if (v) {
            const int pos = base + E + __popc(bv & lanemask_lt(lane));
            w.trail[pos] = (uint16_t)g;
            w.fst[g] = FOUT;
            w.dpos[g] = (uint16_t)(pos + 1);
        }
        E += __popc(bv);
#pragma unroll
        for (int i = 0; i < 4; ++i) rem &= rem - 1u;
    }
    __syncwarp();
    if (E) apply_exclusions(w, mp, base, base + E, lane);
    w.tl += E;
    __syncwarp();
}

__device__ __forceinline__ void undo_include(Warp& w, const MapView& mp, int f, int lane) {
    const int n = mp.n;
    const bool act = lane < n;
    int r = 0;
    unsigned b = 0;
    if (act) {
        r = __ldg(mp.fr + f * FR + lane);
        b = w.rs[r];
    }
    const unsigned c = b & 3u, a = b >> 2;
    if (act) w.rs[r] = (uint8_t)((c - 1u) | ((a + 1u) << 2));
    const bool was_open = act && c == 1u, was_closed = act && c == 2u;
    if (was_open || was_closed) atomicXor(&w.open[r >> 5], 1u << (r & 31));
    const unsigned bo = __ballot_sync(FULL, was_open), bc = __ballot_sync(FULL, was_closed);
    const unsigned bd = __ballot_sync(FULL, was_open && a == 0u);
    w.nopen += __popc(bc) - __popc(bo);
    w.ndead -= __popc(bd);
    if (lane == 0) {
        w.fst[f] = FU;
        w.inb[f >> 5] &= ~(1u << (f & 31));
    }
    w.size -= 1;
    __syncwarp();
}

__device__ __noinline__ void undo_to(Warp& w, const MapView& mp, int mark, int lane) {
    while (w.tl > mark) {
        const int idx = w.tl - 1 - lane;
        const bool valid = idx >= mark;
        const unsigned e = valid ? w.trail[idx] : 0u;
        const unsigned bi = __ballot_sync(FULL, valid && (e & TR_INC));
        if (bi & 1u) {
            const int f = (int)(__shfl_sync(FULL, e, 0) & 0x7FFFu);
            undo_include(w, mp, f, lane);
            w.tl -= 1;
        } else {
            const int run = bi ? (__ffs(bi) - 1) : __popc(__ballot_sync(FULL, valid));
            undo_exclusions(w, mp, w.tl - run, w.tl, lane);
            w.tl -= run;
        }
    }
}

// open ridge with the fewest undecided candidates, ties by lowest id
__device__ __forceinline__ int select_ridge(const Warp& w, int nw, int lane) {
    unsigned best = 0xFFFFFFFFu;
    for (int i = lane; i < nw; i += 32) {
        unsigned bits = w.open[i];
        while (bits) {
            const int r = i * 32 + __ffs(bits) - 1;
            bits &= bits - 1u;
            const unsigned key = ((unsigned)(w.rs[r] >> 2) << 16) | (unsigned)r;
            best = min(best, key);
        }
    }
    best = __reduce_min_sync(FULL, best);
    return (int)(best & 0xFFFFu);
}

// --------------------------------------------------------------- the search

struct Ctx {
    SearchParams p;
    Layout L;
};

__device__ __forceinline__ void emit(Warp& w, const MapView& mp, const SearchParams& p, int lane) {
    unsigned long long slot = 0;
    if (lane == 0) {
        slot = atomicAdd(&p.out_ctl[0], 1ull);
        atomicAdd(&p.per_map[mp.map], 1ull);
    }
    slot = __shfl_sync(FULL, slot, 0);
    if (slot < p.out_cap) {
        uint32_t* o = p.out_bits + slot * (unsigned long long)p.w32;
        const int mw = (mp.M + 31) >> 5;
        for (int i = lane; i < p.w32; i += 32) o[i] = i < mw ? w.inb[i] : 0u;
        if (lane == 0) p.out_map[slot] = (uint16_t)mp.map;
    } else if (lane == 0) {
        atomicExch(&p.out_ctl[1], 1ull);
    }
}

// node entry after an include (or a task entry): emit / prune / push a frame.
// Returns true if a frame was pushed.
__device__ __forceinline__ bool enter_node(Warp& w, const MapView& mp, const SearchParams& p, int nw,
                                           int mark, bool may_emit, int lane) {
    if (w.ndead) return false;
    if (w.nopen == 0) {
        if (may_emit && w.size > 0) emit(w, mp, p, lane);
        if (w.size + mp.n + 1 > mp.cap) return false;
        if (lane == 0) {
            w.frames[w.depth].a = (uint32_t)mark | ((uint32_t)CLOSED_FRAME << 16);
            w.frames[w.depth].b = 0xFFFF0000u;  // pos 0, cur none
        }
    } else {
        if (w.size + (w.nopen + mp.n - 1) / mp.n > mp.cap) return false;
        const int r = select_ridge(w, nw, lane);
        if (lane == 0) {
            w.frames[w.depth].a = (uint32_t)mark | ((uint32_t)r << 16);
            w.frames[w.depth].b = 0xFFFF0000u;
        }
    }
    w.depth += 1;
    __syncwarp();
    return true;
}

// next undecided child of frame fr starting at its pos; -1 if none
__device__ __forceinline__ int next_child(const Warp& w, const MapView& mp, uint32_t fa, uint32_t fb,
                                          int* new_pos, int lane) {
    const int ridge = (int)(fa >> 16), pos = (int)(fb & 0xFFFFu);
    if (ridge == CLOSED_FRAME) {
        for (int p0 = pos; p0 < mp.M; p0 += 32) {
            const int f = p0 + lane;
            const bool ok = f < mp.M && w.fst[f] == FU;
            const unsigned b = __ballot_sync(FULL, ok);
            if (b) {
                const int c = p0 + __ffs(b) - 1;
                *new_pos = c + 1;
                return c;
            }
        }
        return -1;
    }
    const int np = __ldg(mp.npar + ridge);
    int g = 0;
    bool ok = false;
    if (lane < np && lane >= pos) {
        g = __ldg(mp.rp + ridge * RP + lane);
        ok = w.fst[g] == FU;
    }
    const unsigned b = __ballot_sync(FULL, ok);
    if (!b) return -1;
    const int q = __ffs(b) - 1;
    *new_pos = q + 1;
    return __shfl_sync(FULL, g, q);
}

// rebuild the per-warp state from an IN/OUT record (+ closure: a ridge with
// two IN candidates excludes the rest).  Returns false if infeasible.
__device__ bool load_state(Warp& w, const MapView& mp, const uint32_t* rec_in, const uint32_t* rec_out,
                           int nw, int lane) {
    const int M = mp.M, N = mp.N, mw = (M + 31) >> 5;
    int size = 0;
    for (int i = lane; i < mw; i += 32) {
        const uint32_t iv = __ldcg(rec_in + i);
        w.inb[i] = iv;
        size += __popc(iv);
    }
    for (int f = lane; f < M; f += 32) {
        const uint32_t iv = __ldcg(rec_in + (f >> 5)), ov = __ldcg(rec_out + (f >> 5));
        const uint32_t bit = 1u << (f & 31);
        w.fst[f] = (iv & bit) ? FIN : ((ov & bit) ? FOUT : FU);
        w.dpos[f] = 0;
    }
    w.size = __reduce_add_sync(FULL, (unsigned)size);
    __syncwarp();
    // pass 1: IN counts; a count >= 3 is infeasible
    bool bad = false;
    for (int r = lane; r < N; r += 32) {
        const int np = __ldg(mp.npar + r);
        unsigned c = 0;
        for (int q = 0; q < np; ++q) c += w.fst[__ldg(mp.rp + r * RP + q)] == FIN;
        if (c > 2u) bad = true;
        w.rs[r] = (uint8_t)min(c, 2u);
    }
    if (__any_sync(FULL, bad)) return false;
    __syncwarp();
    // closure: undecided facets on a closed ridge are excluded
    for (int f = lane; f < M; f += 32) {
        if (w.fst[f] != FU) continue;
        bool on_closed = false;
        for (int k = 0; k < mp.n; ++k) on_closed |= w.rs[__ldg(mp.fr + f * FR + k)] == 2u;
        if (on_closed) w.fst[f] = FOUT;
    }
    __syncwarp();
    // pass 2: undecided counts, open bitset, open/dead tallies
    int nopen = 0, ndead = 0;
    for (int r0 = 0; r0 < nw * 32; r0 += 32) {
        const int r = r0 + lane;
        bool op = false, dd = false;
        if (r < N) {
            const int np = __ldg(mp.npar + r);
            unsigned a = 0;
            for (int q = 0; q < np; ++q) a += w.fst[__ldg(mp.rp + r * RP + q)] == FU;
            const unsigned c = w.rs[r];
            w.rs[r] = (uint8_t)(c | (a << 2));
            op = c == 1u;
            dd = op && a == 0u;
        }
        const unsigned bo = __ballot_sync(FULL, op);
        if (lane == 0) w.open[r0 >> 5] = bo;
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

// donate the shallowest frame that still has an untried child
__device__ void try_donate(Warp& w, const MapView& mp, const SearchParams& p, int lane) {
    const int M = mp.M, mw = (M + 31) >> 5;
    for (int d = 0; d < w.depth; ++d) {
        const uint32_t fa = w.frames[d].a, fb = w.frames[d].b;
        const bool top = d + 1 == w.depth;
        const int mk = top ? w.tl : (int)(w.frames[d + 1].a & 0xFFFFu);
        const int cur = top ? -1 : (int)(fb >> 16);
        const int ridge = (int)(fa >> 16), pos = (int)(fb & 0xFFFFu);
        bool any = false;
        if (ridge == CLOSED_FRAME) {
            for (int f0 = pos; f0 < M && !any; f0 += 32) {
                const int f = f0 + lane;
                const bool ok = f < M && f != cur && (w.fst[f] == FU || (int)w.dpos[f] > mk);
                any = __any_sync(FULL, ok);
            }
        } else {
            const int np = __ldg(mp.npar + ridge);
            bool ok = false;
            if (lane < np && lane >= pos) {
                const int g = __ldg(mp.rp + ridge * RP + lane);
                ok = g != cur && (w.fst[g] == FU || (int)w.dpos[g] > mk);
            }
            any = __any_sync(FULL, ok);
        }
        if (!any) continue;
        // claim a queue slot
        unsigned long long t = 0;
        if (lane == 0) {
            atomicAdd(&p.qctl[2], 1ull);  // pending, before publishing
            t = atomicAdd(&p.qctl[1], 1ull);
        }
        t = __shfl_sync(FULL, t, 0);
        uint32_t* rec = p.qrec + (t % (unsigned long long)p.qcap) * (unsigned long long)p.recw;
        if (lane == 0) {
            rec[0] = (uint32_t)mp.map | ((ridge == CLOSED_FRAME ? (uint32_t)T_CLOSED : (uint32_t)T_OPEN) << 24);
            rec[1] = (uint32_t)ridge;
            rec[2] = (uint32_t)pos;
            rec[3] = 0;
        }
        for (int f0 = 0; f0 < mw * 32; f0 += 32) {
            const int f = f0 + lane;
            bool in = false, out = false;
            if (f < M) {
                const uint8_t s = w.fst[f];
                const bool before = (int)w.dpos[f] <= mk;
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
            atomicExch(&p.qready[t % (unsigned long long)p.qcap], t + 1ull);
            w.frames[d].b = (fb & 0xFFFF0000u) | 0xFFFFu;  // exhausted
        }
        __syncwarp();
        return;
    }
}

__global__ void __launch_bounds__(128) k3_search(SearchParams p, Layout L) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t* base = smem + (size_t)wid * L.bytes;
    Warp w;
    w.rs = base + L.rs;
    w.rsw = reinterpret_cast<uint32_t*>(base + L.rs);
    w.fst = base + L.fst;
    w.dpos = reinterpret_cast<uint16_t*>(base + L.dpos);
    w.open = reinterpret_cast<uint32_t*>(base + L.open);
    w.inb = reinterpret_cast<uint32_t*>(base + L.inb);
    w.trail = reinterpret_cast<uint16_t*>(base + L.trail);
    w.frames = reinterpret_cast<Frame*>(base + L.frames);
    unsigned long long nodes = 0, tasks = 0;
    unsigned backoff = 64;

    for (;;) {
        // ---- pop a task (lane 0), broadcast
        long long t = -1;
        if (lane == 0) {
            for (;;) {
                const unsigned long long h = atomicAdd(&p.qctl[0], 0ull);
                const unsigned long long tl = atomicAdd(&p.qctl[1], 0ull);
                if (h >= tl) break;
                if (atomicCAS(&p.qctl[0], h, h + 1ull) == h) {
                    t = (long long)h;
                    break;
                }
            }
            if (t < 0) {
                const unsigned long long pend = atomicAdd(&p.qctl[2], 0ull);
                if (pend == 0ull) t = -2;
            }
        }
        t = __shfl_sync(FULL, t, 0);
        if (t == -2) break;
        if (t == -1) {
            __nanosleep(backoff);
            backoff = min(backoff * 2u, 4096u);
            continue;
        }
        backoff = 64;
        const unsigned long long slot = (unsigned long long)t % (unsigned long long)p.qcap;
        if (lane == 0)
            while (atomicAdd(&p.qready[slot], 0ull) != (unsigned long long)t + 1ull) __nanosleep(32);
        __syncwarp();
        __threadfence();
        const uint32_t* rec = p.qrec + slot * (unsigned long long)p.recw;
        const uint32_t h0 = __ldcg(rec), h1 = __ldcg(rec + 1), h2 = __ldcg(rec + 2);
        const int map = (int)(h0 & 0xFFFFu);
        const uint32_t kind = h0 >> 24;
        const MapDesc md = p.maps[map];
        MapView mp;
        mp.M = md.M;
        mp.N = md.N;
        mp.n = md.n;
        mp.cap = md.cap;
        mp.map = map;
        mp.fr = p.fr + md.fr_off;
        mp.rp = p.rp + md.rp_off;
        mp.npar = p.npar + md.np_off;
        const int nw = (mp.N + 31) >> 5;
        ++tasks;

        bool alive = load_state(w, mp, rec + 4, rec + 4 + p.mw, nw, lane);
        if (alive) {
            if (kind == T_SINGLE) {
                const int f = (int)h1;
                include_facet(w, mp, f, lane);
                ++nodes;
                enter_node(w, mp, p, nw, 0, true, lane);
            } else if (kind == T_ENTRY) {
                enter_node(w, mp, p, nw, 0, true, lane);
            } else if (w.ndead == 0) {
                if (lane == 0) {
                    w.frames[0].a = (kind == T_CLOSED) ? ((uint32_t)CLOSED_FRAME << 16) : (h1 << 16);
                    w.frames[0].b = 0xFFFF0000u | (h2 & 0xFFFFu);
                }
                w.depth = 1;
                __syncwarp();
            }
        }
        // ---- the DFS
        unsigned since_check = 0;
        while (w.depth > 0) {
            Frame& F = w.frames[w.depth - 1];
            const uint32_t fa = F.a, fb = F.b;
            int npos = 0;
            const int c = ((fb & 0xFFFFu) == 0xFFFFu) ? -1 : next_child(w, mp, fa, fb, &npos, lane);
            if (c < 0) {
                undo_to(w, mp, (int)(fa & 0xFFFFu), lane);
                w.depth -= 1;
                if (w.depth > 0) {
                    Frame& P = w.frames[w.depth - 1];
                    const uint32_t pb = P.b;
                    exclude_one(w, mp, (int)(pb >> 16), lane);
                    if ((P.a >> 16) != CLOSED_FRAME && w.ndead) {
                        if (lane == 0) P.b = pb | 0xFFFFu;
                        __syncwarp();
                    }
                }
                continue;
            }
            if (lane == 0) F.b = ((uint32_t)c << 16) | (uint32_t)npos;
            __syncwarp();
            const int mark = w.tl;
            include_facet(w, mp, c, lane);
            ++nodes;
            if (!enter_node(w, mp, p, nw, mark, true, lane)) {
                undo_to(w, mp, mark, lane);
                exclude_one(w, mp, c, lane);
                if ((fa >> 16) != CLOSED_FRAME && w.ndead) {
                    if (lane == 0) F.b = (F.b & 0xFFFF0000u) | 0xFFFFu;
                    __syncwarp();
                }
            }
            if (++since_check >= 16u) {
                since_check = 0;
                int hungry = 0;
                if (lane == 0) {
                    const unsigned long long h = *(volatile unsigned long long*)&p.qctl[0];
                    const unsigned long long tl = *(volatile unsigned long long*)&p.qctl[1];
                    hungry = (tl - h) < (unsigned long long)p.hungry;
                }
                if (__shfl_sync(FULL, hungry, 0)) try_donate(w, mp, p, lane);
            }
        }
        // task finished
        if (lane == 0) atomicAdd(&p.qctl[2], (unsigned long long)-1ll);
    }
    if (lane == 0) {
        atomicAdd(&p.qctl[3], tasks);
        atomicAdd(&p.qctl[4], nodes);
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
    uint32_t* rec = p.qrec + (size_t)t * p.recw;
    if (lane == 0) {
        rec[0] = (uint32_t)map | ((uint32_t)kind << 24);
        rec[1] = (uint32_t)f;
        rec[2] = 0;
        rec[3] = 0;
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
    if (lane == 0) p.qready[t] = (unsigned long long)t + 1ull;
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

int launch_k3_search(const SearchParams& p, int num_sms, cudaStream_t st, int* warps_out) {
    const Layout L = make_layout(p.max_M, p.max_N, p.max_depth);
    const int wpb = 4;  // warps per CTA
    const size_t smem = (size_t)L.bytes * wpb;
    if (cudaFuncSetAttribute(k3_search, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k3_search, 32 * wpb, smem) != cudaSuccess ||
        per_sm < 1)
        return 0;
    const int grid = per_sm * num_sms;
    k3_search<<<grid, 32 * wpb, smem, st>>>(p, L);
    if (cudaGetLastError() != cudaSuccess) return 0;
    if (warps_out) *warps_out = grid * wpb;
    return grid;
}

int k3_layout_bytes(int maxM, int maxN, int maxDepth) { return make_layout(maxM, maxN, maxDepth).bytes; }

}  // namespace wpm
