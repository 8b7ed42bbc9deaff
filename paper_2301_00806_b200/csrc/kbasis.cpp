// kbasis.cpp -- the reference's kernel-basis construction (host, product side).
//
// Algorithm 1 of the paper enumerates the GF(2) kernel of the ridge-facet
// incidence matrix through a "convenient" basis and its combination space.
// The device odometer (k6_odometer.cu) visits exactly the reference's leaves,
// so the basis must be the reference's basis, bit for bit:
//   gf2_kernel              bitmatrix.hpp:125-153 (on incidence.hpp:59-61)
//   try_make_block          kernel_basis.hpp:84-190
//   convenient_basis        kernel_basis.hpp:198-235
//   apply_link_constraints  kernel_basis.hpp:248-321
//   combination_space       search.hpp:81-104, block deltas search.hpp:156-166,
//                           widest blocks first search.hpp:168-170
// Generators are M-bit vectors over the facet universe (std::vector<uint64_t>).
#include <algorithm>
#include <cstdint>
#include <functional>
#include <utility>
#include <vector>

#include "kbasis.h"

namespace wpm {

namespace {

using Vec = std::vector<uint64_t>;

inline bool test(const Vec& v, int i) { return (v[i >> 6] >> (i & 63)) & 1u; }
inline void setb(Vec& v, int i) { v[i >> 6] |= uint64_t{1} << (i & 63); }
inline void xor_into(Vec& d, const Vec& s) {
    for (size_t w = 0; w < d.size(); ++w) d[w] ^= s[w];
}
inline int lead(uint64_t v) { return 63 - __builtin_clzll(v); }

// reduce v against an echelon kept in descending order (kernel_basis.hpp:63-67)
uint64_t reduce(uint64_t v, const std::vector<uint64_t>& ech) {
    for (uint64_t e : ech)
        if (v && lead(v) == lead(e)) v ^= e;
    return v;
}

uint64_t restrict_to(const Vec& g, const std::vector<int>& rows) {  // :69-74
    uint64_t v = 0;
    for (size_t i = 0; i < rows.size(); ++i)
        if (test(g, rows[i])) v |= uint64_t{1} << i;
    return v;
}

struct Basis {
    int M = 0;
    std::vector<Vec> gens;
    std::vector<std::pair<int, int>> blocks;  // (offset, width)
    int ones = 0, zeros = 0;
};

// raw kernel: one generator per free column, ascending (bitmatrix.hpp:125-153)
std::vector<Vec> gf2_kernel(const HostIncidence& A) {
    const int M = A.M, N = A.N, W = (M + 63) / 64;
    std::vector<Vec> a(N, Vec(W, 0));
    for (int j = 0; j < M; ++j)
        for (int r : A.cols[j]) setb(a[r], j);
    std::vector<int> pivot_col;
    int rank = 0;
    for (int c = 0; c < M && rank < N; ++c) {
        int piv = -1;
        for (int r = rank; r < N && piv < 0; ++r)
            if (test(a[r], c)) piv = r;
        if (piv < 0) continue;
        std::swap(a[rank], a[piv]);
        for (int r = 0; r < N; ++r)
            if (r != rank && test(a[r], c)) xor_into(a[r], a[rank]);
        pivot_col.push_back(c);
        ++rank;
    }
    std::vector<char> is_piv(M, 0);
    for (int c : pivot_col) is_piv[c] = 1;
    std::vector<Vec> out;
    for (int fc = 0; fc < M; ++fc) {
        if (is_piv[fc]) continue;
        Vec v(W, 0);
        setb(v, fc);
        for (int r = 0; r < rank; ++r)
            if (test(a[r], fc)) setb(v, pivot_col[r]);
        out.push_back(std::move(v));
    }
    return out;
}

bool try_make_block(Basis& kb, const std::vector<int>& P, int offset) {  // :84-190
    const int p = (int)P.size();
    if (p < 3 || p > 64) return false;
    const int s = (int)kb.gens.size();
    std::vector<uint64_t> ech;
    for (int g = offset; g < s; ++g) {
        const uint64_t v = reduce(restrict_to(kb.gens[g], P), ech);
        if (v) {
            ech.push_back(v);
            std::sort(ech.begin(), ech.end(), std::greater<>());
        }
    }
    const int k = (int)ech.size();
    if (k < 2) return false;
    // weight-2 members of the span: union-find on the parent rows (:99-116)
    std::vector<int> comp(p);
    for (int i = 0; i < p; ++i) comp[i] = i;
    auto find = [&](int x) {
        while (comp[x] != x) x = comp[x] = comp[comp[x]];
        return x;
    };
    for (int a = 0; a < p; ++a)
        for (int b = a + 1; b < p; ++b)
            if (reduce((uint64_t{1} << a) | (uint64_t{1} << b), ech) == 0) {
                const int ra = find(a), rb = find(b);
                if (ra != rb) comp[ra] = rb;
            }
    std::vector<int> clique;
    for (int root = 0; root < p && clique.empty(); ++root) {
        if (find(root) != root) continue;
        std::vector<int> mem;
        for (int i = 0; i < p; ++i)
            if (find(i) == root) mem.push_back(i);
        if ((int)mem.size() == k + 1) clique = std::move(mem);
    }
    if (clique.empty()) return false;
    for (int g = 0; g < offset; ++g)
        if (reduce(restrict_to(kb.gens[g], P), ech) != 0) return false;
    // commit: forward echelon with generator bookkeeping (:133-147)
    std::vector<std::pair<uint64_t, int>> piv;
    for (int g = offset; g < s; ++g) {
        uint64_t v = restrict_to(kb.gens[g], P);
        for (auto& [pv, pg] : piv)
            if (v && lead(v) == lead(pv)) {
                v ^= pv;
                xor_into(kb.gens[g], kb.gens[pg]);
            }
        if (v) {
            piv.emplace_back(v, g);
            std::sort(piv.begin(), piv.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
        }
    }
    const int last = clique.back();
    std::vector<Vec> star;
    std::vector<int> star_row;
    for (size_t i = 0; i + 1 < clique.size(); ++i) {  // :152-166
        uint64_t v = (uint64_t{1} << clique[i]) | (uint64_t{1} << last);
        Vec combo(kb.gens[0].size(), 0);
        for (auto& [pv, pg] : piv)
            if (v && lead(v) == lead(pv)) {
                v ^= pv;
                xor_into(combo, kb.gens[pg]);
            }
        if (v) return false;
        star.push_back(std::move(combo));
        star_row.push_back(clique[i]);
    }
    std::vector<Vec> tail;  // star generators first, then the non-pivots (:168-177)
    for (auto& b : star) tail.push_back(std::move(b));
    std::vector<char> is_piv(s, 0);
    for (auto& pp : piv) is_piv[pp.second] = 1;
    for (int g = offset; g < s; ++g)
        if (!is_piv[g]) tail.push_back(std::move(kb.gens[g]));
    for (int g = offset; g < s; ++g) kb.gens[g] = std::move(tail[g - offset]);
    for (int g = 0; g < offset; ++g) {  // clear earlier columns (:180-186)
        const uint64_t u = restrict_to(kb.gens[g], P);
        if (!u) continue;
        for (size_t i = 0; i < star_row.size(); ++i)
            if ((u >> star_row[i]) & 1u) xor_into(kb.gens[g], kb.gens[offset + (int)i]);
    }
    kb.blocks.emplace_back(offset, k);
    return true;
}

void convenient_basis(Basis& kb, const HostIncidence& A) {  // :198-235
    std::vector<char> ridge_used(A.N, 0), facet_used(A.M, 0);
    int offset = 0;
    while (offset < (int)kb.gens.size()) {
        std::vector<int> cand;
        for (int r = 0; r < A.N; ++r) {
            if (ridge_used[r]) continue;
            bool disjoint = true;
            for (int f : A.parents[r])
                if (facet_used[f]) {
                    disjoint = false;
                    break;
                }
            if (disjoint) cand.push_back(r);
        }
        std::sort(cand.begin(), cand.end(), [&](int a, int b) {
            const size_t pa = A.parents[a].size(), pb = A.parents[b].size();
            return pa != pb ? pa > pb : a < b;
        });
        bool advanced = false;
        for (int r : cand) {
            ridge_used[r] = 1;
            if (try_make_block(kb, A.parents[r], offset)) {
                for (int f : A.parents[r]) facet_used[f] = 1;
                offset += kb.blocks.back().second;
                advanced = true;
                break;
            }
        }
        if (!advanced) break;
    }
}

// :248-321; false = infeasible
bool apply_link_constraints(Basis& kb, const std::vector<int>& req, const std::vector<int>& forb) {
    if (req.empty() && forb.empty()) return true;
    for (int r : req)
        for (int f : forb)
            if (r == f) return false;
    std::vector<Vec> gens = kb.gens;
    const int s = (int)gens.size();
    std::vector<std::pair<int, bool>> rows;
    for (int f : req) rows.emplace_back(f, true);
    for (int f : forb) rows.emplace_back(f, false);
    std::vector<int> pivot_of_row(rows.size(), -1);
    int cur = 0;
    for (size_t ri = 0; ri < rows.size(); ++ri) {
        const int facet = rows[ri].first;
        int pivot = -1;
        for (int g = cur; g < s && pivot < 0; ++g)
            if (test(gens[g], facet)) pivot = g;
        if (pivot < 0) continue;
        std::swap(gens[pivot], gens[cur]);
        for (int g = 0; g < s; ++g)
            if (g != cur && test(gens[g], facet)) xor_into(gens[g], gens[cur]);
        pivot_of_row[ri] = cur++;
    }
    std::vector<int> ones, zeros;
    for (size_t ri = 0; ri < rows.size(); ++ri) {
        const int g = pivot_of_row[ri];
        if (g < 0) continue;
        (rows[ri].second ? ones : zeros).push_back(g);
    }
    for (auto& row : rows) {
        bool value = false;
        for (int g : ones)
            if (test(gens[g], row.first)) value = !value;
        if (value != row.second) return false;
    }
    std::vector<Vec> out;
    std::vector<char> placed(s, 0);
    for (int g : ones) out.push_back(gens[g]), placed[g] = 1;
    for (int g : zeros) out.push_back(gens[g]), placed[g] = 1;
    for (int g = 0; g < s; ++g)
        if (!placed[g]) out.push_back(gens[g]);
    kb.gens = std::move(out);
    kb.blocks.clear();  // blocks do not survive the re-elimination (:246-247)
    kb.ones = (int)ones.size();
    kb.zeros = (int)zeros.size();
    return true;
}

}  // namespace

int build_space(const HostIncidence& A, const std::vector<int>& required, const std::vector<int>& forbidden,
                CombinationSpaceHost* out) {
    Basis kb;
    kb.M = A.M;
    kb.gens = gf2_kernel(A);
    if (!kb.gens.empty()) convenient_basis(kb, A);
    out->s = (int)kb.gens.size();
    out->induced_blocks = (int)kb.blocks.size();
    if (!apply_link_constraints(kb, required, forbidden)) return 3;
    const int W32 = (A.M + 31) / 32;
    auto to32 = [&](const Vec& v, uint32_t* dst) {
        for (int w = 0; w < W32; ++w) dst[w] = (uint32_t)(v[w >> 1] >> ((w & 1) * 32));
    };
    Vec base((A.M + 63) / 64, 0);
    for (int g = 0; g < kb.ones; ++g) xor_into(base, kb.gens[g]);
    // combination_space (search.hpp:81-104): each induced block {0, singles,
    // pairs}, then every uncovered generator as a free {0, g}
    std::vector<std::vector<Vec>> blocks;
    std::vector<std::vector<int>> bgens;  // the generators of each block
    const Vec zero(base.size(), 0);
    int covered = kb.ones + kb.zeros;
    for (auto [off, wd] : kb.blocks) {
        std::vector<Vec> c{zero};
        std::vector<int> gi;
        for (int i = 0; i < wd; ++i) c.push_back(kb.gens[off + i]), gi.push_back(off + i);
        for (int i = 0; i < wd; ++i)
            for (int j = i + 1; j < wd; ++j) {
                Vec d = kb.gens[off + i];
                xor_into(d, kb.gens[off + j]);
                c.push_back(std::move(d));
            }
        blocks.push_back(std::move(c));
        bgens.push_back(std::move(gi));
        covered = std::max(covered, off + wd);
    }
    for (int g = covered; g < (int)kb.gens.size(); ++g) blocks.push_back({zero, kb.gens[g]}), bgens.push_back({g});
    // widest blocks outermost (search.hpp:168-170, stable)
    std::vector<int> order(blocks.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return blocks[a].size() > blocks[b].size(); });
    {
        std::vector<std::vector<Vec>> sb;
        std::vector<std::vector<int>> sg;
        for (int i : order) sb.push_back(std::move(blocks[i])), sg.push_back(std::move(bgens[i]));
        blocks = std::move(sb);
        bgens = std::move(sg);
    }
    unsigned long long space = 1;
    bool sat = false;
    for (auto& b : blocks) {
        const unsigned long long c = b.size();
        if (space > ~0ull / c) {
            sat = true;
            break;
        }
        space *= c;
    }
    out->space = sat ? ~0ull : space;
    out->W32 = W32;
    out->base.assign(W32, 0);
    to32(base, out->base.data());
    out->ncand.clear();
    out->deltas.clear();
    out->width.clear();
    out->gens.clear();
    for (auto& gi : bgens) {
        out->width.push_back((int)gi.size());
        for (int g : gi) {
            const size_t at = out->gens.size();
            out->gens.resize(at + W32);
            to32(kb.gens[g], out->gens.data() + at);
        }
    }
    for (auto& b : blocks) {
        out->ncand.push_back((int)b.size());
        for (auto& d : b) {
            const size_t at = out->deltas.size();
            out->deltas.resize(at + W32);
            to32(d, out->deltas.data() + at);
        }
    }
    return 0;
}

}  // namespace wpm
