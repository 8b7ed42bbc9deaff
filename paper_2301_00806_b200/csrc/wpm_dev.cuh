// wpm_dev.cuh -- device-side layout shared by the three sm_100a kernels.
//
// HBM layout per map (built by kernel 1 / kernel 2, read by kernel 3 through
// the read-only path, L1-resident: <= 60 KB per map at n = 11):
//   facets  uint32[M]          vertex masks, bit v = vertex v, ascending
//   ridges  uint32[N]          ascending (complex.hpp:107-119 order)
//   fr      uint16[M * FR]     the n ridge ids of each facet, ascending
//                              (IncidenceMatrix::cols, incidence.hpp:27)
//   rp      uint16[N * RP]     candidate facets of each ridge, ascending,
//                              0xFFFF padded (IncidenceMatrix::parents)
//   npar    uint8[N]
#pragma once
#include <cstdint>

namespace wpm {

constexpr int FR = 16;             // fr stride (n <= 15)
constexpr int RP = 8;              // rp stride (<= 8 candidate facets per ridge)
constexpr int MAXM_LABELS = 16;    // vertex labels 1..16
constexpr int MAX_FACETS = 2048;
constexpr int MAX_RIDGES = 4096;
constexpr uint16_t NONE16 = 0xFFFF;

struct MapDesc {
    int32_t M, N, n, m;
    int32_t cap;        // facet cap (INT32_MAX = none)
    int32_t fr_stride;  // = n
    int32_t rp_stride;  // = min(8, m - n + 1); 0xFFFF padded
    int32_t pad0;
    uint32_t facet_off; // into facets (uint32)
    uint32_t ridge_off; // into ridges (uint32)
    uint32_t fr_off;    // into fr (uint16)
    uint32_t rp_off;    // into rp (uint16)
    uint32_t np_off;    // into npar (uint8)
    uint32_t pad1;
};

// binomials C(a, b), a, b <= 16
struct Binom {
    uint32_t c[17][17];
};

__host__ __device__ inline uint32_t binom_small(int a, int b) {
    if (b < 0 || a < b) return 0;
    uint32_t r = 1;
    for (int i = 1; i <= b; ++i) r = r * (uint32_t)(a - b + i) / (uint32_t)i;
    return r;
}

// built once per process (a kernel argument of every launch that ranks subsets)
inline const Binom& make_binom() {
    static const Binom tab = [] {
        Binom b;
        for (int a = 0; a <= 16; ++a)
            for (int k = 0; k <= 16; ++k) b.c[a][k] = binom_small(a, k);
        return b;
    }();
    return tab;
}

}  // namespace wpm
