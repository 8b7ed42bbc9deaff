// kbasis.h -- the reference's kernel basis / combination space (host, kbasis.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace wpm {

// IncidenceMatrix (incidence.hpp:18-32): ridges in canonical order
struct HostIncidence {
    int M = 0, N = 0;
    std::vector<std::vector<int>> cols;     // M: the ridges of each facet, ascending
    std::vector<std::vector<int>> parents;  // N: the facets of each ridge, ascending
};

// the combination space of one job, ready for the device odometer
struct CombinationSpaceHost {
    int s = 0;                    // kernel dimension
    int induced_blocks = 0;       // blocks of convenient_basis (before pinning)
    unsigned long long space = 0; // size_saturated() (search.hpp:70-78)
    int W32 = 0;                  // uint32 words per M-bit vector
    std::vector<uint32_t> base;   // XOR of the pinned-in generators
    std::vector<int> ncand;       // candidates per block, widest block first
    std::vector<uint32_t> deltas; // sum(ncand) * W32: XOR mask per candidate (candidate 0 = none)
    // coordinates: the usable generators (every generator of a block or free
    // singleton, i.e. everything but the pinned ones) in block order -- block b
    // of the sorted list owns gens [lo_b, lo_b + width_b), lo_b = sum of the
    // widths before it; its candidates are none, the singles, then the pairs
    // (i < j), in deltas order (search.hpp:88-93)
    std::vector<int> width;       // per block (1 = free singleton)
    std::vector<uint32_t> gens;   // usable generators * W32
};

// gf2_kernel -> convenient_basis -> apply_link_constraints -> combination
// space.  0 ok, 3 infeasible pins.
int build_space(const HostIncidence& A, const std::vector<int>& required, const std::vector<int>& forbidden,
                CombinationSpaceHost* out);

}  // namespace wpm
