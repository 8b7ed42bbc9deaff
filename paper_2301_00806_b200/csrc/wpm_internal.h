// wpm_internal.h -- host-side launchers of the device kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "wpm_dev.cuh"

namespace wpm {

// kernel 1: universes of num_maps characteristic maps (m columns each)
int launch_k1_universe(int n, int m, int num_maps, const uint32_t* d_cols, uint32_t* d_facets,
                       int facet_stride, int32_t* d_M, cudaStream_t st);

// kernel 2: incidence tables for every map of `maps` (facets already placed)
int launch_k2_incidence(int num_maps, const MapDesc* d_maps, int max_m, int max_n,
                        const uint32_t* d_facets, uint32_t* d_ridges, uint16_t* d_fr, uint16_t* d_rp,
                        uint8_t* d_npar, int32_t* d_N, int32_t* d_err, cudaStream_t st);

// kernel 3: the persistent work-sharing DFS
struct SearchParams {
    int num_maps;
    int max_M, max_N, max_n, max_depth;  // sizing of per-warp shared state
    const MapDesc* maps;
    const uint16_t* fr;
    const uint16_t* rp;
    const uint8_t* npar;  // host-side parity hook only
    // work queue
    uint32_t* qrec;
    unsigned long long* qready;
    unsigned long long* qctl;  // [0] tail << 32 | head, [2] pending, [3] tasks done, [4] nodes
    int qcap, recw, mw;
    int hungry;                 // donate while queued tasks < hungry
    int backoff_max;            // ns, idle warps' polling backoff cap
    // output
    uint32_t* out_bits;         // out_cap * w32
    uint16_t* out_map;
    unsigned long long* out_ctl;  // [0] count, [1] overflow flag
    unsigned long long* per_map;  // num_maps counts
    unsigned long long out_cap;
    int w32;
};

// seeds root tasks (map, f) in queue order; required/forbidden lists for ENTRY tasks
int launch_seed_tasks(const SearchParams& p, int ntasks, const int32_t* d_task_map,
                      const int32_t* d_task_f, const int32_t* d_task_kind, const uint32_t* d_pin_in,
                      const uint32_t* d_pin_out, cudaStream_t st);

// returns grid size used (0 on error)
int launch_k3_search(const SearchParams& p, int num_sms, cudaStream_t st, int* warps_out);

// canonical sort: orders out_bits/out_map (count rows) by (map, canonical order)
// into sorted_bits, reports duplicates
int canon_sort(const uint32_t* d_bits, const uint16_t* d_map, long long count, int w32,
               uint32_t* d_sorted_bits, uint16_t* d_sorted_map, void* d_temp, size_t temp_bytes,
               uint32_t* d_idx_a, long long* d_first_row, unsigned long long* d_dups, cudaStream_t st);
size_t canon_sort_temp_bytes(long long count, int w32);

// INT32 lane-op issue peak (LOP3 + IADD3 chains over every SM), ops/s
int int_peak_measure(int device, double* ops_per_s);

}  // namespace wpm
