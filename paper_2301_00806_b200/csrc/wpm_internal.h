// wpm_internal.h -- host-side launchers of the device kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

#include "wpm_dev.cuh"

namespace wpm {

// Resident CTAs per SM of kernel `fn` at (threads, dynamic smem) on the
// current device, with its dynamic-smem limit raised to at least `smem`: the
// per-launch cudaFuncSetAttribute + occupancy query pair cost ~3-5 us of host
// time per launch (WPM_TRACE=2), paid by every one-shot call.  The limit only
// ever grows (a later launch with less smem must not lower it under an
// earlier, larger one).  0 on error.
inline int occupancy_cached(const void* fn, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, size_t, int>, int> memo;
    static std::map<std::pair<const void*, int>, size_t> limit;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    std::lock_guard<std::mutex> lk(mu);
    size_t& lim = limit[std::make_pair(fn, dev)];
    if (lim < smem) {
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
        lim = smem;
    }
    const auto key = std::make_tuple(fn, threads, smem, dev);
    auto it = memo.find(key);
    if (it != memo.end()) return it->second;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess) return 0;
    memo[key] = per_sm;
    return per_sm;
}

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
    int fr_words, rp_words;  // uint16 entries of fr / rp over every map (16-byte padded arrays)
    // work queue
    uint32_t* qrec;
    unsigned long long* qready;
    unsigned long long* qctl;  // [0] tail << 32 | head, [2] pending, [3] tasks done, [4] nodes
    int qcap, recw, mw;
    int hungry;                 // donate while queued tasks < hungry
    int backoff_min;            // ns, idle warps' first polling sleep
    int backoff_max;            // ns, idle warps' polling backoff cap
    int check_every;            // search nodes between looks at the queue word (donation check)
    int first_check;            // ... and before the first look of a task (<= check_every)
    int starve_at, starve_check;  // more than starve_at warps waiting: look every starve_check nodes
    int donate_max;             // frames donated per check while warps wait
    // output: one key row per WPM = kw bitset words (zero padded) + the map id
    uint32_t* out_keys;         // out_cap * rw
    unsigned long long* out_ctl;  // [0] count, [1] duplicates (after the sort)
    unsigned long long* per_map;  // scratch: first row per map (after the sort)
    unsigned long long out_cap;
    int rw;                     // key row words = key_words_for(w32) + 1
    // node budget (0 = none): warps flush their node counts into qctl[1]
    // at every queue check and stop once the total reaches it (out_ctl[3]
    // = 1: the run is truncated -- a throughput stress, not an enumeration)
    unsigned long long node_budget;
    // frontier expansion (cutoff > 0): a branch frame at absolute depth >=
    // cutoff is not explored; its state is appended to front_out (a task
    // record) instead -- the split of the search tree below the root
    int cutoff;
    uint32_t* front_out;
    unsigned long long* front_ctl;   // [0] records written (may exceed front_cap: rerun)
    unsigned long long front_cap;
    // claim mode: idle warps pull frontier records claim_recs[i] (a local
    // copy) by i = atomicAdd on *claim_ctr -- one counter shared by every GPU
    // of the job (peer or IPC memory, system-scope atomics) -- while fewer
    // than claim_low tasks are pending on this GPU
    const uint32_t* claim_recs;
    long long claim_count;
    unsigned long long* claim_ctr;
    int claim_low;
    // progress (search.hpp:54, :244): root_pend[root] = unfinished tasks of
    // each root task (header word 3); a finished root bumps roots_done and
    // publishes it to host-mapped memory (optional)
    unsigned int* root_pend;
    unsigned long long* roots_done;
    unsigned long long* progress_host;
    unsigned long long* root_nodes;  // optional: search nodes per root task / frontier record
    // one queue per map (k3_map_queues): queue q = qctl[8 (q + 1) ..], qready
    // / qrec from q * qcap; root task t of map q is slot t - map_first[q]
    int map_queues;
    int ma_tab_bytes;          // shared bytes of the largest map's fr + rp tables (16-byte padded each)
    const int32_t* map_first;  // num_maps + 1 prefix of root tasks per map
};
// kernel 3 for this plan runs one queue per map (see SearchParams::map_queues)
bool k3_map_queues(const SearchParams& p);

// task record header (queue, frontier): [0] map | kind << 24, [1] facet or
// ridge, [2] resume position | absolute branch depth << 16, [3] root task id;
// then the IN and OUT facet bitsets (mw words each)
int launch_seed_records(const SearchParams& p, const uint32_t* d_recs, long long count, cudaStream_t st);
int launch_fill_u32(unsigned int* d, unsigned int v, long long count, cudaStream_t st);

// seeds root tasks (map, f) in queue order; required/forbidden lists for ENTRY tasks
int launch_seed_tasks(const SearchParams& p, int ntasks, const int32_t* d_task_map,
                      const int32_t* d_task_f, const int32_t* d_task_kind, const uint32_t* d_pin_in,
                      const uint32_t* d_pin_out, cudaStream_t st);

// returns grid size used (0 on error)
int launch_k3_search(const SearchParams& p, int num_sms, cudaStream_t st, int* warps_out);

// canonical sort (k4_canon.cu).  Key rows: key_words_for(w32) bitset words +
// the map id.  canon_sort_keys sorts them in place by (map, canonical order)
// and splits them into sorted_bits (w32 words per row) / sorted_map, with the
// first row of each map and the adjacent-duplicate count.
int key_words_for(int w32);
// record layout of every sort input (kernel 3, kernel 6, the line-13 union):
// w32 bitset words, zero padding, the map id in the last word; the record is
// a whole number of 16-byte vectors
__host__ __device__ inline int rec_words(int w32) { return (w32 + 1 + 3) & ~3; }
size_t canon_sort_temp_bytes(long long count, int w32);
// d_count (optional): the row count on the device (read by the kernel,
// capped at `count`, which then only sizes the launch)
int canon_sort_keys(uint32_t* d_keys, long long count, int w32, uint32_t* d_sorted_bits, uint16_t* d_sorted_map,
                    void* d_temp, size_t temp_bytes, long long* d_first_row, unsigned long long* d_dups,
                    cudaStream_t st, const unsigned long long* d_count = nullptr, long long grid_rows = 0,
                    int out_words = 0);
// the general form: records of rw words (a multiple of 4, >= w32 + 1; the
// map id last), compared on (map, w32 bitset words) and then -- tie >= 0 --
// on word `tie` (a payload carried through the sort, written to d_payload);
// temp >= 2 * count * rw * 4 bytes; d_sorted_map / d_payload may be null
int canon_sort_records(uint32_t* d_keys, long long count, int w32, int rw, int tie, uint32_t* d_sorted_bits,
                       uint16_t* d_sorted_map, uint32_t* d_payload, void* d_temp, size_t temp_bytes,
                       long long* d_first_row, unsigned long long* d_dups, cudaStream_t st,
                       const unsigned long long* d_count = nullptr, long long grid_rows = 0,
                       int out_words = 0);
// (out_words > w32: sorted_bits rows of out_words words, zero beyond w32 --
// kernel 3 emits only the mw words a plan's bitsets use, the C-ABI rows are
// whole 64-bit words)
// the bucketed form for kernel-3 rows of a plan (k4_bucket): rows bucketed
// by (map, three lowest facets) and sorted per bucket; output as above.
// scratch: bucket_sort_scratch_words(cap, total_facets) uint32 words whose
// count block (bucket_sort_count_offset(cap), B = 64 x total_facets words)
// is zero before the first sort (each sort leaves it zero)
size_t bucket_sort_scratch_words(long long cap, long long total_facets);
size_t bucket_sort_count_offset(long long cap);
int canon_sort_bucketed(const uint32_t* d_keys, long long cap, const unsigned long long* d_count, int w32, int rw,
                        int out_words, const MapDesc* d_maps, int num_maps, long long total_facets,
                        uint32_t* d_sorted_bits, uint16_t* d_sorted_map, long long* d_first_row,
                        unsigned long long* d_dups, void* d_temp, size_t temp_bytes, uint32_t* d_scratch,
                        size_t scratch_words, cudaStream_t st, long long grid_rows = 0);
// stream compaction (one cooperative launch, hand-written): out[j] = the j-th
// i < n (ascending) with flags[i] != 0, as in[i] (in = null: i itself);
// *d_num = the count.  temp: compact_temp_bytes() bytes
size_t compact_temp_bytes();
int compact_flagged(const uint32_t* in, const uint8_t* flags, long long n, uint32_t* out, int* d_num, void* d_temp,
                    cudaStream_t st);
// rows (w32 words) + uint16 map ids -> key rows
int canon_pack(const uint32_t* d_bits, const uint16_t* d_map, long long count, int w32, uint32_t* d_keys,
               cudaStream_t st);

// Algorithm 2 lines 7 / 13 (k5_line13.cu)
int l13_global_rank(int num_maps, const MapDesc* d_maps, const uint32_t* d_facets, uint16_t* d_gidx,
                    cudaStream_t st);
int l13_remap(const uint32_t* d_rows, const uint16_t* d_map, long long count, int w32, const MapDesc* d_maps,
              const uint16_t* d_gidx, int kw, int rw, uint32_t* d_keys, int num_sms, cudaStream_t st);
size_t l13_select_temp_bytes(long long count);
int l13_unique(const uint32_t* d_sorted, long long count, int gw, uint8_t* d_flags, uint32_t* d_iota,
               uint32_t* d_uidx, int* d_num, void* d_temp, size_t temp_bytes, cudaStream_t st);
int l13_filter(const uint32_t* d_sorted, int gw, const uint32_t* d_uidx, const int* d_num, long long max_count,
               const uint16_t* d_unrank, int m, int maxf, uint8_t* d_keep, uint32_t* d_sidx, int* d_num13,
               void* d_temp, size_t temp_bytes, int num_sms, cudaStream_t st);
int l13_seed_flags(const uint16_t* d_masks, const long long* d_off, long long count, int m, int maxf,
                   uint8_t* d_flags, int num_sms, cudaStream_t st);
int l13_gather(const uint32_t* d_rows, int gw, const uint32_t* d_idx, long long count, uint32_t* d_out,
               cudaStream_t st);

// Algorithm 1 on the device (k6_odometer.cu): the reference's combination
// space, one map per OdoMap; vectors are Wb uint32 words (Wb =
// odo_words_bucket(W32), zero padded)
struct OdoMap {
    int32_t map, n, fs, cap;      // plan map id, facet size, fr stride, facet cap (INT32_MAX = none)
    int32_t nb, r, blk, pad;      // blocks (widest first), inner blocks (the last r), first block entry
    uint32_t fr_off, base_off;    // into fr (uint16); base vector into words
    uint32_t delta_off, step_off; // candidate / step vectors of the map's blocks into words
    long long outer, task0, inner;  // outer prefixes, first warp task, leaves per prefix
};
struct OdoParams {
    const OdoMap* maps;
    int num_maps;
    const int* blk_ncand;   // candidates per block
    const int* blk_first;   // first candidate of each block within its map
    const uint32_t* words;  // base / delta / step vectors
    const uint16_t* fr;
    unsigned long long* task_ctr;
    long long total_tasks;
    int cnt_words;          // ridge bitset words: ceil(max N / 32)
    uint32_t* out_keys;
    unsigned long long* out_ctl;  // [0] rows
    unsigned long long out_cap;
    int rw;
    unsigned long long* leaf_ctr;  // [0] leaves visited, [1] cap-passing leaves checked
};
int odo_max_inner();
int odo_words_bucket(int W32);
int launch_odometer(const OdoParams& p, int Wb, int num_sms, cudaStream_t st);

// Algorithm 2 line 15 (k7_line15.cu): canonical forms, one warp per
// complex; per-warp shared-memory layout (byte offsets) sized on the host
struct L15Layout {
    int m, n, kmax, mnfcap, P, seqcap, bmw, gw, mode;
    int o_fl, o_rm, o_fb, o_mb, o_mnf, o_keys, o_ids, o_seq, o_best, o_bnd, o_misc, bytes;
};
L15Layout l15_layout(int m, int n, int kmax, int mnfcap, int gw);
size_t l15_smem_bytes(const L15Layout& L);
// max facet count over rows (idx may be null)
int l15_max_facets(const uint32_t* d_rows, int gw, const uint32_t* d_idx, long long count, int* d_out,
                   cudaStream_t st);
// row mode (d_rows != null: complexes = rows[idx[i]], gw words, count from
// *d_num if given) or CSR mode (0-based masks ascending, offsets); d_ctl[4]:
// ticket, overflow count (> 0: rerun with a larger mnfcap), labelings, placements, cache hits;
// d_cache_key (cache_slots, a power of two; null = no cache) + d_cache_data
// (cache_slots * (kmax + 1) uint16): the canonical-form cache
int l15_launch(const L15Layout& L, const uint32_t* d_rows, const uint32_t* d_idx, const int* d_num,
               const uint16_t* d_unrank, const uint16_t* d_masks, const long long* d_off, long long count,
               uint32_t* d_out_rows, uint16_t* d_out_masks, int8_t* d_cls, unsigned long long* d_cost,
               unsigned long long* d_ctl, unsigned long long* d_cache_key, uint16_t* d_cache_data, int cache_slots,
               int num_sms, cudaStream_t st);
size_t l15_dedupe_temp_bytes(long long count, int gw);
int l15_dedupe(const uint32_t* d_rows, long long count, int gw, uint32_t* d_sidx, uint32_t* d_iota, uint8_t* d_first,
               uint32_t* d_rep, int* d_nrep, void* d_temp, size_t temp_bytes, cudaStream_t st);
int l15_gather(const uint32_t* d_rows, int gw, const uint32_t* d_idx, long long count, uint32_t* d_out,
               cudaStream_t st);

// verification of a result (k8_verify.cu): soundness of every row and, with
// reach, its coordinates in the reference basis
struct VerifyMap {
    int32_t M, N, n, cap, fs, W32;
    uint32_t fr_off;
    int32_t s;          // usable generators; -1 = no reachability data
    uint32_t gens_off;  // s * W32 words (words)
    uint32_t base_off;  // W32 words (words)
    uint32_t piv_off;   // s pivot facets (ints)
    uint32_t inv_off;   // s inverse columns (u64s)
    uint32_t blk_off;   // nblk induced-block generator masks (u64s)
    int32_t nblk;
};
struct VerifyParams {
    const VerifyMap* maps;
    const uint16_t* fr;
    const uint32_t* words;
    const int32_t* ints;
    const unsigned long long* u64s;
    const uint32_t* rows;
    const uint16_t* row_map;
    long long count;
    int w32, cnt_words, reach;
    unsigned long long* coords;  // optional, one per row
    uint8_t* flags;              // optional: bit 0 unsound, 1 outside the span, 2 > 2 generators in a block
    unsigned long long* ctl;     // [0..2] rows with flag bit 0 / 1 / 2
};
int launch_k8_verify(const VerifyParams& p, int num_sms, cudaStream_t st);

// INT32 lane-op issue peak (LOP3 + IADD3 chains over every SM), ops/s
int int_peak_measure(int device, double* ops_per_s);

}  // namespace wpm
