/*
 * wpm_b200.h -- C-ABI of the B200-native weak-pseudo-manifold enumerator.
 *
 * The drop-in boundary for the reference's enumeration path
 * ("characteristic map in, WPM facet lists out").  Plain pointers and sizes,
 * no torch or CUDA types.  Every entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj):
 *
 *   wpm_idcm_orbits         <- idcm_orbits(n, p)            include/plseeds/charmap.hpp:212-281
 *   wpm_charmap_of_dcm      <- charmap_of_dcm(d)            include/plseeds/charmap.hpp:155-204
 *   wpm_cyclic_facet_bound  <- cyclic_facet_bound(n)        include/plseeds/affine_property.hpp:35-45
 *   wpm_plan_create_orbits  <- the per-orbit loop prelude   include/plseeds/pipeline.hpp:54-66
 *                              matroid_universe (pipeline.hpp:33-35) = binary_matroid
 *                              (charmap.hpp:117-141) on the GPU (kernel 1), then
 *                              incidence_matrix (incidence.hpp:34-55) on the GPU (kernel 2)
 *   wpm_plan_create_universes <- SearchJob{m, n, facets, properties} (search.hpp:46-55)
 *                              + incidence_matrix (kernel 2); required/forbidden facet
 *                              pins replace apply_link_constraints (kernel_basis.hpp:248-321)
 *   wpm_plan_run            <- enumerate_wpm(const SearchJob&)  search.hpp:141-258 (kernel 3,
 *                              the ridge-driven DFS) + the canonical merge/sort (:247-257)
 *   wpm_plan_fetch / wpm_result_*  <- std::vector<PureComplex> return value (search.hpp:141)
 *   wpm_enumerate           <- enumerate_wpm(job) one-shot     search.hpp:141-258 (job.progress,
 *                              job.threads -> devices: wpm_job_t.progress / .devices)
 *   wpm_plan_set_devices ... wpm_plan_run_claim <- parallel_for_index (parallel.hpp:27-54) across GPUs
 *   wpm_write_cplx          <- write_complexes(os, list)       include/plseeds/complex_io.hpp:21-39
 *   wpm_plan_run_kernel_basis <- enumerate_wpm's own algorithm (kernel basis + combination-space
 *                              odometer, search.hpp:141-258) with every leaf on the GPU
 *   wpm_plan_run_kernel_basis_prefix <- the per-item odometer (search.hpp:204-243) of one outer prefix
 *   wpm_plan_verify         <- is_weak_pseudomanifold_direct (complex.hpp:224-233) on every row, plus
 *                              coordinates in the reference basis (test_gf2.cpp:15-50 style)
 *   wpm_plan_line13         <- Algorithm 2 lines 7 and 13      include/plseeds/pipeline.hpp:58-89
 *                              (std::set union of the per-orbit lists; support == full(m),
 *                              complex.hpp:64-70; is_seed, classify.hpp:51-53)
 *   wpm_seed_flags          <- is_seed(K) / K.support() over a batch (classify.hpp:22-53,
 *                              complex.hpp:192-221)
 *   wpm_pipeline_line13     <- pipeline(n, db) lines 1-13     include/plseeds/pipeline.hpp:52-89
 *   wpm_plan_line15         <- Algorithm 2 line 15             include/plseeds/pipeline.hpp:91-103
 *                              (canonical_form, isomorphism.hpp:228-303, + first-appearance dedupe)
 *   wpm_canonical_forms     <- canonical_form(K) / detail::refine_classes over a batch
 *                              (isomorphism.hpp:162-303)
 *   wpm_pipeline_line15     <- pipeline(n, db) lines 1-15     include/plseeds/pipeline.hpp:52-103
 *
 * Status codes mirror the CLI exit codes (tools/plseeds_cli.cpp:31-35):
 * 0 ok, 2 format/purity/invalid argument, 3 infeasible, 5 cap exceeded,
 * 1 internal / CUDA error (wpm_last_error() has the message).  There is no
 * CPU fallback: without a usable B200 every compute entry point returns 1.
 *
 * Threading: calls block (like enumerate_wpm); distinct plans may be used
 * from distinct host threads; one plan is not re-entrant.
 */
#ifndef WPM_B200_H
#define WPM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WPM_OK 0
#define WPM_EINTERNAL 1
#define WPM_EINVAL 2
#define WPM_EINFEASIBLE 3
#define WPM_ECAP 5

/* facet_cap sentinels */
#define WPM_CAP_NONE (-1)  /* no property: every WPM (classify_full_universe, pipeline.hpp:157-196) */
#define WPM_CAP_UBT (-2)   /* ubt_property(n, M): |K| <= cyclic_facet_bound(n) (affine_property.hpp:49-54) */

/* hard limits of the device layout */
#define WPM_MAX_M 16       /* vertex labels 1..m (VertexSet bits 1..16) */
#define WPM_MAX_FACETS 2048
#define WPM_MAX_RIDGES 4096
#define WPM_MAX_PARENTS 8  /* candidate facets per ridge (m - n + 1 <= 8) */

typedef struct wpm_plan wpm_plan_t;

/* one enumeration job over a single facet universe (SearchJob, search.hpp:46-55) */
typedef struct {
    int32_t m, n;
    int32_t num_facets;          /* M */
    const uint64_t *facets;      /* M masks, bit v = vertex v (1-based), strictly ascending */
    int64_t facet_cap;           /* >= 0, WPM_CAP_NONE or WPM_CAP_UBT */
    const int32_t *required;     /* facet indices pinned into every K */
    int32_t num_required;
    const int32_t *forbidden;    /* facet indices pinned out of every K */
    int32_t num_forbidden;
    int32_t device;              /* CUDA ordinal */
    int32_t shard_index;         /* static root-task partition (a rank's share without a shared */
    int32_t shard_count;         /* frontier): root tasks t with t % count == index (0/1 = all) */
    /* SearchJob::progress (search.hpp:54, called per outer item :244): called
     * from the calling thread while the search runs with (root tasks
     * finished, root tasks), monotone, the last call done == total; NULL = none */
    void (*progress)(int64_t done, int64_t total, void *user);
    void *progress_user;
    /* SearchJob::threads (search.hpp:52) becomes GPUs: devices[0..num_devices)
     * run one job (num_devices <= 1: `device` alone) -- the tree is split
     * below the root and every GPU claims frontier records through one shared
     * counter (wpm_plan_set_devices) */
    const int32_t *devices;
    int32_t num_devices;
} wpm_job_t;

/* enumeration output: WPMs of every map of the plan, grouped by map, each
 * group in canonical order (search.hpp:254-256), as characteristic bitsets
 * over that map's universe (bit j = facet j), `words` uint64 per WPM. */
typedef struct {
    int32_t num_maps;
    int32_t words;
    int64_t total;               /* number of WPMs over all maps */
    int64_t *counts;             /* num_maps */
    int64_t *offsets;            /* num_maps + 1, prefix sums of counts */
    uint64_t *bits;              /* total * words */
    int64_t nodes;               /* DFS search nodes (facet-inclusion steps) */
    int64_t duplicates;          /* adjacent equal WPMs after the sort; always 0 */
    double ms_search;            /* device time of kernel 3 (CUDA events) */
    double ms_sort;              /* device time of the canonical sort + gather */
    int64_t tasks;               /* work items processed (root tasks + donations) */
    double ms_total;             /* device time of the whole run (first to last op on the plan stream) */
    int64_t h2d_bytes;           /* host->device bytes of the create + run + fetch that produced this */
    int64_t d2h_bytes;           /* device->host bytes (result included) */
} wpm_result_t;

/* labeled complexes on [m] with facets of size n (PureComplex, complex.hpp:23-55),
 * in the canonical order of std::set<std::vector<VertexSet>> (pipeline.hpp:58). */
typedef struct {
    int32_t m, n;
    int64_t count;
    int64_t *offsets;            /* count + 1 */
    uint64_t *facets;            /* offsets[count] masks (bit v = vertex v), ascending per complex */
    int32_t words;               /* uint64 words per complex in `bits` */
    uint64_t *bits;              /* count * words: characteristic bitsets over ALL n-subsets of [m]
                                    in ascending mask order (catalog.hpp:112-120) */
    int64_t line7, line13;       /* Algorithm 2 line counts of the run that produced the list */
    double ms_union, ms_filter;  /* device time of the union (line 7) and the filters (line 13) */
    int64_t h2d_bytes, d2h_bytes;
    int64_t line15;              /* Algorithm 2 line 15 count (-1 before wpm_plan_line15) */
    double ms_canon, ms_dedupe;  /* device time of the canonical forms and of the class dedupe */
} wpm_complexes_t;

/* ---------------------------------------------------------------- host */
const char *wpm_last_error(void);
int wpm_device_count(void);
int64_t wpm_cyclic_facet_bound(int32_t n);
/* rows_out: up to cap orbits x (n+p) rows; returns #orbits or -status */
int32_t wpm_idcm_orbits(int32_t n, int32_t p, uint32_t *rows_out, int32_t cap);
/* cols_out: m columns; returns n or -status */
int32_t wpm_charmap_of_dcm(int32_t m, int32_t p, const uint32_t *rows, uint32_t *cols_out);

/* ---------------------------------------------------------------- plans */
/* Every characteristic map of idcm_orbits(n, p): universes by kernel 1 and
 * incidence tables by kernel 2, resident on `device`. */
int wpm_plan_create_orbits(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_plan_t **out);
/* Explicit characteristic maps: num_maps x m lambda columns (n-bit each). */
int wpm_plan_create_charmaps(int32_t n, int32_t m, int32_t num_maps, const uint32_t *cols,
                             int64_t facet_cap, int32_t device, wpm_plan_t **out);
/* Explicit universes (SearchJob.facets), one per map; facet_counts[i] masks
 * each, concatenated in `facets`, in any order (like the reference's
 * incidence_matrix, incidence.hpp:34-55): the plan keeps each universe in
 * canonical (ascending) order -- results and wpm_plan_universe index that
 * order; required/forbidden index the caller's order and apply to map 0 only
 * (pass num_maps == 1 with pins).  Duplicate facets -> 2. */
int wpm_plan_create_universes(int32_t m, int32_t n, int32_t num_maps, const int32_t *facet_counts,
                              const uint64_t *facets, int64_t facet_cap, const int32_t *required,
                              int32_t num_required, const int32_t *forbidden, int32_t num_forbidden,
                              int32_t device, wpm_plan_t **out);
int wpm_plan_num_maps(const wpm_plan_t *plan);
/* kernel-1 / kernel-2 outputs of one map (parity hooks) */
int32_t wpm_plan_universe(wpm_plan_t *plan, int32_t map, uint64_t *facets_out, int32_t cap);
int32_t wpm_plan_incidence(wpm_plan_t *plan, int32_t map, uint64_t *ridges_out, int32_t ridges_cap,
                           int32_t *cols_out, int32_t *par_out /* N*WPM_MAX_PARENTS, -1 padded */);
/* Run the search + canonical sort on the device; results stay resident.
 * Returns status; *total_out = number of WPMs. */
int wpm_plan_run(wpm_plan_t *plan, int32_t shard_index, int32_t shard_count, int64_t *total_out);
/* Search-node budget of the following runs (0 = none, the default).  A run
 * that reaches it stops early: its rows are valid WPMs but not all of them,
 * and wpm_plan_truncated() returns 1 -- for throughput / divergence stress on
 * universes whose full enumeration is out of reach (BASELINE configs[4]). */
int wpm_plan_set_node_budget(wpm_plan_t *plan, int64_t budget);
int wpm_plan_truncated(const wpm_plan_t *plan);
/* Copy the last run's results to the host. */
int wpm_plan_fetch(wpm_plan_t *plan, wpm_result_t **out);
/* Device-side timing of the last run (ms) and node count, without a fetch. */
int wpm_plan_stats(const wpm_plan_t *plan, double *ms_search, double *ms_sort, int64_t *nodes,
                   int64_t *tasks);
/* ms_total of the last run, and the kernel-3 launch geometry (warps). */
int wpm_plan_timing(const wpm_plan_t *plan, double *ms_total, int32_t *warps);
/* Resident result of the last run: device pointers (uint32 words, 2 per
 * uint64 word; uint16 map ids) in canonical order, valid until the next run. */
int wpm_plan_device_result(const wpm_plan_t *plan, const uint32_t **bits32, const uint16_t **map_ids,
                           int64_t *count, int32_t *words32);

/* ---------------------------------------------------------------- multi-GPU
 * One job on several GPUs of one process (SearchJob::threads ->
 * parallel_for_index, parallel.hpp:27-54, becomes GPUs): devices[0] must be
 * the plan's device; the others get plans of the same maps.  wpm_plan_run
 * then splits the search tree below the root, every GPU its share of the
 * root tasks in parallel (split rounds until the frontiers hold >= 640
 * records per GPU), copies the concatenated frontier to every GPU, and each
 * GPU's kernel 3 pulls records through one claim counter
 * in devices[0]'s HBM (peer atomics over NVLink) and shares them further by
 * donation; the rows are gathered into devices[0] (peer copies) and sorted
 * canonically there.  No GPU waits for another.  ndev <= 1 detaches. */
int wpm_plan_set_devices(wpm_plan_t *plan, const int32_t *devices, int32_t ndev);
int wpm_plan_create_orbits_multi(int32_t n, int32_t p, int64_t facet_cap, const int32_t *devices, int32_t ndev,
                                 wpm_plan_t **out);
/* per device of the last multi-GPU run: kernel-3 ms and search nodes; returns the device count */
int wpm_plan_device_stats(const wpm_plan_t *plan, int32_t cap, double *ms_out, int64_t *nodes_out);
/* split below the root before the search: first split depth (branch frames;
 * 0 = off for single-GPU runs, multi-GPU runs default to 3) */
int wpm_plan_set_split(wpm_plan_t *plan, int32_t depth);
/* per-root search nodes of the following runs (root tasks, or frontier
 * records after a split): wpm_plan_root_nodes returns the root count, writes
 * at most cap counts and the split phase's own nodes (*split_nodes) -- the
 * measured input of the multi-GPU scaling projection */
int wpm_plan_set_root_stats(wpm_plan_t *plan, int32_t on);
int64_t wpm_plan_root_nodes(wpm_plan_t *plan, int64_t *out, int64_t cap, int64_t *split_nodes);
/* progress callback of the following runs (see wpm_job_t.progress); NULL = off */
int wpm_plan_set_progress(wpm_plan_t *plan, void (*fn)(int64_t done, int64_t total, void *user), void *user);
/* The same protocol across processes (one per GPU): every rank r calls
 * wpm_plan_split(plan, r, world, ...) on its share of the root tasks (rows and
 * nodes above its frontier stay in its plan); the frontiers
 * (wpm_plan_frontier: a device pointer, count x recw uint32) are all-gathered
 * and every rank wpm_plan_load_frontier-s the concatenation (not aliasing its
 * own frontier buffer).  A claim counter made by rank 0
 * (wpm_claim_counter_create, 64-byte CUDA IPC handle) is opened by the others
 * (wpm_claim_counter_open); every rank then wpm_plan_run_claim-s and the
 * canonical rows are gathered to rank 0 (wpm_canonical_sort_device there). */
/* depth <= 0: 5 + ceil(log_1.7(shard_count)), then calibrated from the last
 * split of the same workload (one round per shard, usually);
 * target <= 0: 2048 records */
int wpm_plan_split(wpm_plan_t *plan, int32_t shard_index, int32_t shard_count, int32_t depth, int64_t target,
                   int64_t *count);
int wpm_plan_frontier(const wpm_plan_t *plan, const uint32_t **recs, int64_t *count, int32_t *recw);
int wpm_plan_load_frontier(wpm_plan_t *plan, const uint32_t *recs, int64_t count);
int wpm_claim_counter_create(int32_t device, void **counter, uint8_t *ipc_handle /* 64 bytes, optional */);
int wpm_claim_counter_open(int32_t device, const uint8_t *ipc_handle, void **counter);
int wpm_claim_counter_reset(int32_t device, void *counter);
int wpm_claim_counter_close(int32_t device, void *counter, int32_t opened);
int wpm_plan_run_claim(wpm_plan_t *plan, void *counter, int64_t *total_out);

/* Canonical sort of rows that already live on `device` (e.g. shards gathered
 * over NCCL): orders (map id, canonical WPM order) into out_bits/out_map and
 * returns the number of adjacent duplicates in *dups.  Plain device pointers;
 * stream = a cudaStream_t passed as void* (NULL = legacy default stream). */
int wpm_canonical_sort_device(int32_t device, const uint32_t *bits32, const uint16_t *map_ids, int64_t count,
                              int32_t words32, uint32_t *out_bits32, uint16_t *out_map, int64_t *dups,
                              void *stream);

/* Measured INT32 lane-op peak of `device` (LOP3/IADD3 issue, all SMs), ops/s:
 * the roofline denominator of the integer-issue-bound search. */
int wpm_int_peak(int32_t device, double *ops_per_s);
/* Algorithm 1 exactly as the reference runs it (search.hpp:141-258): the
 * reference's kernel basis per map on the host (gf2_kernel bitmatrix.hpp:125-153,
 * convenient_basis kernel_basis.hpp:198-235, pins via apply_link_constraints
 * :248-321), then EVERY leaf of its combination space (search.hpp:62-104) on
 * the device: XOR of the block deltas, count cap, wpm_counts_ok (:114-131).
 * Same output set and result layout as wpm_plan_run; a space larger than
 * candidate_cap returns 5 (cap_exceeded_error, search.hpp:147-150). */
int wpm_plan_run_kernel_basis(wpm_plan_t *plan, uint64_t candidate_cap, int64_t *total_out);
/* leaves visited (= the sum of the combination-space sizes), leaves inside the
 * cap that went through wpm_counts_ok, host basis time, device leaf time */
int wpm_plan_kernel_basis_stats(const wpm_plan_t *plan, int64_t *leaves, int64_t *checked, double *ms_prep,
                                double *ms_leaves);
/* combination_space(basis).size_saturated(), kernel dimension s and induced
 * blocks of map `map` (after wpm_plan_run_kernel_basis) */
int wpm_plan_combination_space(const wpm_plan_t *plan, int32_t map, uint64_t *space, int32_t *s, int32_t *blocks);
/* Algorithm 1 over ONE map with the first nfixed blocks of its combination
 * space (widest first, search.hpp:168-170) fixed to candidates
 * cand[0..nfixed) (0 = none, 1..w = single generator, then the pairs, the
 * order of search.hpp:88-93): the reference's inner odometer over the
 * remaining blocks.  The result (same layout as wpm_plan_run; other maps
 * empty) is every reference-reachable WPM whose coordinates start with that
 * prefix -- the two-sided completeness check of SURVEY 8(c)(3). */
int wpm_plan_run_kernel_basis_prefix(wpm_plan_t *plan, int32_t map, int32_t nfixed, const int32_t *cand,
                                     uint64_t candidate_cap, int64_t *total_out);
/* widths of map `map`'s combination-space blocks, widest first (1 = free
 * singleton; block b owns usable generators [sum of widths before b, + w));
 * returns the block count (writes at most cap) or -status */
int32_t wpm_plan_space_blocks(wpm_plan_t *plan, int32_t map, int32_t *widths, int32_t cap);
/* Device verification of the last run (kernel 8): *unsound = rows that fail
 * the direct WPM test (complex.hpp:224-233: every ridge in 0 or 2 facets),
 * are empty, leave the universe or exceed the cap.  With reach != 0 also
 * *unreachable = rows whose coordinates in the reference's convenient basis
 * (kernel_basis.hpp:84-235) do not exist or use > 2 generators of an induced
 * block -- rows enumerate_wpm could not produce; coords_out
 * (optional, one per row, canonical order) receives the coordinates, bit g =
 * usable generator g in block order.  Needs <= 64 usable generators. */
int wpm_plan_verify(wpm_plan_t *plan, int32_t reach, int64_t *unsound, int64_t *unreachable, uint64_t *coords_out);
/* Algorithm 2 lines 7 and 13 on the last run's results (pipeline.hpp:58-89),
 * on the device: the union of every map's WPMs as labeled complexes (line 7,
 * exact duplicates across maps removed), then full support and is_seed
 * (line 13).  Needs C(m, n) <= 2048 (every Picard-4 n).  Results stay
 * resident until the next run. */
int wpm_plan_line13(wpm_plan_t *plan, int64_t *line7, int64_t *line13);
int wpm_plan_line13_timing(const wpm_plan_t *plan, double *ms_union, double *ms_filter);
/* Algorithm 2 line 15 on the last line-13 result (pipeline.hpp:91-103), on
 * the device: canonical_form (isomorphism.hpp:228-303) of every survivor,
 * then one representative per isomorphism class in order of first
 * appearance.  Needs m <= 15, n <= 11.  *line15 = number of classes. */
int wpm_plan_line15(wpm_plan_t *plan, int64_t *line15);
/* device ms of the canonical forms and the dedupe; labelings completed and
 * single-vertex placements of the canonical-labeling searches; kernel
 * launches (> 1: a complex had more minimal non-faces than the first sizing);
 * survivors whose canonical form was confirmed from the isomorphism cache */
int wpm_plan_line15_stats(const wpm_plan_t *plan, double *ms_canon, double *ms_dedupe, int64_t *labelings,
                          int64_t *placements, int32_t *launches, int64_t *cache_hits);
/* diagnostics: single-vertex placements of each survivor's canonical-labeling
 * search (survivor order), at most cap entries; returns the survivor count */
int64_t wpm_plan_line15_costs(wpm_plan_t *plan, int64_t *out, int64_t cap);
/* which = 7: the union; which = 13: the survivors of the filters (canonical
 * order); which = 14: the canonical form of every line-13 survivor, in
 * survivor order (the `canon` vector of pipeline.hpp:93-96); which = 15: the
 * line-15 representatives (canonical forms) in order of first appearance */
int wpm_plan_fetch_complexes(wpm_plan_t *plan, int32_t which, wpm_complexes_t **out);
void wpm_complexes_free(wpm_complexes_t *list);
/* write_complexes (complex_io.hpp:34-39) of a list; returns bytes needed */
int64_t wpm_write_complexes(const wpm_complexes_t *list, char *buf, int64_t buf_len);
/* Batch of pure complexes (CSR facet masks, any facet order): flags_out[i]
 * bit 0 = is_seed(K) (classify.hpp:51), bit 1 = K.support() == full(m).
 * Validates like PureComplex (complex.hpp:37-55): labels in 1..m, every
 * facet of size n, no duplicates -> 2.  m <= 16, <= WPM_MAX_FACETS facets. */
int wpm_seed_flags(int32_t m, int32_t n, int64_t count, const int64_t *offsets, const uint64_t *facets,
                   int32_t device, uint8_t *flags_out);
/* Batch canonical_form (isomorphism.hpp:228-303) of pure complexes (CSR facet
 * masks, any order; validated like wpm_seed_flags): canon_out receives each
 * complex's canonical facet masks, ascending, at the same offsets;
 * classes_out (optional, count * m) the refined class of every vertex
 * (detail::refine_classes, isomorphism.hpp:162-218).  m <= 15, n <= 11. */
int wpm_canonical_forms(int32_t m, int32_t n, int64_t count, const int64_t *offsets, const uint64_t *facets,
                        int32_t device, uint64_t *canon_out, int8_t *classes_out);
void wpm_plan_destroy(wpm_plan_t *plan);

/* ---------------------------------------------------------------- one-shot */
int wpm_enumerate(const wpm_job_t *job, wpm_result_t **out);
/* Algorithm-2 loop for one n: every orbit map, UBT (or given) cap. */
int wpm_enumerate_orbits(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_result_t **out);
void wpm_result_free(wpm_result_t *res);
/* Algorithm 2 lines 1-13 for one n (pipeline.hpp:52-89): orbits, search,
 * union, filters; the line-13 survivors with both line counts. */
int wpm_pipeline_line13(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_complexes_t **out);
/* Algorithm 2 lines 1-15 for one n (pipeline.hpp:52-103): lines 1-13, then
 * the canonical forms and the first-appearance class representatives
 * (line 15); the list holds the representatives and the line 7/13/15 counts. */
int wpm_pipeline_line15(int32_t n, int32_t p, int64_t facet_cap, int32_t device, wpm_complexes_t **out);

/* complex_io.hpp:21-39 for map `map` of a result; returns bytes needed,
 * writes at most buf_len. */
int64_t wpm_write_cplx(const wpm_result_t *res, int32_t map, int32_t m, int32_t n,
                       const uint64_t *universe, char *buf, int64_t buf_len);

#ifdef __cplusplus
}
#endif
#endif
