/*
 * oracle/dfs_port.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Single-threaded CPU restatement of the product's ridge-driven backtracking
 * search (paper_2301_00806_b200/csrc/dfs.cu), used by the tests as the
 * node-count reference for the GPU kernel and as a second, independent
 * oracle for the output set.  It is not the reference's algorithm (that is
 * plseeds_port.c, restating search.hpp:141-258); both define the same output
 * set -- every nonempty weak pseudo-manifold K inside the universe with
 * |K| <= cap (search.hpp:135-140) -- which the tests check against each other.
 */
#ifndef DFS_PORT_H
#define DFS_PORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t count;     /* WPMs found */
    int words;
    uint64_t *bits;    /* count * words, canonical order */
    int64_t nodes;     /* facet-inclusion steps (the DFS "search node") */
} dfs_result;

/* facets: canonical universe; cap < 0: no cap.  required/forbidden: facet
 * indices pinned in/out before the search (apply_link_constraints
 * semantics, kernel_basis.hpp:248-321).  want_bits = 0 counts only.
 * root_lo/root_hi restrict the root branches ("minimum facet" in
 * [root_lo, root_hi)); pass 0, M for the whole search.
 * Returns 0, or 2 on a malformed universe. */
int dfs_enumerate(int n, const uint64_t *facets, int M, int64_t cap, const int32_t *required,
                  int nreq, const int32_t *forbidden, int nforb, int want_bits, int root_lo,
                  int root_hi, dfs_result *out);
int dfs_enumerate_shard(int n, const uint64_t *facets, int M, int64_t cap, int want_bits,
                        int shard_index, int shard_count, dfs_result *out);
void dfs_result_free(dfs_result *r);

#ifdef __cplusplus
}
#endif
#endif
