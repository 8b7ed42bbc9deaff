/*
 * oracle/plseeds_port.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference (`plseeds`, /root/reference/proj) for
 * the WPM-enumeration hot path.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library, and
 * only as the checker.  The product path (paper_2301_00806_b200/) never links
 * it: there is no CPU fallback.
 *
 * Every function cites the reference file:line it restates.  Facets, ridges
 * and vertex sets use the reference's encoding (vertex_set.hpp:20-68): a
 * uint64 mask, bit v = vertex v, labels 1-based.
 *
 * Parity pinning: the restatement is checked against the compiled reference
 * (oracle/_ref, built by oracle/Makefile from the reference headers in place)
 * and against the golden counts/digests in SURVEY.md App. A/C
 * (tests/golden/).
 */
#ifndef PLSEEDS_PORT_H
#define PLSEEDS_PORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirror plseeds_cli.cpp:31-35 exit codes) */
#define PO_OK 0
#define PO_EINVAL 2      /* std::invalid_argument / purity_error */
#define PO_EINFEASIBLE 3 /* apply_link_constraints -> nullopt */
#define PO_ECAP 5        /* cap_exceeded_error */
#define PO_ENOMEM 1

/* charmap.hpp:212-281.  Writes up to `cap` representatives, each n+p rows
 * (identity rows appended), into rows_out[i*(n+p) ...].  Returns the number of
 * orbits or -PO_EINVAL. */
int po_idcm_orbits(int n, int p, uint32_t *rows_out, int cap);

/* charmap.hpp:155-204.  cols_out gets m columns of an n x m map (n = m - p).
 * Returns n, or -PO_EINVAL on a rank-deficient DCM. */
int po_charmap_of_dcm(int m, int p, const uint32_t *rows, uint32_t *cols_out);

/* charmap.hpp:117-141 + complex.hpp:31-35: facets of the binary matroid in
 * canonical (ascending bitmask) order.  Returns M or -PO_EINVAL (rank
 * deficient). */
int po_binary_matroid(int n, int m, const uint32_t *cols, uint64_t *facets_out, int cap);

/* catalog.hpp:112-120 */
int po_all_subsets_universe(int m, int n, uint64_t *facets_out, int cap);

/* affine_property.hpp:35-45 */
int64_t po_cyclic_facet_bound(int n);

/* incidence.hpp:34-55: N ridges (canonical order), cols[j*n+k] = k-th ridge
 * index of facet j (ascending), parents CSR.  Returns N or -PO_EINVAL. */
int po_incidence(const uint64_t *facets, int M, uint64_t *ridges_out, int ridges_cap,
                 int32_t *cols_out, int32_t *par_off_out, int32_t *par_out);

/* Result of an enumeration: `count` WPMs, each `words` uint64 words of a
 * characteristic vector over the universe, canonical order
 * (search.hpp:247-257). */
typedef struct {
    int64_t count;
    int words;
    uint64_t *bits;     /* count * words */
    uint64_t space;     /* combination_space size (search.hpp:70-78), saturated */
    int s;              /* kernel dimension */
    int nblocks;        /* induced blocks of the convenient basis */
} po_result;

/* The full reference path for one job (search.hpp:141-258 fed by
 * incidence.hpp:59 -> kernel_basis.hpp:198-235 [-> :248-321]):
 * facet_cap < 0 means no property; otherwise ubt-style count cap
 * (affine_property.hpp:27-31, search.hpp:181-187).  required/forbidden are
 * facet indices (apply_link_constraints).  candidate_cap mirrors
 * SearchJob::candidate_cap (search.hpp:53, :147-150).
 * Returns PO_OK, PO_EINVAL, PO_EINFEASIBLE or PO_ECAP. */
int po_enumerate_wpm(int m, int n, const uint64_t *facets, int M, int64_t facet_cap,
                     const int32_t *required, int nreq, const int32_t *forbidden, int nforb,
                     uint64_t candidate_cap, po_result *out);
void po_result_free(po_result *r);

/* acceptance.cpp:54-92: Gray-code brute force over all 2^M subsets. */
int64_t po_brute_force_count(const uint64_t *facets, int M, const int32_t *required, int nreq,
                             const int32_t *forbidden, int nforb, int64_t facet_cap);

/* complex.hpp:224-233 on a facet list (any order). 1 = WPM. */
int po_is_wpm_direct(const uint64_t *facets, int k);

/* complex_io.hpp:21-39: serialise `count` complexes given as bitsets over
 * `universe`.  Returns bytes needed; writes at most buf_len bytes. */
int64_t po_write_cplx(int m, int n, const uint64_t *universe, int M, const uint64_t *bits,
                      int64_t count, int words, char *buf, int64_t buf_len);

/* canonical complex order on bitsets (search.hpp:254-255): <0, 0, >0 */
int po_bits_cmp(const uint64_t *a, const uint64_t *b, int words);

/* ---- Algorithm 2 lines 7 and 13 (oracle/line13_port.c) */
/* complex.hpp:192-221: minimal non-faces of a complex on [m] (facet masks),
 * canonical order; returns the count (writes at most cap) or -status */
int po_minimal_nonfaces(int m, const uint64_t *facets, int k, uint64_t *out, int cap);
/* classify.hpp:22-48: 1 and the witness (u < v) if some edge meets no
 * minimal non-face in exactly one vertex, else 0 */
int po_wedge_witness(const uint64_t *facets, int k, const uint64_t *mnfs, int nm, int *u, int *v);
/* classify.hpp:51-53 (literal: face set -> minimal non-faces -> witness) */
int po_is_seed(int m, const uint64_t *facets, int k);
/* the same predicate by the swap characterisation (pure complex, facets
 * ascending): no edge {u,v} met by every facet with K = (u v) K */
int po_is_seed_swap(int m, const uint64_t *facets, int k);
/* pipeline.hpp:58-89 on `count` complexes given as bitsets (words uint64)
 * over po_all_subsets_universe(m, n): union (sort + unique, *line7_out),
 * then full support + is_seed (literal != 0: po_is_seed, else the swap
 * form).  Returns line13 and writes the survivors' rows in order. */
int64_t po_line13(int m, int n, int words, const uint64_t *rows, int64_t count, int literal, int64_t *line7_out,
                  uint64_t *survivors_out, int64_t *line7_rows_count);

/* line15_port.c -- Algorithm 2 line 15 (pipeline.hpp:91-103) */
/* isomorphism.hpp:17-24 as histograms: counts_out[v*16 + s] = #mnfs of size s containing v */
int po_color_sequences(int m, const uint64_t *mnfs, int nm, int *counts_out);
/* isomorphism.hpp:162-218: cls_out[v-1] = refined class of vertex v; returns the class count */
int po_refine_classes(int m, const uint64_t *facets, int k, int *cls_out);
/* isomorphism.hpp:228-303: the canonical relabeling's facets (ascending) into out;
 * returns k (or -status); *leaves_out = complete labelings visited */
int po_canonical_form(int m, const uint64_t *facets, int k, uint64_t *out, long long *leaves_out);

#ifdef __cplusplus
}
#endif
#endif
