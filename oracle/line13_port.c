/*
 * oracle/line13_port.c -- TEST INFRASTRUCTURE ONLY (see plseeds_port.h).
 *
 * Plain-C restatement of Algorithm 2 lines 7 and 13 of the reference
 * pipeline (pipeline.hpp:58-89): the union of the per-orbit WPM lists as
 * labeled complexes, then the Picard (full support) and seedness filters.
 *
 *   po_minimal_nonfaces   <- minimal_nonfaces      complex.hpp:192-221
 *   po_wedge_witness      <- wedge_witness         classify.hpp:22-48
 *   po_is_seed            <- is_seed               classify.hpp:51-53
 *   po_line13             <- pipeline.hpp:58-89 (std::set union, :76-89 filters)
 *
 * po_is_seed restates the reference literally (face set, minimal non-faces,
 * edges, witness scan).  po_is_seed_swap is the characterisation the device
 * filter uses (an edge {u,v} is a witness iff every facet meets {u,v} and the
 * transposition (u v) maps facets to facets -- see DESIGN.md); the tests
 * check the two agree, and against the reference's own is_seed
 * (oracle/_ref/plseeds_ref seed).
 */
#include <stdlib.h>
#include <string.h>

#include "plseeds_port.h"

static int popc64(uint64_t x) { return __builtin_popcountll(x); }
static int ctz64(uint64_t x) { return __builtin_ctzll(x); }

/* face set of a complex on [m] as a bitmap over masks >> 1 (bit 0 unused) */
static uint8_t *face_bitmap(int m, const uint64_t *facets, int k) {
    uint8_t *face = (uint8_t *)calloc((size_t)1 << m, 1);
    if (!face) return NULL;
    for (int i = 0; i < k; ++i) {
        /* complex.hpp:176-185: every subset of every facet */
        const uint64_t f = facets[i];
        uint64_t sub = f;
        for (;;) {
            face[sub >> 1] = 1;
            if (sub == 0) break;
            sub = (sub - 1) & f;
        }
    }
    return face;
}

int po_minimal_nonfaces(int m, const uint64_t *facets, int k, uint64_t *out, int cap) {
    if (m < 1 || m > 20) return -PO_EINVAL;
    uint8_t *face = face_bitmap(m, facets, k);
    if (!face) return -PO_ENOMEM;
    const size_t sz = (size_t)1 << m;
    uint8_t *cand = (uint8_t *)calloc(sz, 1);
    if (!cand) {
        free(face);
        return -PO_ENOMEM;
    }
    const uint64_t full = (((uint64_t)1 << m) - 1) << 1;
    face[0] = 0; /* complex.hpp:195: the empty face stays implicit */
    /* :199-202 ghost vertices give singleton non-faces */
    for (int v = 1; v <= m; ++v)
        if (!face[((uint64_t)1 << v) >> 1]) cand[((uint64_t)1 << v) >> 1] = 1;
    /* :203-208 extend every face by one vertex */
    for (size_t s = 1; s < sz; ++s) {
        if (!face[s]) continue;
        const uint64_t f = (uint64_t)s << 1;
        for (uint64_t r = full & ~f; r; r &= r - 1) {
            const uint64_t ext = f | (r & (0 - r));
            if (!face[ext >> 1]) cand[ext >> 1] = 1;
        }
    }
    /* :210-217 keep the inclusion-minimal ones; :218 canonical (ascending) order */
    int cnt = 0;
    for (size_t s = 1; s < sz; ++s) {
        if (!cand[s]) continue;
        const uint64_t c = (uint64_t)s << 1;
        int minimal = 1;
        for (uint64_t r = c; r; r &= r - 1) {
            /* the empty set is not in face_set (faces_by_card erases it,
             * complex.hpp:185), so a singleton candidate is never minimal */
            const uint64_t sub = c & ~(r & (0 - r));
            if (!sub || !face[sub >> 1]) minimal = 0;
        }
        if (minimal) {
            if (cnt < cap) out[cnt] = c;
            ++cnt;
        }
    }
    free(face);
    free(cand);
    return cnt;
}

static int cmp_u64(const void *a, const void *b) {
    const uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

int po_wedge_witness(const uint64_t *facets, int k, const uint64_t *mnfs, int nm, int *u_out, int *v_out) {
    /* classify.hpp:24-35: the edges of K, canonical order */
    uint64_t *edges = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(k * 120 + 1));
    if (!edges) return -PO_ENOMEM;
    int ne = 0;
    for (int i = 0; i < k; ++i)
        for (uint64_t a = facets[i]; a; a &= a - 1)
            for (uint64_t b = a & (a - 1); b; b &= b - 1) edges[ne++] = (a & (0 - a)) | (b & (0 - b));
    qsort(edges, (size_t)ne, sizeof(uint64_t), cmp_u64);
    int w = 0;
    for (int i = 0; i < ne; ++i)
        if (i == 0 || edges[i] != edges[i - 1]) edges[w++] = edges[i];
    ne = w;
    /* :36-46 the first edge no minimal non-face meets in exactly one vertex */
    for (int i = 0; i < ne; ++i) {
        int witness = 1;
        for (int j = 0; j < nm && witness; ++j)
            if (popc64(edges[i] & mnfs[j]) == 1) witness = 0;
        if (witness) {
            if (u_out) *u_out = ctz64(edges[i]);
            if (v_out) *v_out = ctz64(edges[i] & (edges[i] - 1));
            free(edges);
            return 1;
        }
    }
    free(edges);
    return 0;
}

int po_is_seed(int m, const uint64_t *facets, int k) {
    const int cap = 1 << 16;
    uint64_t *mnfs = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)cap);
    if (!mnfs) return -PO_ENOMEM;
    const int nm = po_minimal_nonfaces(m, facets, k, mnfs, cap);
    if (nm < 0 || nm > cap) {
        free(mnfs);
        return -PO_EINVAL;
    }
    const int w = po_wedge_witness(facets, k, mnfs, nm, NULL, NULL);
    free(mnfs);
    return w < 0 ? w : !w;
}

/* the device filter's characterisation: pure complex, facets ascending */
static int has_facet(const uint64_t *facets, int k, uint64_t f) {
    int lo = 0, hi = k - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (facets[mid] == f) return 1;
        if (facets[mid] < f) lo = mid + 1;
        else hi = mid - 1;
    }
    return 0;
}

int po_is_seed_swap(int m, const uint64_t *facets, int k) {
    for (int u = 1; u <= m; ++u)
        for (int v = u + 1; v <= m; ++v) {
            const uint64_t e = ((uint64_t)1 << u) | ((uint64_t)1 << v);
            int edge = 0, witness = 1;
            for (int i = 0; i < k && witness; ++i) {
                const uint64_t hit = facets[i] & e;
                if (!hit) witness = 0;
                else if (hit == e) edge = 1;
                else if (!has_facet(facets, k, facets[i] ^ e)) witness = 0;
            }
            if (witness && edge) return 0;
        }
    return 1;
}

/* ---- pipeline.hpp:58-89 over complexes given as bitsets over the
 * all-subsets universe of (m, n) (catalog.hpp:112-120, ascending masks) */
static int g_words;
static int cmp_rows(const void *a, const void *b) {
    return po_bits_cmp((const uint64_t *)a, (const uint64_t *)b, g_words);
}

int64_t po_line13(int m, int n, int words, const uint64_t *rows, int64_t count, int literal, int64_t *line7_out,
                  uint64_t *survivors_out, int64_t *line7_rows_count) {
    uint64_t uni[4096];
    const int U = po_all_subsets_universe(m, n, uni, 4096);
    if (U < 0 || U > words * 64) return -PO_EINVAL;
    uint64_t *all = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(count * words + 1));
    uint64_t *facets = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(U + 1));
    if (!all || !facets) {
        free(all);
        free(facets);
        return -PO_ENOMEM;
    }
    memcpy(all, rows, sizeof(uint64_t) * (size_t)(count * words));
    /* :58-70 std::set<std::vector<VertexSet>> labeled: sorted, unique */
    g_words = words;
    qsort(all, (size_t)count, sizeof(uint64_t) * (size_t)words, cmp_rows);
    int64_t u = 0;
    for (int64_t i = 0; i < count; ++i)
        if (i == 0 || memcmp(all + i * words, all + (u - 1) * words, sizeof(uint64_t) * (size_t)words)) {
            if (u != i) memcpy(all + u * words, all + i * words, sizeof(uint64_t) * (size_t)words);
            ++u;
        }
    *line7_out = u;
    if (line7_rows_count) *line7_rows_count = u;
    /* :76-89 keep full support and seeds, in the labeled set's order */
    const uint64_t full = (((uint64_t)1 << m) - 1) << 1;
    int64_t kept = 0;
    for (int64_t i = 0; i < u; ++i) {
        const uint64_t *K = all + i * words;
        int k = 0;
        uint64_t sup = 0;
        for (int w = 0; w < words; ++w)
            for (uint64_t x = K[w]; x; x &= x - 1) {
                facets[k] = uni[w * 64 + ctz64(x)];
                sup |= facets[k++];
            }
        if (sup != full) continue;
        const int s = literal ? po_is_seed(m, facets, k) : po_is_seed_swap(m, facets, k);
        if (s < 0) {
            free(all);
            free(facets);
            return s;
        }
        if (!s) continue;
        if (survivors_out) memcpy(survivors_out + kept * words, K, sizeof(uint64_t) * (size_t)words);
        ++kept;
    }
    free(all);
    free(facets);
    return kept;
}
