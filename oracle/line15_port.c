/*
 * oracle/line15_port.c -- TEST INFRASTRUCTURE ONLY (see plseeds_port.h).
 *
 * Plain-C restatement of Algorithm 2 line 15 of the reference pipeline
 * (pipeline.hpp:91-103): one representative per isomorphism class, via
 * canonical forms, kept in order of first appearance.
 *
 *   po_color_sequences   <- color_sequences          isomorphism.hpp:17-24
 *   po_refine_classes    <- detail::refine_classes   isomorphism.hpp:162-218
 *   po_canonical_form    <- canonical_form           isomorphism.hpp:228-303
 *
 * Both are restated literally: the refinement keys are the reference's
 * variable-length integer vectors ([rank, -1, env entry, -1, env entry, ...]
 * with env entries [0, |S|, sorted ranks] per minimal non-face and
 * [1, sorted ranks] per facet), ranked by lexicographic order exactly as
 * ranks_of does; the canonical relabeling is the reference's class-by-class
 * permutation search with its prefix pruning at class boundaries.  The
 * device kernel (k7_line15.cu) computes the same result by other means
 * (order-preserving 64-bit entry codes, pruning at every placement); the
 * tests compare the two, and this file against oracle/_ref (the reference
 * itself: plseeds_ref classes / line15).
 */
#include <stdlib.h>
#include <string.h>

#include "plseeds_port.h"

typedef struct {
    long long *a;
    int len, cap;
} lvec;

static void lv_push(lvec *v, long long x) {
    if (v->len == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 16;
        v->a = (long long *)realloc(v->a, (size_t)v->cap * sizeof(long long));
    }
    v->a[v->len++] = x;
}

/* std::vector<long long> operator< : lexicographic, a proper prefix first */
static int lv_cmp(const lvec *x, const lvec *y) {
    const int n = x->len < y->len ? x->len : y->len;
    for (int i = 0; i < n; ++i)
        if (x->a[i] != y->a[i]) return x->a[i] < y->a[i] ? -1 : 1;
    return (x->len > y->len) - (x->len < y->len);
}

static int lv_cmp_q(const void *p, const void *q) { return lv_cmp((const lvec *)p, (const lvec *)q); }
static int ll_cmp_q(const void *p, const void *q) {
    const long long a = *(const long long *)p, b = *(const long long *)q;
    return (a > b) - (a < b);
}
static int u64_cmp_q(const void *p, const void *q) {
    const uint64_t a = *(const uint64_t *)p, b = *(const uint64_t *)q;
    return (a > b) - (a < b);
}

/* ranks_of (isomorphism.hpp:168-179): rank[v] = index of key[v] among the
 * sorted distinct keys of vertices 1..m. Returns the number of classes. */
static int ranks_of(int m, lvec *key, int *rank) {
    lvec *d = (lvec *)malloc((size_t)m * sizeof(lvec));
    memcpy(d, key + 1, (size_t)m * sizeof(lvec));
    qsort(d, (size_t)m, sizeof(lvec), lv_cmp_q);
    int nd = 0;
    for (int i = 0; i < m; ++i)
        if (nd == 0 || lv_cmp(&d[nd - 1], &d[i]) != 0) d[nd++] = d[i];
    for (int v = 1; v <= m; ++v) {
        int lo = 0, hi = nd; /* lower_bound */
        while (lo < hi) {
            const int mid = (lo + hi) / 2;
            if (lv_cmp(&d[mid], &key[v]) < 0) lo = mid + 1;
            else hi = mid;
        }
        rank[v] = lo;
    }
    rank[0] = nd;
    free(d);
    return nd;
}

static int popc64(uint64_t x) { return __builtin_popcountll(x); }

int po_color_sequences(int m, const uint64_t *mnfs, int nm, int *counts_out) {
    /* isomorphism.hpp:17-24 as per-vertex size histograms: counts_out[v*16+s] */
    memset(counts_out, 0, (size_t)(m + 1) * 16 * sizeof(int));
    for (int i = 0; i < nm; ++i)
        for (uint64_t r = mnfs[i]; r; r &= r - 1) counts_out[__builtin_ctzll(r) * 16 + popc64(mnfs[i])]++;
    return 0;
}

int po_refine_classes(int m, const uint64_t *facets, int k, int *cls_out) {
    if (m < 1 || m > 20) return -PO_EINVAL;
    uint64_t *mnfs = (uint64_t *)malloc(sizeof(uint64_t) << m);
    const int nm = po_minimal_nonfaces(m, facets, k, mnfs, 1 << m);
    if (nm < 0) {
        free(mnfs);
        return nm;
    }
    lvec *key = (lvec *)calloc((size_t)m + 1, sizeof(lvec));
    /* :166-169 key[v] = color sequence of v (sorted mnf sizes, :17-24) */
    for (int i = 0; i < nm; ++i)
        for (uint64_t r = mnfs[i]; r; r &= r - 1) lv_push(&key[__builtin_ctzll(r)], popc64(mnfs[i]));
    for (int v = 1; v <= m; ++v) qsort(key[v].a, (size_t)key[v].len, sizeof(long long), ll_cmp_q);
    int *rank = (int *)malloc((size_t)(m + 1) * sizeof(int));
    int *nrank = (int *)malloc((size_t)(m + 1) * sizeof(int));
    int classes = ranks_of(m, key, rank);
    int env_cap = nm + k;
    lvec *env = (lvec *)calloc((size_t)env_cap, sizeof(lvec));
    lvec *next = (lvec *)calloc((size_t)m + 1, sizeof(lvec));
    for (int round = 0; round < m; ++round) { /* :182-216 */
        for (int v = 1; v <= m; ++v) {
            const uint64_t vb = (uint64_t)1 << v;
            next[v].len = 0;
            lv_push(&next[v], rank[v]);
            int ne = 0;
            for (int i = 0; i < nm; ++i) {
                if (!(mnfs[i] & vb)) continue;
                lvec *e = &env[ne++];
                e->len = 0;
                lv_push(e, 0);
                lv_push(e, popc64(mnfs[i]));
                for (uint64_t r = mnfs[i]; r; r &= r - 1) lv_push(e, rank[__builtin_ctzll(r)]);
                qsort(e->a + 2, (size_t)e->len - 2, sizeof(long long), ll_cmp_q);
            }
            for (int i = 0; i < k; ++i) {
                if (!(facets[i] & vb)) continue;
                lvec *e = &env[ne++];
                e->len = 0;
                lv_push(e, 1);
                for (uint64_t r = facets[i]; r; r &= r - 1) lv_push(e, rank[__builtin_ctzll(r)]);
                qsort(e->a + 1, (size_t)e->len - 1, sizeof(long long), ll_cmp_q);
            }
            qsort(env, (size_t)ne, sizeof(lvec), lv_cmp_q);
            for (int i = 0; i < ne; ++i) {
                lv_push(&next[v], -1);
                for (int j = 0; j < env[i].len; ++j) lv_push(&next[v], env[i].a[j]);
            }
        }
        const int nc = ranks_of(m, next, nrank);
        if (nc == classes) break;
        memcpy(rank, nrank, (size_t)(m + 1) * sizeof(int));
        classes = nc;
    }
    for (int v = 1; v <= m; ++v) cls_out[v - 1] = rank[v];
    for (int i = 0; i < env_cap; ++i) free(env[i].a);
    for (int v = 0; v <= m; ++v) {
        free(key[v].a);
        free(next[v].a);
    }
    free(env);
    free(next);
    free(key);
    free(rank);
    free(nrank);
    free(mnfs);
    return classes;
}

/* ---- canonical_form (isomorphism.hpp:228-303) ------------------------------ */

typedef struct {
    int m, k;
    const uint64_t *facets;
    int label[21];
    int taken[21];
    int next_label;
    int nclass;
    int members[21][21];
    int nmem[21];
    uint64_t *best, *tmp;
    int have_best, nbest;
    long long leaves;
} cf_state;

/* prefix (:240-256): the facets fully labeled so far, relabeled, sorted */
static int cf_prefix(cf_state *s, uint64_t *out) {
    int c = 0;
    for (int i = 0; i < s->k; ++i) {
        uint64_t g = 0;
        int full = 1;
        for (uint64_t r = s->facets[i]; r; r &= r - 1) {
            const int v = __builtin_ctzll(r);
            if (s->label[v] == 0) full = 0;
            else g |= (uint64_t)1 << s->label[v];
        }
        if (full) out[c++] = g;
    }
    qsort(out, (size_t)c, sizeof(uint64_t), u64_cmp_q);
    return c;
}

static void cf_rec(cf_state *s, int class_idx);

static void cf_place(cf_state *s, int class_idx, int depth) {
    const int *mem = s->members[class_idx];
    const int nm = s->nmem[class_idx];
    if (depth == nm) {
        if (s->have_best) { /* :267-273 prune at the class boundary */
            const int c = cf_prefix(s, s->tmp);
            const int len = c < s->nbest ? c : s->nbest;
            for (int i = 0; i < len; ++i) {
                if (s->tmp[i] < s->best[i]) break;
                if (s->best[i] < s->tmp[i]) return;
            }
        }
        cf_rec(s, class_idx + 1);
        return;
    }
    for (int j = 0; j < nm; ++j) { /* :276-285 */
        const int v = mem[j];
        if (s->taken[v]) continue;
        s->taken[v] = 1;
        s->label[v] = s->next_label++;
        cf_place(s, class_idx, depth + 1);
        --s->next_label;
        s->label[v] = 0;
        s->taken[v] = 0;
    }
}

static void cf_rec(cf_state *s, int class_idx) {
    if (class_idx == s->nclass) { /* :259-265 */
        ++s->leaves;
        const int c = cf_prefix(s, s->tmp);
        int less = !s->have_best;
        if (!less) {
            for (int i = 0; i < c; ++i)
                if (s->tmp[i] != s->best[i]) {
                    less = s->tmp[i] < s->best[i];
                    break;
                }
        }
        if (less) {
            memcpy(s->best, s->tmp, (size_t)c * sizeof(uint64_t));
            s->nbest = c;
            s->have_best = 1;
        }
        return;
    }
    cf_place(s, class_idx, 0);
}

int po_canonical_form(int m, const uint64_t *facets, int k, uint64_t *out, long long *leaves_out) {
    if (m < 1 || m > 20) return -PO_EINVAL;
    if (k == 0) return 0; /* :229 */
    int cls[21];
    const int nc = po_refine_classes(m, facets, k, cls);
    if (nc < 0) return nc;
    cf_state s;
    memset(&s, 0, sizeof(s));
    s.m = m;
    s.k = k;
    s.facets = facets;
    s.nclass = nc;
    for (int v = 1; v <= m; ++v) { /* :232-233 members in ascending vertex order */
        const int c = cls[v - 1];
        s.members[c][s.nmem[c]++] = v;
    }
    s.best = (uint64_t *)malloc((size_t)k * sizeof(uint64_t));
    s.tmp = (uint64_t *)malloc((size_t)k * sizeof(uint64_t));
    s.next_label = 1;
    cf_rec(&s, 0);
    memcpy(out, s.best, (size_t)s.nbest * sizeof(uint64_t));
    if (leaves_out) *leaves_out = s.leaves;
    free(s.best);
    free(s.tmp);
    return s.nbest;
}
