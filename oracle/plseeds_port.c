/*
 * oracle/plseeds_port.c -- TEST INFRASTRUCTURE ONLY (see plseeds_port.h).
 *
 * Plain-C restatement of the reference's WPM-enumeration path: IDCM orbits,
 * the binary-matroid facet universe, the ridge-facet incidence, the GF(2)
 * kernel with its convenient (block) basis, link-constraint pinning, the
 * kernel-basis odometer of Algorithm 1 and the canonical output order.
 * Single-threaded; deterministic.  Each function cites what it restates.
 */
#include "plseeds_port.h"

#include <stdlib.h>
#include <string.h>
#include <stdio.h>

/* ------------------------------------------------------------------ util */

static int popc64(uint64_t x) { return __builtin_popcountll(x); }
static int ctz64(uint64_t x) { return __builtin_ctzll(x); }
static int lead64(uint64_t x) { return 63 - __builtin_clzll(x); } /* kernel_basis.hpp:60 */

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

/* bit vectors of `w` words */
static void bv_xor(uint64_t *d, const uint64_t *s, int w) { for (int i = 0; i < w; ++i) d[i] ^= s[i]; }
static int bv_test(const uint64_t *v, int i) { return (int)((v[i >> 6] >> (i & 63)) & 1u); }
static void bv_set(uint64_t *v, int i) { v[i >> 6] |= (uint64_t)1 << (i & 63); }

/* --------------------------------------------------------------- orbits */

/* gf2col::rank, charmap.hpp:92-107: min-reduction against a descending list */
static int gf2col_rank(const uint32_t *in, int k) {
    if (k <= 0) return 0;
    uint32_t v[64];
    int rank = 0;
    for (int i = 0; i < k; ++i) {
        uint32_t x = in[i];
        for (int j = 0; j < rank; ++j) {
            uint32_t y = x ^ v[j];
            if (y < x) x = y;
        }
        if (x) {
            v[rank] = x;
            for (int j = rank; j > 0 && v[j] > v[j - 1]; --j) {
                uint32_t t = v[j]; v[j] = v[j - 1]; v[j - 1] = t;
            }
            ++rank;
        }
    }
    return rank;
}

static int cmp_u32(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return x < y ? -1 : x > y;
}

static int lex_less_u32(const uint32_t *a, const uint32_t *b, int k) {
    for (int i = 0; i < k; ++i)
        if (a[i] != b[i]) return a[i] < b[i];
    return 0;
}

/* idcm_orbits, charmap.hpp:212-281 */
int po_idcm_orbits(int n, int p, uint32_t *rows_out, int cap) {
    if (n < 1 || p < 1 || p > 8) return -PO_EINVAL;
    if (n + p > (1 << p) - 1) return -PO_EINVAL;
    uint32_t pool[256];
    int pool_size = 0;
    for (uint32_t v = 1; v < (1u << p); ++v)
        if ((v & (v - 1)) != 0) pool[pool_size++] = v; /* :218-220 */
    if (n > pool_size) return -PO_EINVAL;

    /* all p! bit permutations in next_permutation order (:223-230) */
    int nperm = 1;
    for (int i = 2; i <= p; ++i) nperm *= i;
    int *perms = (int *)malloc(sizeof(int) * (size_t)nperm * (size_t)p);
    {
        int base[8];
        for (int i = 0; i < p; ++i) base[i] = i;
        for (int q = 0; q < nperm; ++q) {
            memcpy(perms + q * p, base, sizeof(int) * (size_t)p);
            /* next_permutation */
            int i = p - 2;
            while (i >= 0 && base[i] >= base[i + 1]) --i;
            if (i < 0) break;
            int j = p - 1;
            while (base[j] <= base[i]) --j;
            int t = base[i]; base[i] = base[j]; base[j] = t;
            for (int a = i + 1, b = p - 1; a < b; ++a, --b) { t = base[a]; base[a] = base[b]; base[b] = t; }
        }
    }

    int reps_cap = 1024, nreps = 0;
    uint32_t *reps = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)reps_cap * (size_t)n);
    int idx[64];
    for (int i = 0; i < n; ++i) idx[i] = i;
    uint32_t rows[64], best[64], tmp[64];
    for (;;) {
        for (int i = 0; i < n; ++i) rows[i] = pool[idx[i]];
        /* canonical(): lex-min sorted permuted row list (:237-249) */
        qsort(rows, (size_t)n, sizeof(uint32_t), cmp_u32);
        memcpy(best, rows, sizeof(uint32_t) * (size_t)n);
        for (int q = 0; q < nperm; ++q) {
            const int *perm = perms + q * p;
            for (int i = 0; i < n; ++i) {
                uint32_t o = 0;
                for (int b = 0; b < p; ++b)
                    if ((rows[i] >> b) & 1u) o |= 1u << perm[b];
                tmp[i] = o;
            }
            qsort(tmp, (size_t)n, sizeof(uint32_t), cmp_u32);
            if (q == 0 || lex_less_u32(tmp, best, n)) memcpy(best, tmp, sizeof(uint32_t) * (size_t)n);
        }
        int found = 0;
        for (int r = 0; r < nreps && !found; ++r)
            if (memcmp(reps + (size_t)r * n, best, sizeof(uint32_t) * (size_t)n) == 0) found = 1;
        if (!found) {
            if (nreps == reps_cap) {
                reps_cap *= 2;
                reps = (uint32_t *)realloc(reps, sizeof(uint32_t) * (size_t)reps_cap * (size_t)n);
            }
            memcpy(reps + (size_t)nreps * n, best, sizeof(uint32_t) * (size_t)n);
            ++nreps;
        }
        /* next combination (:261-266) */
        int pos = n - 1;
        while (pos >= 0 && idx[pos] == pool_size - (n - pos)) --pos;
        if (pos < 0) break;
        ++idx[pos];
        for (int i = pos + 1; i < n; ++i) idx[i] = idx[i - 1] + 1;
    }
    /* std::sort(reps) (:268): lexicographic; insertion sort is enough */
    for (int i = 1; i < nreps; ++i) {
        memcpy(tmp, reps + (size_t)i * n, sizeof(uint32_t) * (size_t)n);
        int j = i - 1;
        while (j >= 0 && lex_less_u32(tmp, reps + (size_t)j * n, n)) {
            memcpy(reps + (size_t)(j + 1) * n, reps + (size_t)j * n, sizeof(uint32_t) * (size_t)n);
            --j;
        }
        memcpy(reps + (size_t)(j + 1) * n, tmp, sizeof(uint32_t) * (size_t)n);
    }
    const int m = n + p;
    for (int r = 0; r < nreps && r < cap; ++r) {
        for (int i = 0; i < n; ++i) rows_out[(size_t)r * m + i] = reps[(size_t)r * n + i];
        for (int i = 0; i < p; ++i) rows_out[(size_t)r * m + n + i] = 1u << i; /* :277 */
    }
    free(reps);
    free(perms);
    return nreps;
}

/* charmap_of_dcm, charmap.hpp:155-204 */
int po_charmap_of_dcm(int m, int p, const uint32_t *rows, uint32_t *cols) {
    const int n = m - p;
    for (int i = 0; i < m; ++i) cols[i] = 0;
    int standard = 1; /* standard_form(), :78-82 */
    for (int i = 0; i < p; ++i)
        if (rows[m - p + i] != (1u << i)) standard = 0;
    if (standard) {
        for (int i = 0; i < n; ++i) cols[i] = 1u << i;
        for (int j = 0; j < p; ++j) {
            uint32_t c = 0;
            for (int i = 0; i < n; ++i)
                if ((rows[i] >> j) & 1u) c |= 1u << i;
            cols[n + j] = c;
        }
        return n;
    }
    /* general case (:171-203) */
    uint64_t mat[32];
    for (int j = 0; j < p; ++j) {
        mat[j] = 0;
        for (int v = 0; v < m; ++v)
            if ((rows[v] >> j) & 1u) mat[j] |= (uint64_t)1 << v;
    }
    int pivot_col[32], rank = 0;
    for (int c = 0; c < m && rank < p; ++c) {
        int piv = -1;
        for (int r = rank; r < p; ++r)
            if ((mat[r] >> c) & 1u) { piv = r; break; }
        if (piv < 0) continue;
        uint64_t t = mat[rank]; mat[rank] = mat[piv]; mat[piv] = t;
        for (int r = 0; r < p; ++r)
            if (r != rank && ((mat[r] >> c) & 1u)) mat[r] ^= mat[rank];
        pivot_col[rank++] = c;
    }
    if (rank != p) return -PO_EINVAL;
    int row = 0;
    for (int fc = 0; fc < m; ++fc) {
        int is_piv = 0;
        for (int r = 0; r < rank; ++r)
            if (pivot_col[r] == fc) is_piv = 1;
        if (is_piv) continue;
        cols[fc] |= 1u << row;
        for (int r = 0; r < rank; ++r)
            if ((mat[r] >> fc) & 1u) cols[pivot_col[r]] |= 1u << row;
        ++row;
    }
    return n;
}

/* binary_matroid, charmap.hpp:117-141 (then PureComplex sorts, complex.hpp:33) */
int po_binary_matroid(int n, int m, const uint32_t *cols, uint64_t *facets, int cap) {
    if (gf2col_rank(cols, m) != n) return -PO_EINVAL;
    int idx[64], M = 0;
    for (int i = 0; i < n; ++i) idx[i] = i + 1;
    uint32_t sel[64] = {0};
    for (;;) {
        for (int i = 0; i < n; ++i) sel[i] = cols[idx[i] - 1];
        if (gf2col_rank(sel, n) == n) {
            uint64_t f = 0;
            for (int i = 0; i < n; ++i) f |= (uint64_t)1 << idx[i];
            if (M < cap) facets[M] = f;
            ++M;
        }
        int pos = n - 1;
        while (pos >= 0 && idx[pos] == m - (n - 1 - pos)) --pos;
        if (pos < 0) break;
        ++idx[pos];
        for (int i = pos + 1; i < n; ++i) idx[i] = idx[i - 1] + 1;
    }
    if (M <= cap) qsort(facets, (size_t)M, sizeof(uint64_t), cmp_u64);
    return M;
}

/* all_subsets_universe, catalog.hpp:112-120 */
int po_all_subsets_universe(int m, int n, uint64_t *facets, int cap) {
    int M = 0;
    for (uint64_t s = 0; s < ((uint64_t)1 << m); ++s)
        if (popc64(s) == n) {
            if (M < cap) facets[M] = s << 1;
            ++M;
        }
    return M; /* ascending already */
}

/* cyclic_facet_bound, affine_property.hpp:35-45 */
static int64_t binom64(int64_t top, int64_t k) {
    if (top < k) return 0;
    int64_t r = 1;
    for (int64_t i = 1; i <= k; ++i) r = r * (top - k + i) / i;
    return r;
}
int64_t po_cyclic_facet_bound(int n) {
    const int64_t ch = (n + 1) / 2, fh = n / 2;
    return binom64(n + 4 - ch, 4) + binom64(n + 3 - fh, 4);
}

/* ------------------------------------------------------------ incidence */

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return x < y ? -1 : x > y;
}

static int find_u64(const uint64_t *arr, int len, uint64_t key) {
    int lo = 0, hi = len - 1;
    while (lo <= hi) {
        int mid = (lo + hi) / 2;
        if (arr[mid] == key) return mid;
        if (arr[mid] < key) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* ridges_of (complex.hpp:107-119) + incidence_matrix (incidence.hpp:34-55).
 * par_off has N+1 entries. */
int po_incidence(const uint64_t *facets, int M, uint64_t *ridges, int ridges_cap,
                 int32_t *cols, int32_t *par_off, int32_t *par) {
    if (M <= 0) return -PO_EINVAL; /* purity_error on empty */
    const int n = popc64(facets[0]);
    if (n < 1) return -PO_EINVAL;
    uint64_t *all = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M * (size_t)n);
    int k = 0;
    for (int j = 0; j < M; ++j) {
        if (popc64(facets[j]) != n) { free(all); return -PO_EINVAL; }
        for (uint64_t b = facets[j]; b; b &= b - 1) all[k++] = facets[j] & ~((uint64_t)1 << ctz64(b));
    }
    qsort(all, (size_t)k, sizeof(uint64_t), cmp_u64);
    int N = 0;
    for (int i = 0; i < k; ++i)
        if (i == 0 || all[i] != all[i - 1]) all[N++] = all[i];
    if (N > ridges_cap) { free(all); return N; }
    memcpy(ridges, all, sizeof(uint64_t) * (size_t)N);
    free(all);
    if (!cols) return N;
    for (int r = 0; r <= N; ++r) par_off[r] = 0;
    for (int j = 0; j < M; ++j) {
        int c = 0;
        for (uint64_t b = facets[j]; b; b &= b - 1)
            cols[j * n + c++] = find_u64(ridges, N, facets[j] & ~((uint64_t)1 << ctz64(b)));
        qsort(cols + j * n, (size_t)n, sizeof(int32_t), cmp_i32);
        for (int q = 0; q < n; ++q) par_off[cols[j * n + q] + 1]++;
    }
    for (int r = 0; r < N; ++r) par_off[r + 1] += par_off[r];
    int32_t *fill = (int32_t *)calloc((size_t)N, sizeof(int32_t));
    for (int j = 0; j < M; ++j)
        for (int q = 0; q < n; ++q) {
            int r = cols[j * n + q];
            par[par_off[r] + fill[r]++] = j; /* ascending j, as :300 */
        }
    free(fill);
    return N;
}

/* ------------------------------------------------------- kernel / basis */

typedef struct {
    int M, W;        /* facets, words per generator */
    int s;           /* generators */
    uint64_t *gens;  /* s * W */
    int nblocks;
    int *boff, *bwid, *bridge;
    int pinned_ones, pinned_zeros;
} kbasis;

#define GEN(kb, g) ((kb)->gens + (size_t)(g) * (size_t)(kb)->W)

/* gf2_kernel, bitmatrix.hpp:125-153, on the N x M incidence (incidence.hpp:59-61) */
static void gf2_kernel(int N, int M, int n, const int32_t *cols, kbasis *kb) {
    const int W = (M + 63) / 64;
    uint64_t *a = (uint64_t *)calloc((size_t)N * (size_t)W, sizeof(uint64_t));
    for (int j = 0; j < M; ++j)
        for (int q = 0; q < n; ++q) bv_set(a + (size_t)cols[j * n + q] * W, j);
    int *pivot_col = (int *)malloc(sizeof(int) * (size_t)(M + 1));
    int rank = 0;
    for (int c = 0; c < M && rank < N; ++c) {
        int piv = -1;
        for (int r = rank; r < N; ++r)
            if (bv_test(a + (size_t)r * W, c)) { piv = r; break; }
        if (piv < 0) continue;
        if (piv != rank)
            for (int w = 0; w < W; ++w) {
                uint64_t t = a[(size_t)rank * W + w];
                a[(size_t)rank * W + w] = a[(size_t)piv * W + w];
                a[(size_t)piv * W + w] = t;
            }
        for (int r = 0; r < N; ++r)
            if (r != rank && bv_test(a + (size_t)r * W, c)) bv_xor(a + (size_t)r * W, a + (size_t)rank * W, W);
        pivot_col[rank++] = c;
    }
    char *is_piv = (char *)calloc((size_t)M, 1);
    for (int r = 0; r < rank; ++r) is_piv[pivot_col[r]] = 1;
    kb->M = M;
    kb->W = W;
    kb->s = M - rank;
    kb->gens = (uint64_t *)calloc((size_t)(kb->s > 0 ? kb->s : 1) * (size_t)W, sizeof(uint64_t));
    int g = 0;
    for (int fc = 0; fc < M; ++fc) {
        if (is_piv[fc]) continue;
        uint64_t *v = GEN(kb, g);
        bv_set(v, fc);
        for (int r = 0; r < rank; ++r)
            if (bv_test(a + (size_t)r * W, fc)) bv_set(v, pivot_col[r]);
        ++g;
    }
    kb->nblocks = 0;
    kb->boff = (int *)malloc(sizeof(int) * (size_t)(kb->s + 1));
    kb->bwid = (int *)malloc(sizeof(int) * (size_t)(kb->s + 1));
    kb->bridge = (int *)malloc(sizeof(int) * (size_t)(kb->s + 1));
    kb->pinned_ones = kb->pinned_zeros = 0;
    free(a);
    free(pivot_col);
    free(is_piv);
}

static void kb_free(kbasis *kb) {
    free(kb->gens);
    free(kb->boff);
    free(kb->bwid);
    free(kb->bridge);
}

/* reduce_value, kernel_basis.hpp:63-67 (echelon kept in descending order) */
static uint64_t reduce_value(uint64_t v, const uint64_t *ech, int k) {
    for (int i = 0; i < k; ++i)
        if (v && lead64(v) == lead64(ech[i])) v ^= ech[i];
    return v;
}

/* restrict_to, kernel_basis.hpp:69-74 */
static uint64_t restrict_to(const uint64_t *g, const int32_t *P, int p) {
    uint64_t v = 0;
    for (int i = 0; i < p; ++i)
        if (bv_test(g, P[i])) v |= (uint64_t)1 << i;
    return v;
}

static void sort_desc_u64(uint64_t *v, int k) { /* insertion: new item at end */
    for (int j = k - 1; j > 0 && v[j] > v[j - 1]; --j) {
        uint64_t t = v[j]; v[j] = v[j - 1]; v[j - 1] = t;
    }
}

static int uf_find(int *comp, int x) { /* path halving as kernel_basis.hpp:108-111 */
    while (comp[x] != x) x = comp[x] = comp[comp[x]];
    return x;
}

/* try_make_block, kernel_basis.hpp:84-190 */
static int try_make_block(kbasis *kb, const int32_t *P, int p, int ridge, int offset) {
    if (p < 3 || p > 64) return 0;
    const int s = kb->s, W = kb->W;
    uint64_t ech[64];
    int k = 0;
    for (int g = offset; g < s; ++g) {
        uint64_t v = reduce_value(restrict_to(GEN(kb, g), P, p), ech, k);
        if (v) { ech[k++] = v; sort_desc_u64(ech, k); }
    }
    if (k < 2) return 0;
    int comp[64];
    for (int i = 0; i < p; ++i) comp[i] = i;
    for (int a = 0; a < p; ++a)
        for (int b = a + 1; b < p; ++b)
            if (reduce_value(((uint64_t)1 << a) | ((uint64_t)1 << b), ech, k) == 0) {
                int ra = uf_find(comp, a), rb = uf_find(comp, b);
                if (ra != rb) comp[ra] = rb;
            }
    int clique[64], csz = 0;
    for (int root = 0; root < p && csz == 0; ++root) {
        if (uf_find(comp, root) != root) continue;
        int mem[64], nm = 0;
        for (int i = 0; i < p; ++i)
            if (uf_find(comp, i) == root) mem[nm++] = i;
        if (nm == k + 1) { memcpy(clique, mem, sizeof(int) * (size_t)nm); csz = nm; }
    }
    if (csz == 0) return 0;
    for (int g = 0; g < offset; ++g)
        if (reduce_value(restrict_to(GEN(kb, g), P, p), ech, k) != 0) return 0;

    /* commit: forward echelon with generator bookkeeping (:133-147) */
    uint64_t pv[64];
    int pg[64], np = 0;
    for (int g = offset; g < s; ++g) {
        uint64_t v = restrict_to(GEN(kb, g), P, p);
        for (int i = 0; i < np; ++i)
            if (v && lead64(v) == lead64(pv[i])) {
                v ^= pv[i];
                bv_xor(GEN(kb, g), GEN(kb, pg[i]), W);
            }
        if (v) {
            pv[np] = v; pg[np] = g; ++np;
            for (int j = np - 1; j > 0 && pv[j] > pv[j - 1]; --j) {
                uint64_t t = pv[j]; pv[j] = pv[j - 1]; pv[j - 1] = t;
                int u = pg[j]; pg[j] = pg[j - 1]; pg[j - 1] = u;
            }
        }
    }
    const int last = clique[csz - 1];
    const int nstar = csz - 1;
    uint64_t *star = (uint64_t *)calloc((size_t)nstar * (size_t)W, sizeof(uint64_t));
    int star_row[64];
    for (int i = 0; i < nstar; ++i) {
        uint64_t v = ((uint64_t)1 << clique[i]) | ((uint64_t)1 << last);
        for (int q = 0; q < np; ++q)
            if (v && lead64(v) == lead64(pv[q])) {
                v ^= pv[q];
                bv_xor(star + (size_t)i * W, GEN(kb, pg[q]), W);
            }
        if (v != 0) { free(star); return 0; } /* unreachable (:162) */
        star_row[i] = clique[i];
    }
    /* rebuild the tail (:168-177) */
    uint64_t *tail = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(s - offset) * (size_t)W);
    int t = 0;
    for (int i = 0; i < nstar; ++i, ++t) memcpy(tail + (size_t)t * W, star + (size_t)i * W, sizeof(uint64_t) * (size_t)W);
    char *is_piv = (char *)calloc((size_t)s, 1);
    for (int i = 0; i < np; ++i) is_piv[pg[i]] = 1;
    for (int g = offset; g < s; ++g)
        if (!is_piv[g]) { memcpy(tail + (size_t)t * W, GEN(kb, g), sizeof(uint64_t) * (size_t)W); ++t; }
    memcpy(GEN(kb, offset), tail, sizeof(uint64_t) * (size_t)(s - offset) * (size_t)W);
    /* clear earlier columns on the parent rows (:180-186) */
    for (int g = 0; g < offset; ++g) {
        const uint64_t u = restrict_to(GEN(kb, g), P, p);
        if (!u) continue;
        for (int i = 0; i < nstar; ++i)
            if ((u >> star_row[i]) & 1u) bv_xor(GEN(kb, g), GEN(kb, offset + i), W);
    }
    kb->boff[kb->nblocks] = offset;
    kb->bwid[kb->nblocks] = k;
    kb->bridge[kb->nblocks] = ridge;
    kb->nblocks++;
    free(star);
    free(tail);
    free(is_piv);
    return 1;
}

/* convenient_basis, kernel_basis.hpp:198-235 */
static void convenient_basis(kbasis *kb, int N, int M, const int32_t *par_off, const int32_t *par) {
    char *ridge_used = (char *)calloc((size_t)N, 1);
    char *facet_used = (char *)calloc((size_t)M, 1);
    int *cand = (int *)malloc(sizeof(int) * (size_t)(N + 1));
    int offset = 0;
    while (offset < kb->s) {
        int nc = 0;
        for (int r = 0; r < N; ++r) {
            if (ridge_used[r]) continue;
            int disjoint = 1;
            for (int q = par_off[r]; q < par_off[r + 1]; ++q)
                if (facet_used[par[q]]) { disjoint = 0; break; }
            if (disjoint) cand[nc++] = r;
        }
        /* stable order: parent count desc, index asc (:216-220) */
        for (int i = 1; i < nc; ++i) {
            int x = cand[i], px = par_off[x + 1] - par_off[x];
            int j = i - 1;
            while (j >= 0) {
                int y = cand[j], py = par_off[y + 1] - par_off[y];
                if (py > px || (py == px && y < x)) break;
                cand[j + 1] = cand[j];
                --j;
            }
            cand[j + 1] = x;
        }
        int advanced = 0;
        for (int i = 0; i < nc; ++i) {
            int r = cand[i];
            ridge_used[r] = 1;
            if (try_make_block(kb, par + par_off[r], par_off[r + 1] - par_off[r], r, offset)) {
                for (int q = par_off[r]; q < par_off[r + 1]; ++q) facet_used[par[q]] = 1;
                offset += kb->bwid[kb->nblocks - 1];
                advanced = 1;
                break;
            }
        }
        if (!advanced) break;
    }
    free(ridge_used);
    free(facet_used);
    free(cand);
}

/* apply_link_constraints, kernel_basis.hpp:248-321.  0 ok, PO_EINFEASIBLE */
static int apply_link_constraints(kbasis *kb, const int32_t *req, int nreq, const int32_t *forb, int nforb) {
    if (nreq == 0 && nforb == 0) return PO_OK;
    for (int i = 0; i < nreq; ++i)
        for (int j = 0; j < nforb; ++j)
            if (req[i] == forb[j]) return PO_EINFEASIBLE;
    const int s = kb->s, W = kb->W, nrows = nreq + nforb;
    int *rf = (int *)malloc(sizeof(int) * (size_t)(nrows + 1));
    char *rt = (char *)malloc((size_t)(nrows + 1));
    for (int i = 0; i < nreq; ++i) { rf[i] = req[i]; rt[i] = 1; }
    for (int i = 0; i < nforb; ++i) { rf[nreq + i] = forb[i]; rt[nreq + i] = 0; }
    int *pivot_of_row = (int *)malloc(sizeof(int) * (size_t)(nrows + 1));
    uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)W);
    int cur = 0;
    for (int ri = 0; ri < nrows; ++ri) {
        pivot_of_row[ri] = -1;
        int pivot = -1;
        for (int g = cur; g < s; ++g)
            if (bv_test(GEN(kb, g), rf[ri])) { pivot = g; break; }
        if (pivot < 0) continue;
        memcpy(tmp, GEN(kb, pivot), sizeof(uint64_t) * (size_t)W);
        memcpy(GEN(kb, pivot), GEN(kb, cur), sizeof(uint64_t) * (size_t)W);
        memcpy(GEN(kb, cur), tmp, sizeof(uint64_t) * (size_t)W);
        for (int g = 0; g < s; ++g)
            if (g != cur && bv_test(GEN(kb, g), rf[ri])) bv_xor(GEN(kb, g), GEN(kb, cur), W);
        pivot_of_row[ri] = cur++;
    }
    int *ones = (int *)malloc(sizeof(int) * (size_t)(nrows + 1));
    int *zeros = (int *)malloc(sizeof(int) * (size_t)(nrows + 1));
    int no = 0, nz = 0;
    for (int ri = 0; ri < nrows; ++ri) {
        int g = pivot_of_row[ri];
        if (g < 0) continue;
        if (rt[ri]) ones[no++] = g; else zeros[nz++] = g;
    }
    int feasible = 1;
    for (int ri = 0; ri < nrows && feasible; ++ri) {
        int value = 0;
        for (int i = 0; i < no; ++i)
            if (bv_test(GEN(kb, ones[i]), rf[ri])) value ^= 1;
        if (value != rt[ri]) feasible = 0;
    }
    if (feasible) {
        uint64_t *ng = (uint64_t *)calloc((size_t)(s > 0 ? s : 1) * (size_t)W, sizeof(uint64_t));
        char *placed = (char *)calloc((size_t)(s + 1), 1);
        int t = 0;
        for (int i = 0; i < no; ++i, ++t) { memcpy(ng + (size_t)t * W, GEN(kb, ones[i]), sizeof(uint64_t) * (size_t)W); placed[ones[i]] = 1; }
        for (int i = 0; i < nz; ++i, ++t) { memcpy(ng + (size_t)t * W, GEN(kb, zeros[i]), sizeof(uint64_t) * (size_t)W); placed[zeros[i]] = 1; }
        for (int g = 0; g < s; ++g)
            if (!placed[g]) { memcpy(ng + (size_t)t * W, GEN(kb, g), sizeof(uint64_t) * (size_t)W); ++t; }
        free(kb->gens);
        kb->gens = ng;
        kb->nblocks = 0; /* blocks do not survive (:246-247) */
        kb->pinned_ones = no;
        kb->pinned_zeros = nz;
        free(placed);
    }
    free(rf); free(rt); free(pivot_of_row); free(tmp); free(ones); free(zeros);
    return feasible ? PO_OK : PO_EINFEASIBLE;
}

/* ------------------------------------------------------ canonical order */

int po_bits_cmp(const uint64_t *a, const uint64_t *b, int words) {
    /* lexicographic order of the ascending facet-index lists (search.hpp:254-255,
     * std::vector operator<): the first differing index decides; a proper
     * prefix sorts first. */
    for (int w = 0; w < words; ++w) {
        uint64_t x = a[w] ^ b[w];
        if (!x) continue;
        const uint64_t low = x & (~x + 1);
        const uint64_t above = ~((low << 1) - 1); /* bits strictly above d in word w */
        int a_has_d = (a[w] & low) != 0;
        const uint64_t *other = a_has_d ? b : a;
        int other_more = (other[w] & above) != 0;
        for (int v = w + 1; v < words && !other_more; ++v)
            if (other[v]) other_more = 1;
        /* the list holding d is smaller iff the other list continues past d */
        if (a_has_d) return other_more ? -1 : 1;
        return other_more ? 1 : -1;
    }
    return 0;
}

static int g_sort_words;
static int cmp_bits_q(const void *a, const void *b) {
    return po_bits_cmp((const uint64_t *)a, (const uint64_t *)b, g_sort_words);
}

/* ----------------------------------------------------------- enumerate */

typedef struct {
    int W;
    int64_t count, cap;
    uint64_t *bits;
} bucket;

static void bucket_push(bucket *b, const uint64_t *v) {
    if (b->count == b->cap) {
        b->cap = b->cap ? b->cap * 2 : 1024;
        b->bits = (uint64_t *)realloc(b->bits, sizeof(uint64_t) * (size_t)b->cap * (size_t)b->W);
    }
    memcpy(b->bits + (size_t)b->count * b->W, v, sizeof(uint64_t) * (size_t)b->W);
    b->count++;
}

/* wpm_counts_ok, search.hpp:114-131 */
static int wpm_counts_ok(const uint64_t *K, int W, int n, const int32_t *cols, uint8_t *cnt,
                         int32_t *touched) {
    int nt = 0, ok = 1;
    for (int w = 0; w < W && ok; ++w)
        for (uint64_t x = K[w]; x && ok; x &= x - 1) {
            const int j = w * 64 + ctz64(x);
            for (int q = 0; q < n; ++q) {
                const int r = cols[j * n + q];
                if (cnt[r] == 0) touched[nt++] = r;
                if (++cnt[r] >= 3) { ok = 0; break; }
            }
        }
    if (ok)
        for (int i = 0; i < nt; ++i)
            if (cnt[touched[i]] != 2) { ok = 0; break; }
    for (int i = 0; i < nt; ++i) cnt[touched[i]] = 0;
    return ok;
}

typedef struct {
    int ncand;
    uint64_t *deltas; /* ncand * W */
} pblock;

static int cmp_pblock_desc(const void *a, const void *b) {
    const pblock *x = (const pblock *)a, *y = (const pblock *)b;
    return y->ncand - x->ncand;
}

/* enumerate_wpm, search.hpp:141-258 (single worker; the outer/inner split of
 * :172-178 is kept because it fixes the leaf order only, not the output) */
int po_enumerate_wpm(int m, int n, const uint64_t *facets, int M, int64_t facet_cap,
                     const int32_t *required, int nreq, const int32_t *forbidden, int nforb,
                     uint64_t candidate_cap, po_result *out) {
    memset(out, 0, sizeof(*out));
    (void)m;
    if (M <= 0) return PO_EINVAL;
    for (int j = 0; j < M; ++j)
        if (popc64(facets[j]) != n) return PO_EINVAL;
    const int W = (M + 63) / 64;
    uint64_t *ridges = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M * (size_t)n);
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)M * (size_t)n);
    int32_t *par_off = (int32_t *)malloc(sizeof(int32_t) * ((size_t)M * (size_t)n + 1));
    int32_t *par = (int32_t *)malloc(sizeof(int32_t) * (size_t)M * (size_t)n);
    const int N = po_incidence(facets, M, ridges, M * n, cols, par_off, par);
    if (N < 0) { free(ridges); free(cols); free(par_off); free(par); return PO_EINVAL; }

    kbasis kb;
    gf2_kernel(N, M, n, cols, &kb);
    convenient_basis(&kb, N, M, par_off, par);
    out->s = kb.s;
    out->nblocks = kb.nblocks;
    int rc = apply_link_constraints(&kb, required, nreq, forbidden, nforb);
    if (rc != PO_OK) { kb_free(&kb); free(ridges); free(cols); free(par_off); free(par); return rc; }

    /* combination_space, search.hpp:81-104 */
    const int first_free = kb.pinned_ones + kb.pinned_zeros;
    int covered = first_free;
    int nb = 0;
    pblock *blocks = (pblock *)calloc((size_t)(kb.s + 1), sizeof(pblock));
    for (int b = 0; b < kb.nblocks; ++b) {
        const int off = kb.boff[b], wd = kb.bwid[b];
        const int nc = 1 + wd + wd * (wd - 1) / 2;
        pblock *pb = &blocks[nb++];
        pb->ncand = nc;
        pb->deltas = (uint64_t *)calloc((size_t)nc * (size_t)W, sizeof(uint64_t));
        int c = 1;
        for (int i = 0; i < wd; ++i, ++c) bv_xor(pb->deltas + (size_t)c * W, GEN(&kb, off + i), W);
        for (int i = 0; i < wd; ++i)
            for (int j = i + 1; j < wd; ++j, ++c) {
                bv_xor(pb->deltas + (size_t)c * W, GEN(&kb, off + i), W);
                bv_xor(pb->deltas + (size_t)c * W, GEN(&kb, off + j), W);
            }
        if (off + wd > covered) covered = off + wd;
    }
    for (int g = covered; g < kb.s; ++g) {
        pblock *pb = &blocks[nb++];
        pb->ncand = 2;
        pb->deltas = (uint64_t *)calloc((size_t)2 * (size_t)W, sizeof(uint64_t));
        bv_xor(pb->deltas + W, GEN(&kb, g), W);
    }
    uint64_t space = 1; /* size_saturated, :70-78 */
    for (int b = 0; b < nb; ++b) {
        const uint64_t c = (uint64_t)blocks[b].ncand;
        if (space > UINT64_MAX / c) { space = UINT64_MAX; break; }
        space *= c;
    }
    out->space = space;
    if (space > candidate_cap) {
        for (int b = 0; b < nb; ++b) free(blocks[b].deltas);
        free(blocks); kb_free(&kb); free(ridges); free(cols); free(par_off); free(par);
        return PO_ECAP;
    }
    uint64_t *base = (uint64_t *)calloc((size_t)W, sizeof(uint64_t));
    for (int g = 0; g < kb.pinned_ones; ++g) bv_xor(base, GEN(&kb, g), W);
    /* widest blocks outermost (stable, :168-170) */
    {
        /* stable insertion sort by ncand descending */
        for (int i = 1; i < nb; ++i) {
            pblock x = blocks[i];
            int j = i - 1;
            while (j >= 0 && blocks[j].ncand < x.ncand) { blocks[j + 1] = blocks[j]; --j; }
            blocks[j + 1] = x;
        }
        (void)cmp_pblock_desc;
    }

    bucket bk = {W, 0, 0, NULL};
    uint8_t *cnt = (uint8_t *)calloc((size_t)N, 1);
    int32_t *touched = (int32_t *)malloc(sizeof(int32_t) * (size_t)(N + 1));
    uint64_t *stack = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nb + 1) * (size_t)W);
    int *pos = (int *)calloc((size_t)(nb + 1), sizeof(int));
    memcpy(stack, base, sizeof(uint64_t) * (size_t)W);
    /* odometer over every block (:215-243 with the whole product inner) */
    int level = 0;
    for (;;) {
        if (level == nb) {
            const uint64_t *cand = stack + (size_t)level * W;
            int any = 0, pc = 0;
            for (int w = 0; w < W; ++w) { any |= cand[w] != 0; pc += popc64(cand[w]); }
            if (any && (facet_cap < 0 || pc <= facet_cap) && wpm_counts_ok(cand, W, n, cols, cnt, touched))
                bucket_push(&bk, cand);
            while (level > 0 && pos[level - 1] + 1 == blocks[level - 1].ncand) --level;
            if (level == 0) break;
            ++pos[level - 1];
            memcpy(stack + (size_t)level * W, stack + (size_t)(level - 1) * W, sizeof(uint64_t) * (size_t)W);
            bv_xor(stack + (size_t)level * W, blocks[level - 1].deltas + (size_t)pos[level - 1] * W, W);
            for (int l = level; l < nb; ++l) pos[l] = 0;
            continue;
        }
        memcpy(stack + (size_t)(level + 1) * W, stack + (size_t)level * W, sizeof(uint64_t) * (size_t)W);
        bv_xor(stack + (size_t)(level + 1) * W, blocks[level].deltas + (size_t)pos[level] * W, W);
        ++level;
    }
    /* merge + sort + unique (:247-257) */
    g_sort_words = W;
    if (bk.count > 1) qsort(bk.bits, (size_t)bk.count, sizeof(uint64_t) * (size_t)W, cmp_bits_q);
    int64_t u = 0;
    for (int64_t i = 0; i < bk.count; ++i)
        if (u == 0 || po_bits_cmp(bk.bits + (size_t)(u - 1) * W, bk.bits + (size_t)i * W, W) != 0) {
            if (u != i) memcpy(bk.bits + (size_t)u * W, bk.bits + (size_t)i * W, sizeof(uint64_t) * (size_t)W);
            ++u;
        }
    out->count = u;
    out->words = W;
    out->bits = bk.bits;

    for (int b = 0; b < nb; ++b) free(blocks[b].deltas);
    free(blocks); free(base); free(cnt); free(touched); free(stack); free(pos);
    kb_free(&kb); free(ridges); free(cols); free(par_off); free(par);
    return PO_OK;
}

void po_result_free(po_result *r) {
    if (r && r->bits) free(r->bits);
    if (r) r->bits = NULL;
}

/* --------------------------------------------------------- brute force */

/* brute_force_wpm_count, acceptance.cpp:54-92 */
int64_t po_brute_force_count(const uint64_t *facets, int M, const int32_t *required, int nreq,
                             const int32_t *forbidden, int nforb, int64_t facet_cap) {
    if (M <= 0 || M > 40) return -1;
    const int n = popc64(facets[0]);
    uint64_t *ridges = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M * (size_t)n);
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)M * (size_t)n);
    int32_t *par_off = (int32_t *)malloc(sizeof(int32_t) * ((size_t)M * (size_t)n + 1));
    int32_t *par = (int32_t *)malloc(sizeof(int32_t) * (size_t)M * (size_t)n);
    const int N = po_incidence(facets, M, ridges, M * n, cols, par_off, par);
    if (N < 0) { free(ridges); free(cols); free(par_off); free(par); return -1; }
    int *cnt = (int *)calloc((size_t)N, sizeof(int));
    char in_req[64] = {0}, in_forb[64] = {0}, sel[64] = {0};
    for (int i = 0; i < nreq; ++i) in_req[required[i]] = 1;
    for (int i = 0; i < nforb; ++i) in_forb[forbidden[i]] = 1;
    int bad = 0, missing = nreq, clashes = 0, size = 0;
    int64_t total = 0;
    const uint64_t end = (uint64_t)1 << M;
    for (uint64_t i = 1; i < end; ++i) {
        const int j = ctz64(i);
        const int adding = !sel[j];
        sel[j] ^= 1;
        size += adding ? 1 : -1;
        if (in_req[j]) missing += adding ? -1 : 1;
        if (in_forb[j]) clashes += adding ? 1 : -1;
        for (int q = 0; q < n; ++q) {
            int *c = &cnt[cols[j * n + q]];
            const int was_ok = *c == 0 || *c == 2;
            *c += adding ? 1 : -1;
            const int now_ok = *c == 0 || *c == 2;
            bad += was_ok - now_ok;
        }
        if (bad == 0 && size > 0 && missing == 0 && clashes == 0 && (facet_cap < 0 || size <= facet_cap))
            ++total;
    }
    free(cnt); free(ridges); free(cols); free(par_off); free(par);
    return total;
}

/* is_weak_pseudomanifold_direct, complex.hpp:224-233 */
int po_is_wpm_direct(const uint64_t *facets, int k) {
    if (k == 0) return 1;
    const int n = popc64(facets[0]);
    for (int i = 0; i < k; ++i)
        for (uint64_t b = facets[i]; b; b &= b - 1) {
            const uint64_t r = facets[i] & ~((uint64_t)1 << ctz64(b));
            int c = 0;
            for (int j = 0; j < k; ++j)
                if ((r & ~facets[j]) == 0 && ++c > 2) break;
            if (c != 2) return 0;
        }
    (void)n;
    return 1;
}

/* ------------------------------------------------------------ .cplx io */

/* write_complex / write_complexes, complex_io.hpp:21-39 */
int64_t po_write_cplx(int m, int n, const uint64_t *universe, int M, const uint64_t *bits,
                      int64_t count, int words, char *buf, int64_t buf_len) {
    (void)M;
    int64_t len = 0;
    char line[512];
    for (int64_t i = 0; i < count; ++i) {
        int k = 0;
        if (i > 0) line[k++] = '\n';
        k += snprintf(line + k, sizeof(line) - (size_t)k, "%d %d\n", m, n);
        if (len + k <= buf_len) memcpy(buf + len, line, (size_t)k);
        len += k;
        const uint64_t *K = bits + (size_t)i * (size_t)words;
        for (int w = 0; w < words; ++w)
            for (uint64_t x = K[w]; x; x &= x - 1) {
                const uint64_t f = universe[w * 64 + ctz64(x)];
                k = 0;
                int first = 1;
                for (uint64_t y = f; y; y &= y - 1) {
                    if (!first) line[k++] = ' ';
                    k += snprintf(line + k, sizeof(line) - (size_t)k, "%d", ctz64(y));
                    first = 0;
                }
                line[k++] = '\n';
                if (len + k <= buf_len) memcpy(buf + len, line, (size_t)k);
                len += k;
            }
    }
    return len;
}
