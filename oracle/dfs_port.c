/*
 * oracle/dfs_port.c -- TEST INFRASTRUCTURE ONLY (see dfs_port.h).
 *
 * The search tree (identical to the GPU kernel's, node for node):
 *   state   : facet status U/IN/OUT, per-ridge IN-count c(r) and undecided
 *             parent count a(r); dead iff some ridge has c=1, a=0.
 *   include : f -> IN; every ridge of f gains a count; a ridge reaching c=2
 *             excludes its remaining undecided parents (propagation).
 *   open    : (some c(r)=1) prune if |S| + ceil(open/n) > cap; pick the open
 *             ridge with the fewest undecided parents (ties: lowest index),
 *             branch "include u_i, exclude u_1..u_{i-1}" over its undecided
 *             parents in ascending order.
 *   closed  : (no c(r)=1) emit S if nonempty; if |S| + n + 1 <= cap branch
 *             "include f, exclude every undecided facet < f" over the
 *             undecided facets f in ascending order (next component by its
 *             minimum facet; a nonempty WPM has >= n+1 facets).
 * Every nonempty WPM is emitted exactly once (branches are disjoint and
 * exhaustive).  One "node" = one include step.
 */
#include "dfs_port.h"

#include <stdlib.h>
#include <string.h>

#include "plseeds_port.h"

enum { ST_U = 0, ST_IN = 1, ST_OUT = 2 };

typedef struct {
    int n, M, N, W;
    int64_t cap;
    const int32_t *fr;   /* M*n ridges of each facet */
    int32_t *rp;         /* N*8 parents, -1 padded */
    uint8_t *npar;
    uint8_t *st;
    uint8_t *cnt, *av;
    int size, nopen, ndead;
    int32_t *trail;      /* encoded ops: (f<<1)|is_include */
    int ntrail;
    int64_t nodes;
    int want_bits;
    int64_t count, bcap;
    uint64_t *bits;
} dfs_ctx;

static void ridge_dec_av(dfs_ctx *c, int r) {
    c->av[r]--;
    if (c->cnt[r] == 1 && c->av[r] == 0) c->ndead++;
}
static void ridge_inc_av(dfs_ctx *c, int r) {
    if (c->cnt[r] == 1 && c->av[r] == 0) c->ndead--;
    c->av[r]++;
}

static void do_exclude(dfs_ctx *c, int g) {
    c->st[g] = ST_OUT;
    for (int k = 0; k < c->n; ++k) ridge_dec_av(c, c->fr[g * c->n + k]);
    c->trail[c->ntrail++] = g << 1;
}

static void do_include(dfs_ctx *c, int f) {
    c->st[f] = ST_IN;
    c->size++;
    c->trail[c->ntrail++] = (f << 1) | 1;
    for (int k = 0; k < c->n; ++k) {
        const int r = c->fr[f * c->n + k];
        const int wasdead = c->cnt[r] == 1 && c->av[r] == 0;
        c->av[r]--;
        c->cnt[r]++;
        if (c->cnt[r] == 1) {
            c->nopen++;
            if (c->av[r] == 0) c->ndead++;
        } else { /* 1 -> 2: closes; wasdead impossible since f was undecided */
            (void)wasdead;
            c->nopen--;
        }
    }
    for (int k = 0; k < c->n; ++k) {
        const int r = c->fr[f * c->n + k];
        if (c->cnt[r] != 2) continue;
        for (int q = 0; q < c->npar[r]; ++q) {
            const int g = c->rp[r * 8 + q];
            if (c->st[g] == ST_U) do_exclude(c, g);
        }
    }
}

static void undo_to(dfs_ctx *c, int mark) {
    while (c->ntrail > mark) {
        const int e = c->trail[--c->ntrail];
        const int f = e >> 1;
        if (e & 1) {
            for (int k = 0; k < c->n; ++k) {
                const int r = c->fr[f * c->n + k];
                if (c->cnt[r] == 1) {
                    if (c->av[r] == 0) c->ndead--;
                    c->nopen--;
                } else {
                    c->nopen++;
                }
                c->cnt[r]--;
                c->av[r]++;
            }
            c->size--;
        } else {
            for (int k = 0; k < c->n; ++k) ridge_inc_av(c, c->fr[f * c->n + k]);
        }
        c->st[f] = ST_U;
    }
}

static void emit(dfs_ctx *c) {
    c->count++;
    if (!c->want_bits) return;
    if (c->count > c->bcap) {
        c->bcap = c->bcap ? c->bcap * 2 : 1024;
        c->bits = (uint64_t *)realloc(c->bits, sizeof(uint64_t) * (size_t)c->bcap * (size_t)c->W);
    }
    uint64_t *o = c->bits + (size_t)(c->count - 1) * c->W;
    memset(o, 0, sizeof(uint64_t) * (size_t)c->W);
    for (int f = 0; f < c->M; ++f)
        if (c->st[f] == ST_IN) o[f >> 6] |= (uint64_t)1 << (f & 63);
}

static int choose_ridge(dfs_ctx *c) {
    int best = -1, bav = 99;
    for (int r = 0; r < c->N; ++r)
        if (c->cnt[r] == 1 && c->av[r] < bav) {
            bav = c->av[r];
            best = r;
            if (bav <= 1) break;
        }
    return best;
}

static void search(dfs_ctx *c);

/* branch: include f as a node, recurse, undo the include */
static void child(dfs_ctx *c, int f) {
    const int mark = c->ntrail;
    do_include(c, f);
    c->nodes++;
    if (c->ndead == 0) search(c);
    undo_to(c, mark);
}

static void search(dfs_ctx *c) {
    const int mark = c->ntrail;
    if (c->nopen == 0) {
        if (c->size > 0) emit(c);
        if (c->cap >= 0 && c->size + c->n + 1 > c->cap) return;
        for (int f = 0; f < c->M; ++f) {
            if (c->st[f] != ST_U) continue;
            child(c, f);
            do_exclude(c, f);
        }
    } else {
        if (c->cap >= 0 && c->size + (c->nopen + c->n - 1) / c->n > c->cap) return;
        const int r = choose_ridge(c);
        for (int q = 0; q < c->npar[r]; ++q) {
            const int u = c->rp[r * 8 + q];
            if (c->st[u] != ST_U) continue;
            child(c, u);
            do_exclude(c, u);
            if (c->ndead) break;
        }
    }
    undo_to(c, mark);
}

static int g_words;
static int cmp_bits(const void *a, const void *b) {
    return po_bits_cmp((const uint64_t *)a, (const uint64_t *)b, g_words);
}

static int g_shard_index = 0, g_shard_count = 1;

/* dfs_enumerate restricted to the root branches f with f % count == index
 * (the single-map case of the device root-task split, api.cu plan_search) */
int dfs_enumerate_shard(int n, const uint64_t *facets, int M, int64_t cap, int want_bits,
                        int shard_index, int shard_count, dfs_result *out) {
    g_shard_index = shard_index;
    g_shard_count = shard_count;
    const int rc = dfs_enumerate(n, facets, M, cap, 0, 0, 0, 0, want_bits, 0, M - 1 < 0 ? 0 : M, out);
    g_shard_index = 0;
    g_shard_count = 1;
    return rc;
}

int dfs_enumerate(int n, const uint64_t *facets, int M, int64_t cap, const int32_t *required,
                  int nreq, const int32_t *forbidden, int nforb, int want_bits, int root_lo,
                  int root_hi, dfs_result *out) {
    memset(out, 0, sizeof(*out));
    if (M <= 0) return 2;
    uint64_t *ridges = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)M * (size_t)n);
    int32_t *fr = (int32_t *)malloc(sizeof(int32_t) * (size_t)M * (size_t)n);
    int32_t *po = (int32_t *)malloc(sizeof(int32_t) * ((size_t)M * (size_t)n + 1));
    int32_t *pa = (int32_t *)malloc(sizeof(int32_t) * (size_t)M * (size_t)n);
    const int N = po_incidence(facets, M, ridges, M * n, fr, po, pa);
    if (N < 0) { free(ridges); free(fr); free(po); free(pa); return 2; }
    dfs_ctx c;
    memset(&c, 0, sizeof(c));
    c.n = n; c.M = M; c.N = N; c.W = (M + 63) / 64; c.cap = cap; c.fr = fr;
    c.rp = (int32_t *)malloc(sizeof(int32_t) * (size_t)N * 8);
    c.npar = (uint8_t *)calloc((size_t)N, 1);
    c.st = (uint8_t *)calloc((size_t)M, 1);
    c.cnt = (uint8_t *)calloc((size_t)N, 1);
    c.av = (uint8_t *)calloc((size_t)N, 1);
    c.trail = (int32_t *)malloc(sizeof(int32_t) * (size_t)(M + 1) * 2);
    c.want_bits = want_bits;
    for (int r = 0; r < N; ++r) {
        c.npar[r] = (uint8_t)(po[r + 1] - po[r]);
        for (int q = 0; q < c.npar[r]; ++q) c.rp[r * 8 + q] = pa[po[r] + q];
        c.av[r] = c.npar[r];
    }
    for (int i = 0; i < nforb; ++i)
        if (c.st[forbidden[i]] == ST_U) do_exclude(&c, forbidden[i]);
    int ok = 1;
    for (int i = 0; i < nreq && ok; ++i) {
        const int f = required[i];
        if (c.st[f] == ST_OUT) ok = 0;
        else if (c.st[f] == ST_U) do_include(&c, f);
    }
    if (ok && c.ndead) ok = 0;
    if (ok) {
        if (nreq > 0 || root_lo > 0 || root_hi < M || g_shard_count > 1) {
            if (nreq > 0) {
                search(&c);
            } else {
                /* root branches [root_lo, root_hi): minimum facet f */
                for (int f = 0; f < root_hi; ++f) {
                    if (c.st[f] != ST_U) continue;
                    if (f >= root_lo && f % g_shard_count == g_shard_index && (cap < 0 || n + 1 <= cap))
                        child(&c, f);
                    do_exclude(&c, f);
                }
            }
        } else {
            search(&c);
        }
    }
    out->count = c.count;
    out->nodes = c.nodes;
    out->words = c.W;
    if (want_bits && c.count > 1) {
        g_words = c.W;
        qsort(c.bits, (size_t)c.count, sizeof(uint64_t) * (size_t)c.W, cmp_bits);
    }
    out->bits = c.bits;
    free(c.rp); free(c.npar); free(c.st); free(c.cnt); free(c.av); free(c.trail);
    free(ridges); free(fr); free(po); free(pa);
    return 0;
}

void dfs_result_free(dfs_result *r) {
    if (r && r->bits) free(r->bits);
    if (r) r->bits = NULL;
}
