/*
 * tools/split_sim.c -- dev probe for the multi-GPU frontier split (not product,
 * not a test).  Runs the CPU restatement of the device search tree (same tree
 * as oracle/dfs_port.c / k3_search.cu: forced moves chained, frames only at
 * real branch points) and writes one line per branch item -- a child of a real
 * frame (the root's closed frame included) -- up to branch depth DMAX:
 *   id parent depth kind nodes
 * nodes = search nodes in the item's subtree (its own include included);
 * kind 0 = child of an OPEN frame, 1 = child of a CLOSED frame.
 * Usage: split_sim n map [dmax]  (IDCM orbit map index, UBT cap)
 * Build: gcc -O2 -o tools/split_sim tools/split_sim.c -Loracle -loracle
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../oracle/plseeds_port.h"

enum { U = 0, IN = 1, OUT = 2 };
static int n, M, N, cap, dmax;
static int32_t *fr, *rp;
static uint8_t *npar, *st, *cnt, *av;
static int size, nopen, ndead, ntr;
static int32_t *trail;
static long long nodes;
static long long nitems;
static FILE *fo;

static void dec_av(int r) {
    av[r]--;
    if (cnt[r] == 1 && av[r] == 0) ndead++;
}
static void exclude(int g) {
    st[g] = OUT;
    for (int k = 0; k < n; ++k) dec_av(fr[g * n + k]);
    trail[ntr++] = g << 1;
}
static void include(int f) {
    st[f] = IN;
    size++;
    trail[ntr++] = (f << 1) | 1;
    for (int k = 0; k < n; ++k) {
        const int r = fr[f * n + k];
        av[r]--;
        cnt[r]++;
        if (cnt[r] == 1) {
            nopen++;
            if (av[r] == 0) ndead++;
        } else
            nopen--;
    }
    for (int k = 0; k < n; ++k) {
        const int r = fr[f * n + k];
        if (cnt[r] != 2) continue;
        for (int q = 0; q < npar[r]; ++q) {
            const int g = rp[r * 8 + q];
            if (st[g] == U) exclude(g);
        }
    }
}
static void undo(int mark) {
    while (ntr > mark) {
        const int e = trail[--ntr], f = e >> 1;
        if (e & 1) {
            for (int k = 0; k < n; ++k) {
                const int r = fr[f * n + k];
                if (cnt[r] == 1) {
                    if (av[r] == 0) ndead--;
                    nopen--;
                } else
                    nopen++;
                cnt[r]--;
                av[r]++;
            }
            size--;
        } else {
            for (int k = 0; k < n; ++k) {
                const int r = fr[f * n + k];
                if (cnt[r] == 1 && av[r] == 0) ndead--;
                av[r]++;
            }
        }
        st[f] = U;
    }
}

static void search(long long parent, int depth);

static void child(int f, long long parent, int depth, int is_item, int kind) {
    const int mark = ntr;
    const long long n0 = nodes;
    long long id = parent;
    if (is_item && depth <= dmax) id = nitems++;
    include(f);
    nodes++;
    if (ndead == 0) search(id, depth + (is_item ? 1 : 0));
    undo(mark);
    if (is_item && depth <= dmax) fprintf(fo, "%lld %lld %d %d %lld\n", id, parent, depth, kind, nodes - n0);
}

static void search(long long parent, int depth) {
    const int mark = ntr;
    if (nopen == 0) {
        if (size + n + 1 > cap) return;
        for (int f = 0; f < M; ++f) {
            if (st[f] != U) continue;
            child(f, parent, depth, 1, 1);
            exclude(f);
        }
    } else {
        if (size + (nopen + n - 1) / n > cap) return;
        int best = -1, bav = 99;
        for (int r = 0; r < N; ++r)
            if (cnt[r] == 1 && av[r] < bav) {
                bav = av[r];
                best = r;
                if (bav <= 1) break;
            }
        const int real = bav >= 2;
        for (int q = 0; q < npar[best]; ++q) {
            const int u = rp[best * 8 + q];
            if (st[u] != U) continue;
            child(u, parent, depth, real, 0);
            exclude(u);
            if (ndead) break;
        }
    }
    undo(mark);
}

int main(int argc, char** argv) {
    if (argc < 3) return 1;
    n = atoi(argv[1]);
    const int map = atoi(argv[2]);
    dmax = argc > 3 ? atoi(argv[3]) : 6;
    const int p = 4, m = n + p;
    uint32_t rows[4096 * 16];
    const int K = po_idcm_orbits(n, p, rows, 4096);
    if (map >= K) return 1;
    uint32_t cols[16];
    po_charmap_of_dcm(m, p, rows + map * m, cols);
    uint64_t fac[4096];
    M = po_binary_matroid(n, m, cols, fac, 4096);
    cap = (int)po_cyclic_facet_bound(n);
    uint64_t* ridges = malloc(sizeof(uint64_t) * M * n);
    fr = malloc(sizeof(int32_t) * M * n);
    int32_t* po = malloc(sizeof(int32_t) * (M * n + 1));
    int32_t* pa = malloc(sizeof(int32_t) * M * n);
    N = po_incidence(fac, M, ridges, M * n, fr, po, pa);
    rp = malloc(sizeof(int32_t) * N * 8);
    npar = calloc(N, 1);
    st = calloc(M, 1);
    cnt = calloc(N, 1);
    av = calloc(N, 1);
    trail = malloc(sizeof(int32_t) * (M + 1) * 2);
    for (int r = 0; r < N; ++r) {
        npar[r] = po[r + 1] - po[r];
        for (int q = 0; q < npar[r]; ++q) rp[r * 8 + q] = pa[po[r] + q];
        av[r] = npar[r];
    }
    fo = stdout;
    search(-1, 0);
    fprintf(stderr, "n=%d map=%d M=%d N=%d nodes=%lld items=%lld\n", n, map, M, N, nodes, nitems);
    return 0;
}
