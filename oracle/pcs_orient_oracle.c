/*
 * pcs_orient_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement, in plain C11, of the reference's orientation step
 * (/root/reference/proj/include/pcstable/orient.hpp), SURVEY.md §8(f) row 1:
 *   find_v_structures  orient.hpp:40-89   (votes from every unshielded triple, an
 *                                           edge voted both ways stays undirected)
 *   meek_rule_1..4     orient.hpp:95-138
 *   apply_meek_rules   orient.hpp:147-167  (passes over the undirected edges in
 *                                           ascending order, (x,y) tried before (y,x),
 *                                           orientations visible within the pass)
 *   orient_skeleton    orient.hpp:170-173
 * The reference's std::set<pair> containers become a p x p byte matrix (membership)
 * plus an append-only list of directed pairs (the rules only ask "does some directed
 * edge exist with ...", so iteration order is irrelevant); the undirected edges of a
 * pass are snapshotted in ascending (x, y) order like the reference's vector copy.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "pcs_oracle.h"

typedef struct {
    int n;
    uint8_t* adj;   /* skeleton, n x n */
    uint8_t* dir;   /* dir[a*n+b]: a -> b */
    uint8_t* und;   /* und[a*n+b] = und[b*n+a]: a - b */
    int32_t* dl;    /* directed pairs (from, to), append-only */
    int64_t nd, capd;
} mixed;

static int has_dir(const mixed* g, int a, int b) { return g->dir[(int64_t)a * g->n + b]; }
static int has_und(const mixed* g, int a, int b) { return g->und[(int64_t)a * g->n + b]; }
static int adjacent(const mixed* g, int a, int b) { return has_und(g, a, b) || has_dir(g, a, b) || has_dir(g, b, a); }

static int add_dir(mixed* g, int a, int b) {
    if (g->nd == g->capd) {
        int64_t cap = g->capd ? g->capd * 2 : 64;
        int32_t* np = (int32_t*)realloc(g->dl, sizeof(int32_t) * 2 * (size_t)cap);
        if (!np) return ORC_ENOMEM;
        g->dl = np;
        g->capd = cap;
    }
    g->dl[2 * g->nd] = a;
    g->dl[2 * g->nd + 1] = b;
    ++g->nd;
    g->dir[(int64_t)a * g->n + b] = 1;
    return ORC_OK;
}

/* orient.hpp:95-101 */
static int rule1(const mixed* g, int a, int b) {
    for (int64_t e = 0; e < g->nd; ++e) {
        const int c = g->dl[2 * e], to = g->dl[2 * e + 1];
        if (to != a || c == b) continue;
        if (!adjacent(g, c, b)) return 1;
    }
    return 0;
}
/* orient.hpp:105-111 */
static int rule2(const mixed* g, int a, int b) {
    for (int64_t e = 0; e < g->nd; ++e) {
        const int from = g->dl[2 * e], c = g->dl[2 * e + 1];
        if (from != a) continue;
        if (has_dir(g, c, b)) return 1;
    }
    return 0;
}
/* orient.hpp:116-124 */
static int rule3(const mixed* g, int a, int b, int32_t* buf) {
    int64_t k = 0;
    for (int64_t e = 0; e < g->nd; ++e) {
        const int c = g->dl[2 * e], to = g->dl[2 * e + 1];
        if (to == b && has_und(g, a, c)) buf[k++] = c;
    }
    for (int64_t x = 0; x < k; ++x)
        for (int64_t y = x + 1; y < k; ++y)
            if (!adjacent(g, buf[x], buf[y])) return 1;
    return 0;
}
/* orient.hpp:129-138 */
static int rule4(const mixed* g, int a, int b) {
    for (int64_t e = 0; e < g->nd; ++e) {
        const int d = g->dl[2 * e], to = g->dl[2 * e + 1];
        if (to != b || d == a) continue;
        for (int64_t f = 0; f < g->nd; ++f) {
            const int c = g->dl[2 * f], mid = g->dl[2 * f + 1];
            if (mid != d || c == a || c == b) continue;
            if (adjacent(g, a, c) && !adjacent(g, c, b)) return 1;
        }
    }
    return 0;
}

static void mixed_free(mixed* g) {
    free(g->adj);
    free(g->dir);
    free(g->und);
    free(g->dl);
}

/* sepset of unordered pair {i, j} in the triangular layout of orc_result_sepsets / core.hpp:329-335 */
static int64_t slot_of(int n, int i, int j) {
    if (i > j) { int t = i; i = j; j = t; }
    return (int64_t)i * (2 * (int64_t)n - i - 1) / 2 + (j - i - 1);
}

/*
 * skeleton: n x n bytes (symmetric); sepsets: per triangular slot level (-1 = none) and offset
 * into members.  directed_in: optional pre-set directed pairs (for apply_meek_rules alone, with
 * stage = 2); stage bit 1 = find_v_structures, bit 2 = apply_meek_rules.
 * Outputs: directed pairs (ascending (from, to), the reference's std::set order) and undirected
 * pairs (ascending, from < to); *n_dir / *n_und receive the counts (buffers sized n*(n-1)/2 pairs).
 */
int orc_orient(int n, const uint8_t* skeleton, const int32_t* sep_level, const int64_t* sep_offset,
               const int32_t* members, int stage, const int32_t* directed_in, int64_t n_directed_in,
               int32_t* dir_out, int64_t* n_dir, int32_t* und_out, int64_t* n_und) {
    mixed g;
    memset(&g, 0, sizeof g);
    g.n = n;
    const size_t nn = (size_t)n * (size_t)n;
    g.adj = (uint8_t*)calloc(nn ? nn : 1, 1);
    g.dir = (uint8_t*)calloc(nn ? nn : 1, 1);
    g.und = (uint8_t*)calloc(nn ? nn : 1, 1);
    int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    if (!g.adj || !g.dir || !g.und || !buf) { mixed_free(&g); free(buf); return ORC_ENOMEM; }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) g.adj[(size_t)i * n + j] = (i != j) && skeleton[(size_t)i * n + j];
    int rc = ORC_OK;
    if (stage & 1) {
        /* find_v_structures: votes[i*n+k] = vote i -> k (orient.hpp:45-71) */
        uint8_t* votes = (uint8_t*)calloc(nn ? nn : 1, 1);
        if (!votes) { mixed_free(&g); free(buf); return ORC_ENOMEM; }
        for (int k = 0; k < n && rc == ORC_OK; ++k) {
            int32_t cnt = 0;
            for (int j = 0; j < n; ++j)
                if (g.adj[(size_t)k * n + j]) buf[cnt++] = j;
            for (int a = 0; a < cnt && rc == ORC_OK; ++a)
                for (int b = a + 1; b < cnt; ++b) {
                    const int i = buf[a], j = buf[b];
                    if (g.adj[(size_t)i * n + j]) continue;
                    const int64_t s = slot_of(n, i, j);
                    if (sep_level[s] < 0) {
                        rc = ORC_EINVAL;  /* nonadjacent but has no separating set (orient.hpp:60-63) */
                        break;
                    }
                    int contains = 0;
                    for (int q = 0; q < sep_level[s]; ++q) contains |= members[sep_offset[s] + q] == k;
                    if (!contains) {
                        votes[(size_t)i * n + k] = 1;
                        votes[(size_t)j * n + k] = 1;
                    }
                }
        }
        if (rc == ORC_OK)
            for (int i = 0; i < n && rc == ORC_OK; ++i)
                for (int j = i + 1; j < n; ++j) {
                    if (!g.adj[(size_t)i * n + j]) continue;
                    const int fwd = votes[(size_t)i * n + j], rev = votes[(size_t)j * n + i];
                    if (fwd && !rev) rc = add_dir(&g, i, j);
                    else if (rev && !fwd) rc = add_dir(&g, j, i);
                    else g.und[(size_t)i * n + j] = g.und[(size_t)j * n + i] = 1;
                    if (rc) break;
                }
        free(votes);
    } else {
        /* caller-provided mixed graph: directed_in pairs, every other skeleton edge undirected */
        for (int64_t e = 0; e < n_directed_in && rc == ORC_OK; ++e)
            rc = add_dir(&g, directed_in[2 * e], directed_in[2 * e + 1]);
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j)
                if (g.adj[(size_t)i * n + j] && !has_dir(&g, i, j) && !has_dir(&g, j, i))
                    g.und[(size_t)i * n + j] = g.und[(size_t)j * n + i] = 1;
    }
    if (rc == ORC_OK && (stage & 2)) {
        /* apply_meek_rules (orient.hpp:147-167) */
        int32_t* edges = (int32_t*)malloc(sizeof(int32_t) * 2 * (nn / 2 + 1));
        if (!edges) rc = ORC_ENOMEM;
        int changed = 1;
        while (rc == ORC_OK && changed) {
            changed = 0;
            int64_t ne = 0;
            for (int x = 0; x < n; ++x)
                for (int y = x + 1; y < n; ++y)
                    if (has_und(&g, x, y)) { edges[2 * ne] = x; edges[2 * ne + 1] = y; ++ne; }
            for (int64_t e = 0; e < ne && rc == ORC_OK; ++e) {
                const int x = edges[2 * e], y = edges[2 * e + 1];
                if (!has_und(&g, x, y)) continue;
                for (int d = 0; d < 2; ++d) {
                    const int a = d ? y : x, b = d ? x : y;
                    if (rule1(&g, a, b) || rule2(&g, a, b) || rule3(&g, a, b, buf) || rule4(&g, a, b)) {
                        g.und[(size_t)x * n + y] = g.und[(size_t)y * n + x] = 0;
                        rc = add_dir(&g, a, b);
                        changed = 1;
                        break;
                    }
                }
            }
        }
        free(edges);
    }
    if (rc == ORC_OK) {
        int64_t nd = 0, nu = 0;
        for (int a = 0; a < n; ++a)
            for (int b = 0; b < n; ++b) {
                if (has_dir(&g, a, b)) { dir_out[2 * nd] = a; dir_out[2 * nd + 1] = b; ++nd; }
                if (a < b && has_und(&g, a, b)) { und_out[2 * nu] = a; und_out[2 * nu + 1] = b; ++nu; }
            }
        *n_dir = nd;
        *n_und = nu;
    }
    mixed_free(&g);
    free(buf);
    return rc;
}
