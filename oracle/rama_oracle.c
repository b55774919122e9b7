/*
 * rama_oracle.c -- CPU restatement of the reference `parcut` hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 kernels and the CPU baseline timed by bench.py.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
 * may load it.  The product package never links or calls it.
 *
 * Every function restates one reference routine (file:line into
 * /root/reference/pkg/src/parcut/) in plain single-threaded C with the
 * reference's exact tie-breaks and fp64 summation orders:
 *   - numpy `x.sum()`            == pairwise(x)               (np_sum)
 *   - numpy `add.reduceat` seg   == x[0] + pairwise(x[1:])    (seg_sum)
 *   - numpy `bincount(weights)`  == sequential per bin in input order
 * (both checked against numpy in tests/test_oracle.py).
 *
 * Node ids and counts are int64 like the reference; costs are double.
 * Functions return 0 on success, a negative code on invalid input:
 *   -1 self-loop, -2 endpoint out of range, -3 bad argument, -4 no memory.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef int64_t i64;
typedef uint64_t u64;

#define ORC_OK 0
#define ORC_SELF_LOOP (-1)
#define ORC_RANGE (-2)
#define ORC_ARG (-3)
#define ORC_NOMEM (-4)

static void *xmalloc(size_t bytes) { return malloc(bytes ? bytes : 1); }
static void *xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s ? s : 1); }

/* ------------------------------------------------------------------ sums */

/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
 * PW_BLOCKSIZE 128, 8-way unrolled leaves). */
static double pairwise(const double *a, i64 n) {
    if (n < 8) {
        double r = -0.0;  /* numpy 2.x starts the short sum at -0.0 (keeps -0.0 sums) */
        for (i64 i = 0; i < n; i++) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        i64 i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    i64 n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
}

/* np.sum(x) for a 1-D float64 array */
double orc_np_sum(const double *a, i64 n) { return pairwise(a, n); }

/* one segment of np.add.reduceat */
double orc_seg_sum(const double *a, i64 n) {
    if (n <= 0) return 0.0;
    return a[0] + pairwise(a + 1, n - 1);
}

/* ------------------------------------------------------------ radix sort */

/* Stable LSD radix sort of (key, val) pairs on the low `bits` key bits.
 * Stability makes it equivalent to numpy lexsort/argsort(kind=stable). */
static int radix_sort_kv(u64 *key, i64 *val, i64 n, int bits) {
    if (n <= 1 || bits <= 0) return ORC_OK;
    u64 *k2 = (u64 *)xmalloc(sizeof(u64) * n);
    i64 *v2 = (i64 *)xmalloc(sizeof(i64) * n);
    if (!k2 || !v2) { free(k2); free(v2); return ORC_NOMEM; }
    const int D = 11, B = 1 << D;
    i64 *cnt = (i64 *)xmalloc(sizeof(i64) * B);
    u64 *ks = key, *kd = k2;
    i64 *vs = val, *vd = v2;
    for (int sh = 0; sh < bits; sh += D) {
        memset(cnt, 0, sizeof(i64) * B);
        for (i64 i = 0; i < n; i++) cnt[(ks[i] >> sh) & (B - 1)]++;
        i64 s = 0;
        for (int b = 0; b < B; b++) { i64 c = cnt[b]; cnt[b] = s; s += c; }
        for (i64 i = 0; i < n; i++) {
            i64 p = cnt[(ks[i] >> sh) & (B - 1)]++;
            kd[p] = ks[i];
            vd[p] = vs[i];
        }
        u64 *tk = ks; ks = kd; kd = tk;
        i64 *tv = vs; vs = vd; vd = tv;
    }
    if (ks != key) {
        memcpy(key, ks, sizeof(u64) * n);
        memcpy(val, vs, sizeof(i64) * n);
    }
    free(k2); free(v2); free(cnt);
    return ORC_OK;
}

static int bits_for(i64 n) {
    int b = 1;
    while (b < 63 && ((i64)1 << b) < n) b++;
    return b;
}

/* permutation sorting pairs (a[i], b[i]) lexicographically, stable.
 * a, b in [0, n). */
static i64 *lex_perm2(const i64 *a, const i64 *b, i64 m, i64 n) {
    i64 *perm = (i64 *)xmalloc(sizeof(i64) * m);
    u64 *key = (u64 *)xmalloc(sizeof(u64) * m);
    if (!perm || !key) { free(perm); free(key); return NULL; }
    int nb = bits_for(n);
    for (i64 i = 0; i < m; i++) perm[i] = i;
    if (2 * nb <= 64) {
        for (i64 i = 0; i < m; i++) key[i] = ((u64)a[i] << nb) | (u64)b[i];
        radix_sort_kv(key, perm, m, 2 * nb);
    } else {
        for (i64 i = 0; i < m; i++) key[i] = (u64)b[i];
        radix_sort_kv(key, perm, m, nb);
        for (i64 i = 0; i < m; i++) key[i] = (u64)a[perm[i]];
        radix_sort_kv(key, perm, m, nb);
    }
    free(key);
    return perm;
}

/* ------------------------------------------------------------- graph ops */

/* WeightedGraph.__init__ canonicalisation (graph.py:29-57): validate,
 * orient u<v, stable lexsort by (lo, hi), sum parallel edges with the
 * reduceat order.  Outputs sized m; *m_out receives the unique count. */
int orc_canonicalize(i64 n, i64 m, const i64 *u, const i64 *v, const double *c,
                     i64 *ou, i64 *ov, double *oc, i64 *m_out) {
    *m_out = 0;
    if (n < 0) return ORC_ARG;
    for (i64 i = 0; i < m; i++)
        if (u[i] == v[i]) return ORC_SELF_LOOP;
    for (i64 i = 0; i < m; i++)
        if (u[i] < 0 || v[i] < 0 || u[i] >= n || v[i] >= n) return ORC_RANGE;
    if (m == 0) return ORC_OK;
    i64 *lo = (i64 *)xmalloc(sizeof(i64) * m), *hi = (i64 *)xmalloc(sizeof(i64) * m);
    for (i64 i = 0; i < m; i++) {
        lo[i] = u[i] < v[i] ? u[i] : v[i];
        hi[i] = u[i] < v[i] ? v[i] : u[i];
    }
    i64 *perm = lex_perm2(lo, hi, m, n);
    double *cs = (double *)xmalloc(sizeof(double) * m);
    for (i64 i = 0; i < m; i++) cs[i] = c[perm[i]];
    i64 k = 0, s = 0;
    for (i64 i = 1; i <= m; i++) {
        if (i == m || lo[perm[i]] != lo[perm[s]] || hi[perm[i]] != hi[perm[s]]) {
            ou[k] = lo[perm[s]];
            ov[k] = hi[perm[s]];
            oc[k] = orc_seg_sum(cs + s, i - s);
            k++;
            s = i;
        }
    }
    *m_out = k;
    free(lo); free(hi); free(perm); free(cs);
    return ORC_OK;
}

/* clustering_cost (graph.py:134-145): np.sum over cut edges' costs */
double orc_clustering_cost(i64 m, const i64 *u, const i64 *v, const double *c,
                           const i64 *labels) {
    double *buf = (double *)xmalloc(sizeof(double) * (m ? m : 1));
    i64 k = 0;
    for (i64 i = 0; i < m; i++)
        if (labels[u[i]] != labels[v[i]]) buf[k++] = c[i];
    double r = pairwise(buf, k);
    free(buf);
    return r;
}

/* --------------------------------------------------------- contraction */

/* connected_components (contraction.py:68-111): union-find toward the
 * smaller id with path halving, then canonical ids = rank of the root
 * (the component minimum) among all roots. */
int orc_components(i64 n, i64 k, const i64 *su, const i64 *sv, i64 *map, i64 *num_targets) {
    for (i64 i = 0; i < k; i++)
        if (su[i] < 0 || sv[i] < 0 || su[i] >= n || sv[i] >= n) return ORC_RANGE;
    i64 *p = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    for (i64 x = 0; x < n; x++) p[x] = x;
    for (i64 i = 0; i < k; i++) {
        i64 a = su[i], b = sv[i];
        while (p[a] != a) { p[a] = p[p[a]]; a = p[a]; }
        while (p[b] != b) { p[b] = p[p[b]]; b = p[b]; }
        if (a < b) p[b] = a;
        else if (b < a) p[a] = b;
    }
    i64 t = 0;
    for (i64 x = 0; x < n; x++) {
        i64 r = x;
        while (p[r] != r) r = p[r];
        p[x] = r;
        if (r == x) map[x] = t++;
        else map[x] = map[r]; /* r < x already numbered */
    }
    *num_targets = t;
    free(p);
    return ORC_OK;
}

/* contract_graph (contraction.py:142-163): relabel, drop merged edges into
 * joined (np.sum order), orient, stable lexsort, reduceat. */
int orc_contract(i64 n, i64 m, const i64 *u, const i64 *v, const double *c,
                 const i64 *map, i64 n_targets, i64 *ou, i64 *ov, double *oc,
                 i64 *m_out, double *joined) {
    (void)n;
    double *jb = (double *)xmalloc(sizeof(double) * (m ? m : 1));
    i64 *lo = (i64 *)xmalloc(sizeof(i64) * (m ? m : 1));
    i64 *hi = (i64 *)xmalloc(sizeof(i64) * (m ? m : 1));
    double *kc = (double *)xmalloc(sizeof(double) * (m ? m : 1));
    i64 nj = 0, nk = 0;
    for (i64 i = 0; i < m; i++) {
        i64 fu = map[u[i]], fv = map[v[i]];
        if (fu == fv) { jb[nj++] = c[i]; continue; }
        lo[nk] = fu < fv ? fu : fv;
        hi[nk] = fu < fv ? fv : fu;
        kc[nk] = c[i];
        nk++;
    }
    *joined = pairwise(jb, nj);
    i64 k = 0;
    if (nk) {
        i64 *perm = lex_perm2(lo, hi, nk, n_targets > 0 ? n_targets : 1);
        double *cs = (double *)xmalloc(sizeof(double) * nk);
        for (i64 i = 0; i < nk; i++) cs[i] = kc[perm[i]];
        i64 s = 0;
        for (i64 i = 1; i <= nk; i++) {
            if (i == nk || lo[perm[i]] != lo[perm[s]] || hi[perm[i]] != hi[perm[s]]) {
                ou[k] = lo[perm[s]];
                ov[k] = hi[perm[s]];
                oc[k] = orc_seg_sum(cs + s, i - s);
                k++;
                s = i;
            }
        }
        free(perm); free(cs);
    }
    *m_out = k;
    free(jb); free(lo); free(hi); free(kc);
    return ORC_OK;
}

/* select_max_edge (contraction.py:166-176) */
int orc_max_edge(i64 m, const double *c, i64 *idx) {
    i64 best = -1;
    for (i64 i = 0; i < m; i++)
        if (c[i] > 0.0 && (best < 0 || c[i] > c[best])) best = i;
    *idx = best;
    return ORC_OK;
}

/* select_matching (contraction.py:179-228): up to `rounds` handshake
 * rounds; a node targets its live positive neighbour of maximum cost, ties
 * toward the smaller neighbour id; mutual pairs (recorded with u<v) are
 * matched.  Output sorted by u (each node is in at most one pair). */
int orc_matching(i64 n, i64 m, const i64 *u, const i64 *v, const double *c, int rounds,
                 i64 *out_u, i64 *out_v, i64 *k_out) {
    char *matched = (char *)xcalloc(n, 1);
    i64 *tgt = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    double *bc = (double *)xmalloc(sizeof(double) * (n ? n : 1));
    i64 *partner = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    for (i64 x = 0; x < n; x++) partner[x] = -1;
    for (int r = 0; r < rounds; r++) {
        for (i64 x = 0; x < n; x++) tgt[x] = -1;
        i64 live = 0;
        for (i64 i = 0; i < m; i++) {
            if (!(c[i] > 0.0) || matched[u[i]] || matched[v[i]]) continue;
            live++;
            for (int side = 0; side < 2; side++) {
                i64 a = side ? v[i] : u[i], b = side ? u[i] : v[i];
                if (tgt[a] < 0 || c[i] > bc[a] || (c[i] == bc[a] && b < tgt[a])) {
                    tgt[a] = b;
                    bc[a] = c[i];
                }
            }
        }
        if (!live) break;
        i64 added = 0;
        for (i64 x = 0; x < n; x++) {
            i64 t = tgt[x];
            if (t >= 0 && x < t && tgt[t] == x) {
                partner[x] = t;
                added++;
            }
        }
        if (!added) break;
        for (i64 x = 0; x < n; x++)
            if (partner[x] >= 0 && !matched[x]) { matched[x] = 1; matched[partner[x]] = 1; }
    }
    i64 k = 0;
    for (i64 x = 0; x < n; x++)
        if (partner[x] > x) { out_u[k] = x; out_v[k] = partner[x]; k++; }
    *k_out = k;
    free(matched); free(tgt); free(bc); free(partner);
    return ORC_OK;
}

/* strict forest order (contraction.py:304): cost desc, then u asc, v asc */
typedef struct { double c; i64 u, v; } edge_t;
static int cmp_forest(const void *pa, const void *pb) {
    const edge_t *a = (const edge_t *)pa, *b = (const edge_t *)pb;
    if (a->c > b->c) return -1;
    if (a->c < b->c) return 1;
    if (a->u != b->u) return a->u < b->u ? -1 : 1;
    if (a->v != b->v) return a->v < b->v ? -1 : 1;
    return 0;
}

static i64 uf_find(i64 *p, i64 x) {
    while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
    return x;
}

/* select_spanning_forest_no_conflicts (contraction.py:287-366).
 * The Boruvka loop (309-327) under a strict total order yields the unique
 * maximum spanning forest, restated here as Kruskal.  The conflict pass
 * (_remove_conflict_edges, 231-284) is literal: repulsive edges in
 * ascending (u, v) order, BFS in the pruned forest, cut the cheapest path
 * edge (ties lexicographically smallest). */
int orc_forest(i64 n, i64 m, const i64 *u, const i64 *v, const double *c,
               i64 *out_u, i64 *out_v, i64 *k_out) {
    *k_out = 0;
    i64 mp = 0;
    for (i64 i = 0; i < m; i++) mp += c[i] > 0.0;
    if (!mp) return ORC_OK;
    edge_t *pe = (edge_t *)xmalloc(sizeof(edge_t) * mp);
    mp = 0;
    for (i64 i = 0; i < m; i++)
        if (c[i] > 0.0) { pe[mp].c = c[i]; pe[mp].u = u[i]; pe[mp].v = v[i]; mp++; }
    qsort(pe, mp, sizeof(edge_t), cmp_forest);
    i64 *p = (i64 *)xmalloc(sizeof(i64) * n);
    for (i64 x = 0; x < n; x++) p[x] = x;
    edge_t *fe = (edge_t *)xmalloc(sizeof(edge_t) * mp);
    i64 k = 0;
    for (i64 i = 0; i < mp; i++) {
        i64 a = uf_find(p, pe[i].u), b = uf_find(p, pe[i].v);
        if (a == b) continue;
        if (a < b) p[b] = a; else p[a] = b;
        fe[k++] = pe[i];
    }
    free(pe);
    char *removed = (char *)xcalloc(k, 1);
    /* forest adjacency */
    i64 *deg = (i64 *)xcalloc(n + 1, sizeof(i64));
    for (i64 e = 0; e < k; e++) { deg[fe[e].u + 1]++; deg[fe[e].v + 1]++; }
    for (i64 x = 0; x < n; x++) deg[x + 1] += deg[x];
    i64 *fill = (i64 *)xmalloc(sizeof(i64) * n);
    memcpy(fill, deg, sizeof(i64) * n);
    i64 *nbr = (i64 *)xmalloc(sizeof(i64) * 2 * (k ? k : 1));
    i64 *eid = (i64 *)xmalloc(sizeof(i64) * 2 * (k ? k : 1));
    for (i64 e = 0; e < k; e++) {
        i64 a = fe[e].u, b = fe[e].v;
        nbr[fill[a]] = b; eid[fill[a]++] = e;
        nbr[fill[b]] = a; eid[fill[b]++] = e;
    }
    i64 *stamp = (i64 *)xcalloc(n, sizeof(i64));
    i64 *pedge = (i64 *)xmalloc(sizeof(i64) * n);
    i64 *queue = (i64 *)xmalloc(sizeof(i64) * n);
    /* repulsive edges are visited in the canonical (u, v) order of g */
    i64 tick = 0;
    for (i64 i = 0; i < m && k; i++) {
        if (!(c[i] < 0.0)) continue;
        i64 a = u[i], b = v[i];
        /* skip quickly when the endpoints were never in one tree */
        if (uf_find(p, a) != uf_find(p, b)) continue;
        tick++;
        i64 head = 0, tail = 0;
        queue[tail++] = a;
        stamp[a] = tick;
        int found = 0;
        while (head < tail && !found) {
            i64 x = queue[head++];
            for (i64 q = deg[x]; q < deg[x + 1]; q++) {
                i64 e = eid[q];
                if (removed[e]) continue;
                i64 y = nbr[q];
                if (stamp[y] == tick) continue;
                stamp[y] = tick;
                pedge[y] = e;
                if (y == b) { found = 1; break; }
                queue[tail++] = y;
            }
        }
        if (!found) continue;
        i64 best = -1, x = b;
        while (x != a) {
            i64 e = pedge[x];
            if (best < 0 || fe[e].c < fe[best].c ||
                (fe[e].c == fe[best].c &&
                 (fe[e].u < fe[best].u || (fe[e].u == fe[best].u && fe[e].v < fe[best].v))))
                best = e;
            x = (fe[e].v == x) ? fe[e].u : fe[e].v;
        }
        removed[best] = 1;
    }
    /* output sorted by (u, v) */
    i64 nk = 0;
    i64 *ku = (i64 *)xmalloc(sizeof(i64) * (k ? k : 1)), *kv = (i64 *)xmalloc(sizeof(i64) * (k ? k : 1));
    for (i64 e = 0; e < k; e++)
        if (!removed[e]) { ku[nk] = fe[e].u; kv[nk] = fe[e].v; nk++; }
    if (nk) {
        i64 *perm = lex_perm2(ku, kv, nk, n);
        for (i64 i = 0; i < nk; i++) { out_u[i] = ku[perm[i]]; out_v[i] = kv[perm[i]]; }
        free(perm);
    }
    *k_out = nk;
    free(ku); free(kv); free(p); free(fe); free(removed); free(deg); free(fill);
    free(nbr); free(eid); free(stamp); free(pedge); free(queue);
    return ORC_OK;
}

/* --------------------------------------------------------------- dual */

/* _positive_csr (dual.py:155-166) + _bfs_paths (dual.py:109-152): one
 * hop-shortest conflicted cycle per repulsive edge (ascending (u, v)),
 * BFS from the smaller endpoint expanding neighbours in ascending id
 * order, depth <= L-1.  out_len[q] = 0 when none.  Rows are width L. */
int orc_separate(i64 n, i64 m, const i64 *u, const i64 *v, const double *c, int L,
                 i64 *out_len, i64 *out_nodes, i64 *num_neg) {
    if (L < 3) return ORC_ARG;
    i64 nn = 0, np_ = 0;
    for (i64 i = 0; i < m; i++) { nn += c[i] < 0.0; np_ += c[i] > 0.0; }
    *num_neg = nn;
    for (i64 q = 0; q < nn; q++) {
        out_len[q] = 0;
        for (int j = 0; j < L; j++) out_nodes[q * L + j] = 0;
    }
    if (!nn || !np_) return ORC_OK;
    /* symmetric CSR of E+ sorted by (head, tail): the canonical edge order
     * already sorts (u -> v) by v within u; merge both directions. */
    i64 *heads = (i64 *)xmalloc(sizeof(i64) * 2 * np_), *tails = (i64 *)xmalloc(sizeof(i64) * 2 * np_);
    i64 t = 0;
    for (i64 i = 0; i < m; i++)
        if (c[i] > 0.0) { heads[t] = u[i]; tails[t] = v[i]; t++; heads[t] = v[i]; tails[t] = u[i]; t++; }
    i64 *perm = lex_perm2(heads, tails, 2 * np_, n);
    i64 *adj = (i64 *)xmalloc(sizeof(i64) * 2 * np_);
    i64 *ptr = (i64 *)xcalloc(n + 1, sizeof(i64));
    for (i64 i = 0; i < 2 * np_; i++) { adj[i] = tails[perm[i]]; ptr[heads[i] + 1]++; }
    for (i64 x = 0; x < n; x++) ptr[x + 1] += ptr[x];
    free(perm); free(heads); free(tails);
    i64 *stamp = (i64 *)xcalloc(n, sizeof(i64));
    i64 *dist = (i64 *)xcalloc(n, sizeof(i64));
    i64 *par = (i64 *)xmalloc(sizeof(i64) * n);
    i64 *queue = (i64 *)xmalloc(sizeof(i64) * n);
    i64 q = 0, tick = 0;
    for (i64 i = 0; i < m; i++) {
        if (!(c[i] < 0.0)) continue;
        i64 a = u[i], b = v[i];
        tick++;
        i64 head = 0, tail = 0;
        queue[tail++] = a;
        stamp[a] = tick;
        dist[a] = 0;
        par[a] = -1;
        int found = 0;
        while (head < tail && !found) {
            i64 x = queue[head++];
            if (dist[x] >= L - 1) break;
            for (i64 p = ptr[x]; p < ptr[x + 1]; p++) {
                i64 y = adj[p];
                if (stamp[y] == tick) continue;
                stamp[y] = tick;
                dist[y] = dist[x] + 1;
                par[y] = x;
                if (y == b) { found = 1; break; }
                queue[tail++] = y;
            }
        }
        if (found) {
            i64 len = dist[b] + 1, x = b;
            out_len[q] = len;
            for (i64 j = len - 1; j >= 0; j--) { out_nodes[q * L + j] = x; x = par[x]; }
        }
        q++;
    }
    free(adj); free(ptr); free(stamp); free(dist); free(par); free(queue);
    return ORC_OK;
}

/* lexicographic dedupe of rows (dual.py:216-225) for width-3 rows */
static i64 dedupe3(i64 *rows, i64 cnt, i64 n) {
    if (!cnt) return 0;
    i64 *perm = (i64 *)xmalloc(sizeof(i64) * cnt);
    u64 *key = (u64 *)xmalloc(sizeof(u64) * cnt);
    int nb = bits_for(n);
    for (i64 i = 0; i < cnt; i++) perm[i] = i;
    for (int col = 2; col >= 0; col--) {
        for (i64 i = 0; i < cnt; i++) key[i] = (u64)rows[perm[i] * 3 + col];
        radix_sort_kv(key, perm, cnt, nb);
    }
    i64 *tmp = (i64 *)xmalloc(sizeof(i64) * 3 * cnt);
    i64 k = 0;
    for (i64 i = 0; i < cnt; i++) {
        const i64 *r = rows + perm[i] * 3;
        if (k && tmp[(k - 1) * 3] == r[0] && tmp[(k - 1) * 3 + 1] == r[1] && tmp[(k - 1) * 3 + 2] == r[2])
            continue;
        tmp[k * 3] = r[0]; tmp[k * 3 + 1] = r[1]; tmp[k * 3 + 2] = r[2];
        k++;
    }
    memcpy(rows, tmp, sizeof(i64) * 3 * k);
    free(perm); free(key); free(tmp);
    return k;
}

static void sort3(i64 *r) {
    i64 t;
    if (r[0] > r[1]) { t = r[0]; r[0] = r[1]; r[1] = t; }
    if (r[1] > r[2]) { t = r[1]; r[1] = r[2]; r[2] = t; }
    if (r[0] > r[1]) { t = r[0]; r[0] = r[1]; r[1] = t; }
}

/* binary search of key (a, b) in canonical sorted edge arrays */
static i64 find_edge(const i64 *eu, const i64 *ev, i64 m, i64 a, i64 b) {
    i64 lo = 0, hi = m;
    while (lo < hi) {
        i64 mid = (lo + hi) / 2;
        if (eu[mid] < a || (eu[mid] == a && ev[mid] < b)) lo = mid + 1;
        else hi = mid;
    }
    if (lo < m && eu[lo] == a && ev[lo] == b) return lo;
    return -1;
}

/* _fan_arrays + _triangulate_arrays (dual.py:228-290).
 * Input: canonical graph, cycle rows (count rows, width L).
 * Output (caller-sized): aug_u/aug_v/base [m + C], tri_nodes/tri_edges
 * [T*3], coverage [m + C].  Augmented edges = originals then new chords in
 * ascending order. */
int orc_triangulate(i64 n, i64 m, const i64 *u, const i64 *v, const double *c,
                    i64 rows, int L, const i64 *lengths, const i64 *nodes,
                    i64 *aug_u, i64 *aug_v, double *base, i64 *m_aug,
                    i64 *tri_nodes, i64 *tri_edges, i64 *T_out, i64 *coverage) {
    i64 ntri = 0, nch = 0;
    for (i64 r = 0; r < rows; r++)
        if (lengths[r] >= 3) { ntri += lengths[r] - 2; nch += lengths[r] - 3; }
    i64 *tri = (i64 *)xmalloc(sizeof(i64) * 3 * (ntri ? ntri : 1));
    i64 *chu = (i64 *)xmalloc(sizeof(i64) * (nch ? nch : 1));
    i64 *chv = (i64 *)xmalloc(sizeof(i64) * (nch ? nch : 1));
    i64 t = 0, h = 0;
    for (i64 r = 0; r < rows; r++) {
        i64 l = lengths[r];
        if (l < 3) continue;
        const i64 *row = nodes + r * L;
        for (i64 j = 1; j < l - 1; j++) {
            tri[t * 3] = row[0]; tri[t * 3 + 1] = row[j]; tri[t * 3 + 2] = row[j + 1];
            sort3(tri + t * 3);
            t++;
        }
        for (i64 j = 2; j < l - 1; j++) {
            chu[h] = row[0] < row[j] ? row[0] : row[j];
            chv[h] = row[0] < row[j] ? row[j] : row[0];
            h++;
        }
    }
    i64 T = dedupe3(tri, t, n);
    /* chords: sort, dedupe, drop the ones already in E */
    i64 nc = 0;
    i64 *cu = (i64 *)xmalloc(sizeof(i64) * (h ? h : 1)), *cv = (i64 *)xmalloc(sizeof(i64) * (h ? h : 1));
    if (h) {
        i64 *perm = lex_perm2(chu, chv, h, n);
        for (i64 i = 0; i < h; i++) {
            i64 a = chu[perm[i]], b = chv[perm[i]];
            if (i && a == chu[perm[i - 1]] && b == chv[perm[i - 1]]) continue;
            if (find_edge(u, v, m, a, b) >= 0) continue;
            cu[nc] = a; cv[nc] = b; nc++;
        }
        free(perm);
    }
    for (i64 i = 0; i < m; i++) { aug_u[i] = u[i]; aug_v[i] = v[i]; base[i] = c[i]; }
    for (i64 i = 0; i < nc; i++) { aug_u[m + i] = cu[i]; aug_v[m + i] = cv[i]; base[m + i] = 0.0; }
    *m_aug = m + nc;
    for (i64 e = 0; e < m + nc; e++) coverage[e] = 0;
    for (i64 i = 0; i < T; i++) {
        i64 a = tri[i * 3], b = tri[i * 3 + 1], d = tri[i * 3 + 2];
        i64 pr[3][2] = {{a, b}, {a, d}, {b, d}};
        tri_nodes[i * 3] = a; tri_nodes[i * 3 + 1] = b; tri_nodes[i * 3 + 2] = d;
        for (int s = 0; s < 3; s++) {
            i64 e = find_edge(u, v, m, pr[s][0], pr[s][1]);
            if (e < 0) {
                e = find_edge(cu, cv, nc, pr[s][0], pr[s][1]);
                if (e < 0) { free(tri); free(chu); free(chv); free(cu); free(cv); return ORC_ARG; }
                e += m;
            }
            tri_edges[i * 3 + s] = e;
            coverage[e]++;
        }
    }
    *T_out = T;
    free(tri); free(chu); free(chv); free(cu); free(cv);
    return ORC_OK;
}

/* reparametrized_edge_costs (dual.py:309-316): base + bincount(lam) */
void orc_reparam(i64 m_aug, const double *base, i64 T, const i64 *tri_edges,
                 const double *lam, double *cl) {
    double *acc = (double *)xcalloc(m_aug, sizeof(double));
    for (i64 s = 0; s < 3 * T; s++) acc[tri_edges[s]] += lam[s];
    for (i64 e = 0; e < m_aug; e++) cl[e] = base[e] + acc[e];
    free(acc);
}

/* _slot_marginals (dual.py:319-336) on one triplet */
static double slot_marginal(const double *l, int slot) {
    double c110 = -(l[0] + l[1]);
    double c101 = -(l[0] + l[2]);
    double c011 = -(l[1] + l[2]);
    double c111 = -(l[0] + l[1] + l[2]);
    double a, b, z;
    if (slot == 0) { a = c110 < c101 ? c110 : c101; b = c111; z = c011; }
    else if (slot == 1) { a = c110 < c011 ? c110 : c011; b = c111; z = c101; }
    else { a = c101 < c011 ? c101 : c011; b = c111; z = c110; }
    double mn = a < b ? a : b;
    double zz = 0.0 < z ? 0.0 : z;
    return mn - zz;
}

/* message_passing_iteration (dual.py:358-392), `iters` times */
void orc_mp(i64 m_aug, const double *base, const i64 *coverage, i64 T, const i64 *tri_edges,
            double *lam, int iters) {
    static const int sched_slot[6] = {0, 1, 2, 0, 1, 0};
    static const double sched_w[6] = {1.0 / 3.0, 0.5, 1.0, 0.5, 1.0, 1.0};
    if (!T) return;
    double *cl = (double *)xmalloc(sizeof(double) * (m_aug ? m_aug : 1));
    for (int it = 0; it < iters; it++) {
        orc_reparam(m_aug, base, T, tri_edges, lam, cl);
        for (i64 s = 0; s < 3 * T; s++) {
            i64 e = tri_edges[s];
            lam[s] = lam[s] - cl[e] / (double)coverage[e];
        }
        for (i64 t = 0; t < T; t++) {
            double *l = lam + 3 * t;
            for (int k = 0; k < 6; k++) {
                double mm = slot_marginal(l, sched_slot[k]);
                volatile double w = sched_w[k] * mm; /* no FMA contraction */
                l[sched_slot[k]] = l[sched_slot[k]] + w;
            }
        }
    }
    free(cl);
}

/* lower_bound (dual.py:395-405) */
double orc_lower_bound(i64 m_aug, const double *base, i64 T, const i64 *tri_edges,
                       const double *lam) {
    double *cl = (double *)xmalloc(sizeof(double) * (m_aug ? m_aug : 1));
    orc_reparam(m_aug, base, T, tri_edges, lam, cl);
    for (i64 e = 0; e < m_aug; e++) cl[e] = cl[e] < 0.0 ? cl[e] : 0.0;
    double total = pairwise(cl, m_aug);
    if (T) {
        double *tm = (double *)xmalloc(sizeof(double) * T);
        for (i64 t = 0; t < T; t++) {
            const double *l = lam + 3 * t;
            double c110 = -(l[0] + l[1]), c101 = -(l[0] + l[2]);
            double c011 = -(l[1] + l[2]), c111 = -(l[0] + l[1] + l[2]);
            double a = c110 < c101 ? c110 : c101;
            double b = c011 < c111 ? c011 : c111;
            double x = a < b ? a : b;
            tm[t] = x < 0.0 ? x : 0.0;
        }
        total += pairwise(tm, T);
        free(tm);
    }
    free(cl);
    return total;
}

/* ----------------------------------------------------------------- GAEC */

typedef struct { double negc; i64 a, b; } hent_t;
static int hless(const hent_t *x, const hent_t *y) {
    if (x->negc != y->negc) return x->negc < y->negc;
    if (x->a != y->a) return x->a < y->a;
    return x->b < y->b;
}
typedef struct { hent_t *d; i64 n, cap; } heap_t;
static void hpush(heap_t *h, hent_t e) {
    if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 1024; h->d = (hent_t *)realloc(h->d, sizeof(hent_t) * h->cap); }
    i64 i = h->n++;
    h->d[i] = e;
    while (i) {
        i64 p = (i - 1) / 2;
        if (!hless(&h->d[i], &h->d[p])) break;
        hent_t t = h->d[i]; h->d[i] = h->d[p]; h->d[p] = t;
        i = p;
    }
}
static hent_t hpop(heap_t *h) {
    hent_t top = h->d[0];
    h->d[0] = h->d[--h->n];
    i64 i = 0;
    for (;;) {
        i64 l = 2 * i + 1, r = l + 1, s = i;
        if (l < h->n && hless(&h->d[l], &h->d[s])) s = l;
        if (r < h->n && hless(&h->d[r], &h->d[s])) s = r;
        if (s == i) break;
        hent_t t = h->d[i]; h->d[i] = h->d[s]; h->d[s] = t;
        i = s;
    }
    return top;
}

/* pair -> cost hash map with deletion (open addressing + tombstones) */
typedef struct { u64 *key; double *val; char *st; i64 cap, used; } pmap_t;
#define PM_EMPTY 0
#define PM_FULL 1
#define PM_DEAD 2
static u64 pm_hash(u64 k) { k ^= k >> 33; k *= 0xff51afd7ed558ccdULL; k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ULL; k ^= k >> 33; return k; }
static void pm_init(pmap_t *p, i64 want) {
    i64 cap = 16;
    while (cap < 2 * want + 16) cap <<= 1;
    p->cap = cap; p->used = 0;
    p->key = (u64 *)xmalloc(sizeof(u64) * cap);
    p->val = (double *)xmalloc(sizeof(double) * cap);
    p->st = (char *)xcalloc(cap, 1);
}
static void pm_free(pmap_t *p) { free(p->key); free(p->val); free(p->st); }
static i64 pm_slot(const pmap_t *p, u64 k) {
    i64 i = pm_hash(k) & (p->cap - 1);
    while (p->st[i] != PM_EMPTY) {
        if (p->st[i] == PM_FULL && p->key[i] == k) return i;
        i = (i + 1) & (p->cap - 1);
    }
    return -1;
}
static void pm_rehash(pmap_t *p);
static void pm_put(pmap_t *p, u64 k, double val) {
    i64 s = pm_slot(p, k);
    if (s >= 0) { p->val[s] = val; return; }
    if (2 * (p->used + 1) > p->cap) pm_rehash(p);
    i64 i = pm_hash(k) & (p->cap - 1);
    while (p->st[i] == PM_FULL) i = (i + 1) & (p->cap - 1);
    if (p->st[i] == PM_EMPTY) p->used++;
    p->st[i] = PM_FULL; p->key[i] = k; p->val[i] = val;
}
static void pm_rehash(pmap_t *p) {
    pmap_t q;
    i64 live = 0;
    for (i64 i = 0; i < p->cap; i++) live += p->st[i] == PM_FULL;
    pm_init(&q, live * 2 + 16);
    for (i64 i = 0; i < p->cap; i++)
        if (p->st[i] == PM_FULL) pm_put(&q, p->key[i], p->val[i]);
    pm_free(p);
    *p = q;
}
static void pm_del(pmap_t *p, u64 k) {
    i64 s = pm_slot(p, k);
    if (s >= 0) p->st[s] = PM_DEAD;
}
static u64 pkey(i64 a, i64 b) { return a < b ? ((u64)a << 32) | (u64)b : ((u64)b << 32) | (u64)a; }

typedef struct { i64 *d; i64 n, cap; } ivec_t;
static void iv_push(ivec_t *v, i64 x) {
    if (v->n == v->cap) { v->cap = v->cap ? 2 * v->cap : 4; v->d = (i64 *)realloc(v->d, sizeof(i64) * v->cap); }
    v->d[v->n++] = x;
}

/* gaec_exhaustive (contraction.py:397-452): lazy max-heap keyed
 * (-c, lo, hi); the smaller id stays representative; parallel edges sum
 * as prev + cx.  map = canonical ids of the final roots. */
int orc_gaec(i64 n, i64 m, const i64 *u, const i64 *v, const double *c, i64 *map,
             i64 *num_targets, double *joined_out) {
    pmap_t pm;
    pm_init(&pm, m);
    ivec_t *nb = (ivec_t *)xcalloc(n, sizeof(ivec_t));
    heap_t h = {0, 0, 0};
    for (i64 i = 0; i < m; i++) {
        pm_put(&pm, pkey(u[i], v[i]), c[i]);
        iv_push(&nb[u[i]], v[i]);
        iv_push(&nb[v[i]], u[i]);
        if (c[i] > 0.0) { hent_t e = {-c[i], u[i], v[i]}; hpush(&h, e); }
    }
    i64 *par = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    for (i64 x = 0; x < n; x++) par[x] = x;
    i64 *mark = (i64 *)xcalloc(n, sizeof(i64));
    i64 epoch = 0;
    double joined = 0.0;
    while (h.n) {
        hent_t top = hpop(&h);
        double cc = -top.negc;
        i64 a = top.a, b = top.b;
        if (par[a] != a || par[b] != b) continue;
        i64 s = pm_slot(&pm, pkey(a, b));
        if (s < 0 || pm.val[s] != cc) continue;
        par[b] = a;
        joined += cc;
        pm_del(&pm, pkey(a, b));
        epoch++;
        /* live neighbours of b, each once */
        ivec_t *lb = &nb[b];
        for (i64 q = 0; q < lb->n; q++) {
            i64 x = lb->d[q];
            if (x == a || mark[x] == epoch) continue;
            i64 sx = pm_slot(&pm, pkey(b, x));
            if (sx < 0) continue;
            mark[x] = epoch;
            double cx = pm.val[sx];
            pm_del(&pm, pkey(b, x));
            i64 sa = pm_slot(&pm, pkey(a, x));
            double newc = sa < 0 ? cx : pm.val[sa] + cx;
            if (sa < 0) { iv_push(&nb[a], x); iv_push(&nb[x], a); }
            pm_put(&pm, pkey(a, x), newc);
            if (newc > 0.0) {
                hent_t e = {-newc, a < x ? a : x, a < x ? x : a};
                hpush(&h, e);
            }
        }
        free(lb->d);
        lb->d = NULL; lb->n = lb->cap = 0;
    }
    i64 t = 0;
    for (i64 x = 0; x < n; x++) {
        i64 r = uf_find(par, x);
        if (r == x) map[x] = t++;
        else map[x] = map[r];
    }
    *num_targets = t;
    *joined_out = joined;
    for (i64 x = 0; x < n; x++) free(nb[x].d);
    free(nb); free(par); free(mark); free(h.d);
    pm_free(&pm);
    return ORC_OK;
}

/* ------------------------------------------------- handshake cleanup (D1)
 *
 * The B200 build's replacement for the sequential GAEC cleanup
 * (solver.py:187-194 -> contraction.py:397-452); DESIGN.md deviation D1.
 * Each round is one handshake on the current quotient: every node targets
 * its live positive neighbour of maximum cost (ties -> smaller id, the
 * select_matching rule, contraction.py:207), mutual pairs (x < t) merge
 * into the smaller id.  Node ids are never renumbered; an edge with a
 * merged endpoint (either side of a pair) is relabelled, dropped if it became internal, and
 * parallel relabelled edges fold into the smallest edge slot with a
 * sequential sum in ascending slot order.  Repeats until no pair forms;
 * the labelling is the canonical component map of all merged pairs. */
typedef struct { u64 key; i64 idx; } tkey_t;

static int cmp_tkey(const void *pa, const void *pb) {
    const tkey_t *a = (const tkey_t *)pa, *b = (const tkey_t *)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

int orc_cleanup_handshake(i64 n, i64 m, const i64 *u, const i64 *v, const double *c, i64 *map,
                          i64 *num_targets, i64 *rounds_out) {
    i64 *eu = (i64 *)xmalloc(sizeof(i64) * (m ? m : 1));
    i64 *ev = (i64 *)xmalloc(sizeof(i64) * (m ? m : 1));
    double *ec = (double *)xmalloc(sizeof(double) * (m ? m : 1));
    char *alive = (char *)xmalloc(m ? m : 1);
    for (i64 i = 0; i < m; i++) { eu[i] = u[i]; ev[i] = v[i]; ec[i] = c[i]; alive[i] = 1; }
    i64 *tgt = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    double *bc = (double *)xmalloc(sizeof(double) * (n ? n : 1));
    i64 *rep = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    i64 *par = (i64 *)xmalloc(sizeof(i64) * (n ? n : 1));
    tkey_t *tk = (tkey_t *)xmalloc(sizeof(tkey_t) * (m ? m : 1));
    for (i64 x = 0; x < n; x++) { par[x] = x; rep[x] = x; }
    i64 rounds = 0;
    while (1) {
        for (i64 x = 0; x < n; x++) tgt[x] = -1;
        for (i64 i = 0; i < m; i++) {
            if (!alive[i] || !(ec[i] > 0.0)) continue;
            for (int side = 0; side < 2; side++) {
                i64 a = side ? ev[i] : eu[i], b = side ? eu[i] : ev[i];
                if (tgt[a] < 0 || ec[i] > bc[a] || (ec[i] == bc[a] && b < tgt[a])) { tgt[a] = b; bc[a] = ec[i]; }
            }
        }
        i64 pairs = 0;
        for (i64 x = 0; x < n; x++) {
            i64 t = tgt[x];
            if (t >= 0 && x < t && tgt[t] == x) { rep[t] = x; par[t] = x; pairs++; }
        }
        /* mark merged nodes (tgt = -2 - partner keeps tgt[] readable above) */
        for (i64 x = 0; x < n; x++)
            if (rep[x] != x) { tgt[x] = -2; tgt[rep[x]] = -2; }
        if (!pairs) break;
        rounds++;
        i64 nt = 0;
        for (i64 i = 0; i < m; i++) {
            if (!alive[i]) continue;
            if (tgt[eu[i]] < -1 || tgt[ev[i]] < -1) {} else continue;  /* no endpoint merged */
            i64 a = rep[eu[i]], b = rep[ev[i]];
            if (a == b) { alive[i] = 0; continue; }
            eu[i] = a < b ? a : b;
            ev[i] = a < b ? b : a;
            tk[nt].key = ((u64)eu[i] << 32) | (u64)ev[i];
            tk[nt].idx = i;
            nt++;
        }
        qsort(tk, nt, sizeof(tkey_t), cmp_tkey);
        for (i64 j = 0; j < nt;) {
            i64 first = tk[j].idx, e = j + 1;
            double acc = ec[first];
            while (e < nt && tk[e].key == tk[j].key) { acc += ec[tk[e].idx]; alive[tk[e].idx] = 0; e++; }
            ec[first] = acc;
            j = e;
        }
        for (i64 x = 0; x < n; x++) rep[x] = x;
    }
    i64 t = 0;
    for (i64 x = 0; x < n; x++) {
        i64 r = uf_find(par, x);
        if (r == x) map[x] = t++;
        else map[x] = map[r];
    }
    *num_targets = t;
    if (rounds_out) *rounds_out = rounds;
    free(eu); free(ev); free(ec); free(alive); free(tgt); free(bc); free(rep); free(par); free(tk);
    return ORC_OK;
}
