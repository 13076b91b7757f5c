/*
 * gts_oracle.c -- CPU restatement of the reference GTS path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * (paper_2404_00966_b200/) never links or calls it.
 *
 * It restates, in plain C with float64 arithmetic, the reference package
 * `metrictree` (arXiv 2404.00966 reference, /root/reference/pkg/src):
 *   - distances ............ metrics.py:54-84 (_edit_pair), 127-133, 166-172
 *                            (L1/L2; numpy's pairwise row-sum order, so the
 *                            results are bit-identical to numpy's)
 *   - tree build ........... tree.py:60-135 (height, addressing, keys),
 *                            tree.py:241-367 (_Builder: map/sort/spawn/ranges)
 *   - BatchSearcher ........ search.py:28-95 (predicates, size limit, groups),
 *                            search.py:116-144 (_KnnPool), 273-570 (driver,
 *                            root table, process/expand/merge/verify/collect)
 *   - MemoryBudget ......... runtime.py:56-88
 *   - brute force .......... oracle.py:19-47
 * Pinned against the tests/golden npz fixtures, produced by running the reference
 * itself (tests/golden/make_golden.py).
 *
 * Compile with -ffp-contract=off: numpy never fuses x*x+acc into an FMA.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif
enum { M_EDIT = 0, M_L1 = 1, M_L2 = 2, M_ANGULAR = 3 };
enum { MODE_RANGE = 0, MODE_KNN = 1 };

/* A payload collection: dataset or query batch (data.py:59-126). */
typedef struct {
    i64 metric;
    i64 n;
    i64 dim;            /* vectors: D */
    const double *vec;  /* [n*dim] row-major f64 */
    const int32_t *codes; /* strings: UTF-32 code points */
    const i64 *off;     /* [n+1] */
    const i64 *ids;     /* [n] strictly increasing (datasets only) */
} orc_ds;

/* FlatPivotTree arrays (tree.py:155-175). Node arrays have nodes+1 slots. */
typedef struct {
    i64 nc, levels, split_rounds, nodes, n;
    i64 *pivot_id, *pivot_row, *pos, *size;
    double *min_dis, *max_dis;
    i64 *rows;
    double *dis;
    uint8_t *tomb;
} orc_tree;

/* ------------------------------------------------------------------ */
/* distances                                                            */
/* ------------------------------------------------------------------ */

/* metrics.py:54-84 -- two-row DP over the shorter string, unit costs. */
static i64 edit_pair(const int32_t *a, i64 la, const int32_t *b, i64 lb, i64 *row)
{
    if (la == 0) return lb;
    if (lb == 0) return la;
    if (lb > la) { const int32_t *t = a; a = b; b = t; i64 tl = la; la = lb; lb = tl; }
    for (i64 j = 0; j <= lb; j++) row[j] = j;
    for (i64 i = 1; i <= la; i++) {
        i64 prev_diag = row[0];
        row[0] = i;
        int32_t ca = a[i - 1];
        for (i64 j = 1; j <= lb; j++) {
            i64 tmp = row[j];
            i64 best = prev_diag + (ca == b[j - 1] ? 0 : 1);
            if (row[j] + 1 < best) best = row[j] + 1;
            if (row[j - 1] + 1 < best) best = row[j - 1] + 1;
            row[j] = best;
            prev_diag = tmp;
        }
    }
    return row[lb];
}

/* numpy pairwise_sum (8-way unrolled below 128 elements, halving above):
 * the order numpy uses for `.sum(axis=1)` over a contiguous row. */
static double pw_sum(const double *a, i64 n)
{
    if (n < 8) {
        double r = 0.0;
        for (i64 i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        i64 i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        i64 n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
    }
}

/* metrics.py:136-163 / 175-193 (angular_one_to_many / angular_row_pairs):
 * norms = sqrt(pairwise sum of squares) (data.py:81-84), dots = pairwise sum
 * of products, cos = clip(dot / (nx * nq), -1, 1), d = arccos(cos); zero
 * vectors sit at pi from non-zero vectors and 0 from each other; d < 1e-6 with
 * identical components -> 0.  The reference's one_to_many takes the query norm
 * from np.dot (BLAS, summation order unspecified); this uses the pairwise sum
 * for both norms, so query distances can differ from the reference in the
 * last bits (tests compare them with a 1e-12 relative tolerance); row_pairs
 * (the build) is the same computation bit for bit. */
static double angular_dist(const double *x, const double *q, i64 D, double *tmp)
{
    for (i64 d = 0; d < D; d++) tmp[d] = x[d] * x[d];
    const double nx = sqrt(pw_sum(tmp, D));
    for (i64 d = 0; d < D; d++) tmp[d] = q[d] * q[d];
    const double nq = sqrt(pw_sum(tmp, D));
    if (nq == 0.0) return nx == 0.0 ? 0.0 : M_PI;
    if (nx == 0.0) return M_PI;
    for (i64 d = 0; d < D; d++) tmp[d] = x[d] * q[d];
    const double dot = pw_sum(tmp, D);
    double c = dot / (nx * nq);
    if (c < -1.0) c = -1.0;
    if (c > 1.0) c = 1.0;
    double r = acos(c);
    if (r < 1e-6) {
        int eq = 1;
        for (i64 d = 0; d < D && eq; d++) eq = x[d] == q[d];
        if (eq) r = 0.0;
    }
    return r;
}

/* metrics.py:127-133 / 166-172: diff = x - q; L1 = sum|diff|, L2 = sqrt(sum diff^2) */
static double vec_dist(i64 metric, const double *x, const double *q, i64 D, double *tmp)
{
    if (metric == M_ANGULAR) return angular_dist(x, q, D, tmp);
    for (i64 d = 0; d < D; d++) {
        double diff = x[d] - q[d];
        tmp[d] = (metric == M_L1) ? fabs(diff) : diff * diff;
    }
    double s = pw_sum(tmp, D);
    return metric == M_L1 ? s : sqrt(s);
}

typedef struct {
    i64 *dprow;   /* edit DP row */
    double *tmp;  /* vector temp */
} scratch;

static void scratch_init(scratch *s, i64 maxlen, i64 dim)
{
    s->dprow = (i64 *)malloc(sizeof(i64) * (size_t)(maxlen + 2));
    s->tmp = (double *)malloc(sizeof(double) * (size_t)(dim + 1));
}
static void scratch_free(scratch *s) { free(s->dprow); free(s->tmp); }

/* distance between row `r` of ds and item `qi` of qs (qs may equal ds). */
static double dist_rq(const orc_ds *ds, i64 r, const orc_ds *qs, i64 qi, scratch *s)
{
    if (ds->metric == M_EDIT) {
        const int32_t *a = ds->codes + ds->off[r];
        const int32_t *b = qs->codes + qs->off[qi];
        return (double)edit_pair(b, qs->off[qi + 1] - qs->off[qi], a, ds->off[r + 1] - ds->off[r], s->dprow);
    }
    return vec_dist(ds->metric, ds->vec + r * ds->dim, qs->vec + qi * qs->dim, ds->dim, s->tmp);
}

static i64 max_len(const orc_ds *d)
{
    i64 m = 0;
    if (d->metric != M_EDIT) return 0;
    for (i64 i = 0; i < d->n; i++) {
        i64 l = d->off[i + 1] - d->off[i];
        if (l > m) m = l;
    }
    return m;
}

/* exported for the metric golden tests */
double orc_edit(const int32_t *a, i64 la, const int32_t *b, i64 lb)
{
    i64 *row = (i64 *)malloc(sizeof(i64) * (size_t)((la > lb ? la : lb) + 2));
    i64 d = edit_pair(a, la, b, lb, row);
    free(row);
    return (double)d;
}
double orc_vec(i64 metric, const double *x, const double *q, i64 D)
{
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(D + 1));
    double d = vec_dist(metric, x, q, D, tmp);
    free(tmp);
    return d;
}

/* ------------------------------------------------------------------ */
/* tree arithmetic (tree.py:60-108)                                     */
/* ------------------------------------------------------------------ */

int orc_tree_height(i64 n, i64 nc, i64 *max_h, i64 *split)
{
    if (nc < 2 || n < 1) return 1;
    i64 t = 0;
    __int128 power = 1;
    while (power < (__int128)n + 1) { power *= nc; t++; }
    *max_h = t - 1;
    *split = (*max_h - 1) > 0 ? (*max_h - 1) : 0;
    return 0;
}

i64 orc_node_count(i64 levels, i64 nc)
{
    __int128 p = 1;
    for (i64 i = 0; i < levels; i++) p *= nc;
    return (i64)((p - 1) / (nc - 1));
}

static void level_range(i64 level, i64 nc, i64 *first, i64 *count)
{
    __int128 c = 1;
    for (i64 i = 1; i < level; i++) c *= nc;
    *count = (i64)c;
    *first = (i64)((c - 1) / (nc - 1) + 1);
}

/* ------------------------------------------------------------------ */
/* build (tree.py:241-367)                                              */
/* ------------------------------------------------------------------ */

typedef struct { double key; i64 tie; i64 idx; } keyrec;

static int keyrec_cmp(const void *pa, const void *pb)
{
    const keyrec *a = (const keyrec *)pa, *b = (const keyrec *)pb;
    if (a->key < b->key) return -1;
    if (a->key > b->key) return 1;
    if (a->tie < b->tie) return -1;
    if (a->tie > b->tie) return 1;
    return 0;
}

/* Build into caller-allocated tree arrays (node arrays sized nodes+1,
 * table arrays sized n).  root_row = rng.integers(0, n) drawn by the
 * caller with numpy's default_rng(seed) (tree.py:263, 288-291). */
int orc_build(const orc_ds *ds, orc_tree *t, i64 root_row, int threads)
{
    i64 n = ds->n, nc = t->nc;
    if (n == 0) { t->levels = 0; return 0; }
    i64 max_h, split;
    orc_tree_height(n, nc, &max_h, &split);
    t->split_rounds = split;
    t->levels = split + 1;
    t->nodes = orc_node_count(t->levels, nc);
    for (i64 i = 0; i <= t->nodes; i++) {
        t->pivot_id[i] = -1; t->pivot_row[i] = -1;
        t->min_dis[i] = 0; t->max_dis[i] = 0; t->pos[i] = 0; t->size[i] = 0;
    }
    t->size[1] = n;
    t->pos[1] = 0;
    for (i64 i = 0; i < n; i++) { t->rows[i] = i; t->dis[i] = 0; t->tomb[i] = 0; }
    double *chain = (double *)malloc(sizeof(double) * (size_t)n);
    double *tmpd = (double *)malloc(sizeof(double) * (size_t)n);
    i64 *tmpr = (i64 *)malloc(sizeof(i64) * (size_t)n);
    i64 *epiv = (i64 *)malloc(sizeof(i64) * (size_t)n);
    keyrec *keys = (keyrec *)malloc(sizeof(keyrec) * (size_t)n);
    int have_chain = 0;
    i64 ml = max_len(ds);
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#endif
    for (i64 level = 1; level <= t->levels; level++) {
        i64 first, count;
        level_range(level, nc, &first, &count);
        /* _map_level: pivots */
        if (level == 1) {
            i64 prow = t->rows[root_row];
            t->pivot_row[1] = prow;
            t->pivot_id[1] = ds->ids[prow];
        } else {
            for (i64 node = first; node < first + count; node++) {
                i64 sz = t->size[node];
                if (sz <= 0) continue;
                i64 p = t->pos[node];
                double best = chain[p];
                for (i64 e = p + 1; e < p + sz; e++) if (chain[e] > best) best = chain[e];
                i64 prow = -1, pid = 0;
                for (i64 e = p; e < p + sz; e++) {
                    if (chain[e] == best) {
                        i64 r = t->rows[e];
                        if (prow < 0 || ds->ids[r] < pid) { prow = r; pid = ds->ids[r]; }
                    }
                }
                t->pivot_row[node] = prow;
                t->pivot_id[node] = pid;
            }
        }
        /* entry pivot per table entry; map distances (row_to_row) */
        {
            i64 e = 0;
            for (i64 node = first; node < first + count; node++)
                for (i64 j = 0; j < t->size[node]; j++) epiv[e++] = t->pivot_row[node];
        }
        #pragma omp parallel
        {
            scratch s;
            scratch_init(&s, ml, ds->dim);
            #pragma omp for schedule(dynamic, 256)
            for (i64 e = 0; e < n; e++) {
                i64 r = t->rows[e], pv = epiv[e];
                double d;
                if (ds->metric == M_EDIT) {
                    d = (double)edit_pair(ds->codes + ds->off[r], ds->off[r + 1] - ds->off[r],
                                          ds->codes + ds->off[pv], ds->off[pv + 1] - ds->off[pv], s.dprow);
                } else {
                    d = vec_dist(ds->metric, ds->vec + r * ds->dim, ds->vec + pv * ds->dim, ds->dim, s.tmp);
                }
                t->dis[e] = d;
            }
            scratch_free(&s);
        }
        if (!have_chain) { memcpy(chain, t->dis, sizeof(double) * (size_t)n); have_chain = 1; }
        else for (i64 e = 0; e < n; e++) if (t->dis[e] < chain[e]) chain[e] = t->dis[e];
        /* _sort_level: key = dis/(level_max+1) + ordinal, tie = object id */
        double lm = t->dis[0];
        for (i64 e = 1; e < n; e++) if (t->dis[e] > lm) lm = t->dis[e];
        {
            i64 e = 0;
            for (i64 o = 0; o < count; o++) {
                i64 node = first + o;
                for (i64 j = 0; j < t->size[node]; j++, e++) {
                    keys[e].key = t->dis[e] / (lm + 1.0) + (double)o;
                    keys[e].tie = ds->ids[t->rows[e]];
                    keys[e].idx = e;
                }
            }
        }
        qsort(keys, (size_t)n, sizeof(keyrec), keyrec_cmp);
        for (i64 e = 0; e < n; e++) { tmpr[e] = t->rows[keys[e].idx]; tmpd[e] = t->dis[keys[e].idx]; }
        memcpy(t->rows, tmpr, sizeof(i64) * (size_t)n);
        memcpy(t->dis, tmpd, sizeof(double) * (size_t)n);
        if (level < t->levels) {
            for (i64 e = 0; e < n; e++) tmpd[e] = chain[keys[e].idx];
            memcpy(chain, tmpd, sizeof(double) * (size_t)n);
            /* _spawn_children + _set_ranges */
            i64 cfirst = (first - 1) * nc + 2;
            for (i64 o = 0; o < count; o++) {
                i64 node = first + o, sz = t->size[node], p = t->pos[node];
                i64 avg = sz / nc;
                for (i64 j = 0; j < nc; j++) {
                    i64 c = cfirst + o * nc + j;
                    t->pos[c] = p + j * avg;
                    t->size[c] = (j == nc - 1) ? sz - avg * (nc - 1) : avg;
                    if (t->size[c] > 0) {
                        t->min_dis[c] = t->dis[t->pos[c]];
                        t->max_dis[c] = t->dis[t->pos[c] + t->size[c] - 1];
                    }
                }
            }
        } else {
            /* _finalize_leaves */
            for (i64 o = 0; o < count; o++) {
                i64 c = first + o;
                if (t->size[c] > 0) {
                    t->min_dis[c] = t->dis[t->pos[c]];
                    t->max_dis[c] = t->dis[t->pos[c] + t->size[c] - 1];
                }
            }
        }
    }
    free(chain); free(tmpd); free(tmpr); free(epiv); free(keys);
    return 0;
}

/* ------------------------------------------------------------------ */
/* search (search.py)                                                   */
/* ------------------------------------------------------------------ */

#define MAX_LAYERS 64

typedef struct {
    i64 nq;
    i64 *counts;         /* [nq] */
    i64 *ids;            /* [total] */
    double *dis;         /* [total] */
    i64 total;
    i64 *verified;       /* [nq] */
    i64 *pruned;         /* [nq] */
    i64 peak;
    i64 limits[MAX_LAYERS]; /* size_limits[layer], 0 = layer not visited */
    int status;          /* 0 ok, 2 budget error */
    char err[256];
} orc_result;

/* _KnnPool (search.py:116-144): best-k (d, row) sorted by (d, id). */
typedef struct { i64 k, cnt; double *d; i64 *row; } pool_t;

typedef struct { double d; i64 id; i64 row; } cand_t;

static int cand_cmp(const void *pa, const void *pb)
{
    const cand_t *a = (const cand_t *)pa, *b = (const cand_t *)pb;
    if (a->d < b->d) return -1;
    if (a->d > b->d) return 1;
    if (a->id < b->id) return -1;
    if (a->id > b->id) return 1;
    return 0;
}

/* growable vectors */
typedef struct { i64 *v; i64 n, cap; } ivec;
typedef struct { double *v; i64 n, cap; } dvec;
static void iv_push(ivec *a, i64 x)
{
    if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 16; a->v = (i64 *)realloc(a->v, sizeof(i64) * (size_t)a->cap); }
    a->v[a->n++] = x;
}
static void dv_push(dvec *a, double x)
{
    if (a->n == a->cap) { a->cap = a->cap ? a->cap * 2 : 16; a->v = (double *)realloc(a->v, sizeof(double) * (size_t)a->cap); }
    a->v[a->n++] = x;
}

typedef struct {
    const orc_tree *t;
    const orc_ds *ds;
    const orc_ds *qs;
    i64 q0, nq;          /* slice of the query batch */
    int mode;
    const double *radii; /* indexed by absolute query id */
    pool_t *pools;       /* [nq] local */
    const uint8_t *row_dead; /* [ds->n] */
    i64 capacity, in_use, peak;
    i64 *limits;
    i64 *verified, *pruned; /* local [nq] */
    ivec *acc_row;       /* range hits per local query */
    dvec *acc_dis;
    cand_t *cbuf; i64 cbuf_cap;
    scratch s;
    int status;
    char *err;
} ctx_t;

static void pool_merge(ctx_t *c, pool_t *p, const double *dv, const i64 *rows, i64 m)
{
    /* take = candidates not already pooled and not excluded (search.py:129-133) */
    i64 need = p->cnt + m;
    if (need > c->cbuf_cap) {
        c->cbuf_cap = need * 2;
        c->cbuf = (cand_t *)realloc(c->cbuf, sizeof(cand_t) * (size_t)c->cbuf_cap);
    }
    i64 nt = 0;
    for (i64 t = 0; t < m; t++) {
        i64 r = rows[t];
        if (c->row_dead[r]) continue;
        int dup = 0;
        for (i64 u = 0; u < p->cnt; u++) if (p->row[u] == r) { dup = 1; break; }
        if (dup) continue;
        c->cbuf[nt].d = dv[t]; c->cbuf[nt].row = r; c->cbuf[nt].id = c->ds->ids[r]; nt++;
    }
    if (nt == 0) return;
    for (i64 u = 0; u < p->cnt; u++) {
        c->cbuf[nt].d = p->d[u]; c->cbuf[nt].row = p->row[u]; c->cbuf[nt].id = c->ds->ids[p->row[u]]; nt++;
    }
    qsort(c->cbuf, (size_t)nt, sizeof(cand_t), cand_cmp);
    i64 keep = nt < p->k ? nt : p->k;
    for (i64 u = 0; u < keep; u++) { p->d[u] = c->cbuf[u].d; p->row[u] = c->cbuf[u].row; }
    p->cnt = keep;
}

static double pool_bound(const pool_t *p)
{
    return p->cnt >= p->k ? p->d[p->k - 1] : INFINITY;
}

/* _Table: (local query, node, dqp) rows in canonical order */
typedef struct { i64 *q; i64 *node; double *dqp; i64 rows; } table_t;

static void tab_free(table_t *t) { free(t->q); free(t->node); free(t->dqp); }

static i64 level_size_limit(i64 cap, i64 nc, i64 split, i64 layer)
{
    i64 share = cap / ((split - layer + 1) * nc);
    return share > 1 ? share : 1;
}

static void process(ctx_t *c, table_t *tab, i64 layer, i64 reserved);

static void release(ctx_t *c, i64 units) { c->in_use -= units; }

static void verify(ctx_t *c, table_t *tab)
{
    const orc_tree *t = c->t;
    i64 i = 0;
    while (i < tab->rows) {
        i64 qv = tab->q[i], stop = i;
        while (stop < tab->rows && tab->q[stop] == qv) stop++;
        i64 qa = c->q0 + qv;
        if (c->mode == MODE_RANGE) {
            /* search.py:507-538 */
            double r = c->radii[qa];
            i64 ver = 0;
            for (i64 x = i; x < stop; x++) {
                i64 node = tab->node[x], p = t->pos[node], sz = t->size[node];
                for (i64 e = p; e < p + sz; e++) {
                    if (t->tomb[e] != 0) continue;
                    if (!(fabs(t->dis[e] - tab->dqp[x]) <= r)) continue;
                    i64 row = t->rows[e];
                    double d = dist_rq(c->ds, row, c->qs, qa, &c->s);
                    ver++;
                    if (d <= r) { iv_push(&c->acc_row[qv], row); dv_push(&c->acc_dis[qv], d); }
                }
            }
            c->verified[qv] += ver;
        } else {
            /* search.py:540-570 */
            pool_t *pool = &c->pools[qv];
            i64 count = 0;
            ivec rows = {0}; dvec dv = {0};
            for (i64 x = i; x < stop; x++) {
                i64 node = tab->node[x], p = t->pos[node], sz = t->size[node];
                double dqp = tab->dqp[x];
                double bound = pool_bound(pool);
                rows.n = 0; dv.n = 0;
                for (i64 e = p; e < p + sz; e++) {
                    if (t->tomb[e] != 0) continue;
                    if (!isinf(bound) && !(fabs(t->dis[e] - dqp) < bound)) continue;
                    iv_push(&rows, t->rows[e]);
                }
                if (rows.n == 0) continue;
                for (i64 u = 0; u < rows.n; u++) dv_push(&dv, dist_rq(c->ds, rows.v[u], c->qs, qa, &c->s));
                pool_merge(c, pool, dv.v, rows.v, rows.n);
                count += rows.n;
            }
            free(rows.v); free(dv.v);
            c->verified[qv] += count;
        }
        i = stop;
    }
}

/* _expand (search.py:405-477) */
static void expand(ctx_t *c, const table_t *part, i64 layer, table_t *out)
{
    const orc_tree *t = c->t;
    i64 nc = t->nc;
    int own = (layer + 1) == t->levels;
    i64 cap = part->rows * nc;
    out->q = (i64 *)malloc(sizeof(i64) * (size_t)(cap + 1));
    out->node = (i64 *)malloc(sizeof(i64) * (size_t)(cap + 1));
    out->dqp = (double *)malloc(sizeof(double) * (size_t)(cap + 1));
    double *cpd = (double *)malloc(sizeof(double) * (size_t)(cap + 1));
    out->rows = 0;
    /* kNN bounds are read once, before the level (search.py:411-412) */
    double *bounds = NULL;
    if (c->mode == MODE_KNN) {
        bounds = (double *)malloc(sizeof(double) * (size_t)c->nq);
        for (i64 q = 0; q < c->nq; q++) bounds[q] = pool_bound(&c->pools[q]);
    }
    for (i64 x = 0; x < part->rows; x++) {
        i64 qv = part->q[x], qa = c->q0 + qv, node = part->node[x];
        double dq = part->dqp[x];
        i64 first = (node - 1) * nc + 2;
        i64 nonempty = 0, kept = 0;
        for (i64 j = 0; j < nc; j++) {
            i64 ch = first + j;
            if (t->size[ch] <= 0) continue;
            nonempty++;
            if (!own) {
                double mn = t->min_dis[ch], mx = t->max_dis[ch];
                if (c->mode == MODE_RANGE) {
                    double r = c->radii[qa];
                    if (!((dq + r >= mn) && (dq - r <= mx))) continue;
                } else {
                    double b = bounds[qv];
                    if (!((dq + b > mn) && (dq - b < mx))) continue;
                }
            }
            kept++;
            i64 o = out->rows++;
            out->q[o] = qv;
            out->node[o] = ch;
            out->dqp[o] = dist_rq(c->ds, t->pivot_row[ch], c->qs, qa, &c->s);
            cpd[o] = dq;
        }
        c->pruned[qv] += nonempty - kept;
    }
    i64 w = 0;
    if (c->mode == MODE_KNN) {
        /* _merge_level (search.py:479-497): per query, merge all new pivot
         * witnesses at once (the merge is a set union, order-free) */
        i64 i = 0;
        ivec prow = {0};
        while (i < out->rows) {
            i64 qv = out->q[i], stop = i;
            while (stop < out->rows && out->q[stop] == qv) stop++;
            prow.n = 0;
            for (i64 x = i; x < stop; x++) iv_push(&prow, t->pivot_row[out->node[x]]);
            pool_merge(c, &c->pools[qv], out->dqp + i, prow.v, stop - i);
            i = stop;
        }
        free(prow.v);
        for (i64 x = 0; x < out->rows; x++) {
            i64 qv = out->q[x];
            double b = pool_bound(&c->pools[qv]);
            double ref = own ? out->dqp[x] : cpd[x];
            double mn = t->min_dis[out->node[x]], mx = t->max_dis[out->node[x]];
            if ((ref + b > mn) && (ref - b < mx)) {
                out->q[w] = out->q[x]; out->node[w] = out->node[x]; out->dqp[w] = out->dqp[x]; w++;
            } else {
                c->pruned[qv] += 1;
            }
        }
        out->rows = w;
    } else if (own) {
        for (i64 x = 0; x < out->rows; x++) {
            i64 qv = out->q[x];
            double r = c->radii[c->q0 + qv];
            double mn = t->min_dis[out->node[x]], mx = t->max_dis[out->node[x]];
            double cd = out->dqp[x];
            if ((cd + r >= mn) && (cd - r <= mx)) {
                out->q[w] = out->q[x]; out->node[w] = out->node[x]; out->dqp[w] = out->dqp[x]; w++;
            } else {
                c->pruned[qv] += 1;
            }
        }
        out->rows = w;
    }
    free(cpd);
    free(bounds);
}

static void expand_into(ctx_t *c, table_t *part, i64 layer)
{
    table_t child;
    expand(c, part, layer, &child);
    if (child.rows == 0) { tab_free(&child); return; }
    if (c->in_use + child.rows > c->capacity) {
        c->status = 2;
        snprintf(c->err, 256, "table of %lld rows overflows budget %lld (in use %lld)",
                 (long long)child.rows, (long long)c->capacity, (long long)c->in_use);
        tab_free(&child);
        return;
    }
    c->in_use += child.rows;
    if (c->in_use > c->peak) c->peak = c->in_use;
    process(c, &child, layer + 1, child.rows);
    tab_free(&child);
}

static void slice_tab(const table_t *src, i64 a, i64 b, table_t *dst)
{
    dst->q = src->q + a; dst->node = src->node + a; dst->dqp = src->dqp + a; dst->rows = b - a;
}

/* _process (search.py:359-392) with compute_query_groups (73-95) */
static void process(ctx_t *c, table_t *tab, i64 layer, i64 reserved)
{
    if (c->status) return;
    if (tab->rows == 0) { if (reserved) release(c, reserved); return; }
    if (layer == c->t->levels) { verify(c, tab); if (reserved) release(c, reserved); return; }
    if (reserved) release(c, reserved);
    i64 s = level_size_limit(c->capacity, c->t->nc, c->t->split_rounds, layer);
    if (layer < MAX_LAYERS && c->limits[layer] == 0) c->limits[layer] = s;
    /* runs */
    ivec rs = {0}, re = {0};
    for (i64 i = 0; i < tab->rows;) {
        i64 j = i;
        while (j < tab->rows && tab->q[j] == tab->q[i]) j++;
        iv_push(&rs, i); iv_push(&re, j);
        i = j;
    }
    i64 nr = rs.n;
    /* greedy first fit */
    i64 *gid = (i64 *)malloc(sizeof(i64) * (size_t)(nr + 1));
    ivec loads = {0};
    for (i64 r = 0; r < nr; r++) {
        i64 cnt = re.v[r] - rs.v[r];
        i64 g;
        for (g = 0; g < loads.n; g++) if (loads.v[g] + cnt <= s) break;
        if (g == loads.n) iv_push(&loads, cnt); else loads.v[g] += cnt;
        gid[r] = g;
    }
    i64 ng = loads.n;
    for (i64 g = 0; g < ng && !c->status; g++) {
        i64 members = 0, only = -1, total = 0;
        for (i64 r = 0; r < nr; r++) if (gid[r] == g) { members++; only = r; total += re.v[r] - rs.v[r]; }
        if (members == 1 && total > s) {
            for (i64 off = rs.v[only]; off < re.v[only] && !c->status; off += s) {
                table_t part;
                i64 end = off + s < re.v[only] ? off + s : re.v[only];
                slice_tab(tab, off, end, &part);
                expand_into(c, &part, layer);
            }
        } else {
            table_t part;
            part.q = (i64 *)malloc(sizeof(i64) * (size_t)total);
            part.node = (i64 *)malloc(sizeof(i64) * (size_t)total);
            part.dqp = (double *)malloc(sizeof(double) * (size_t)total);
            part.rows = 0;
            for (i64 r = 0; r < nr; r++) {
                if (gid[r] != g) continue;
                for (i64 x = rs.v[r]; x < re.v[r]; x++) {
                    part.q[part.rows] = tab->q[x]; part.node[part.rows] = tab->node[x];
                    part.dqp[part.rows] = tab->dqp[x]; part.rows++;
                }
            }
            expand_into(c, &part, layer);
            tab_free(&part);
        }
    }
    free(gid); free(loads.v); free(rs.v); free(re.v);
}

/* _scan_all (search.py:338-355) */
static void scan_all(ctx_t *c)
{
    const orc_tree *t = c->t;
    for (i64 qv = 0; qv < c->nq; qv++) {
        i64 qa = c->q0 + qv;
        ivec rows = {0}; dvec dv = {0};
        for (i64 e = 0; e < t->n; e++) {
            if (t->tomb[e]) continue;
            i64 row = t->rows[e];
            iv_push(&rows, row);
            dv_push(&dv, dist_rq(c->ds, row, c->qs, qa, &c->s));
        }
        c->verified[qv] = rows.n;
        if (c->mode == MODE_RANGE) {
            for (i64 u = 0; u < rows.n; u++)
                if (dv.v[u] <= c->radii[qa]) { iv_push(&c->acc_row[qv], rows.v[u]); dv_push(&c->acc_dis[qv], dv.v[u]); }
        } else {
            pool_merge(c, &c->pools[qv], dv.v, rows.v, rows.n);
        }
        free(rows.v); free(dv.v);
    }
}

static void search_slice(ctx_t *c)
{
    const orc_tree *t = c->t;
    if (!c->ds->n || t->levels == 0) return;
    if (c->mode == MODE_KNN) {
        /* root pivot is a witness (search.py:326-329) */
    }
    /* caller handles pruning flag */
    table_t root;
    root.rows = c->nq;
    root.q = (i64 *)malloc(sizeof(i64) * (size_t)(c->nq + 1));
    root.node = (i64 *)malloc(sizeof(i64) * (size_t)(c->nq + 1));
    root.dqp = (double *)malloc(sizeof(double) * (size_t)(c->nq + 1));
    i64 prow = t->pivot_row[1];
    for (i64 q = 0; q < c->nq; q++) {
        root.q[q] = q; root.node[q] = 1;
        root.dqp[q] = dist_rq(c->ds, prow, c->qs, c->q0 + q, &c->s);
        if (c->mode == MODE_KNN) pool_merge(c, &c->pools[q], &root.dqp[q], &prow, 1);
    }
    process(c, &root, 1, 0);
    tab_free(&root);
}

static int rowcmp_ctx_dummy;

/* Full batch search.  threads > 1 splits the batch into disjoint query
 * slices (each a BatchSearcher call on its slice; answers are identical
 * to one call, SURVEY.md §8(d) mode iii). */
orc_result *orc_search(const orc_tree *t, const orc_ds *ds, const orc_ds *qs, int mode,
                       const double *radii, const i64 *ks, i64 capacity, int pruning, int threads)
{
    (void)rowcmp_ctx_dummy;
    i64 nq = qs->n;
    orc_result *res = (orc_result *)calloc(1, sizeof(orc_result));
    res->nq = nq;
    res->counts = (i64 *)calloc((size_t)(nq + 1), sizeof(i64));
    res->verified = (i64 *)calloc((size_t)(nq + 1), sizeof(i64));
    res->pruned = (i64 *)calloc((size_t)(nq + 1), sizeof(i64));
    if (nq == 0 || t->levels == 0 || ds->n == 0) {
        res->ids = (i64 *)malloc(8); res->dis = (double *)malloc(8);
        return res;
    }
    uint8_t *row_dead = (uint8_t *)calloc((size_t)ds->n, 1);
    for (i64 e = 0; e < t->n; e++) if (t->tomb[e]) row_dead[t->rows[e]] = 1;
    if (threads < 1) threads = 1;
    if (threads > nq) threads = (int)nq;
    i64 ml = max_len(ds), mq = max_len(qs);
    if (mq > ml) ml = mq;
    ctx_t *cs = (ctx_t *)calloc((size_t)threads, sizeof(ctx_t));
    i64 *slice_peak = (i64 *)calloc((size_t)threads, sizeof(i64));
    i64 (*lim)[MAX_LAYERS] = calloc((size_t)threads, sizeof(*lim));
#ifdef _OPENMP
    #pragma omp parallel for num_threads(threads) schedule(static, 1)
#endif
    for (int w = 0; w < threads; w++) {
        ctx_t *c = &cs[w];
        i64 a = nq * w / threads, b = nq * (w + 1) / threads;
        c->t = t; c->ds = ds; c->qs = qs; c->q0 = a; c->nq = b - a;
        c->mode = mode; c->radii = radii; c->row_dead = row_dead;
        c->capacity = capacity; c->limits = lim[w];
        c->verified = res->verified + a; c->pruned = res->pruned + a;
        c->err = res->err;
        c->acc_row = (ivec *)calloc((size_t)(c->nq + 1), sizeof(ivec));
        c->acc_dis = (dvec *)calloc((size_t)(c->nq + 1), sizeof(dvec));
        scratch_init(&c->s, ml, ds->dim);
        if (mode == MODE_KNN) {
            c->pools = (pool_t *)calloc((size_t)(c->nq + 1), sizeof(pool_t));
            for (i64 q = 0; q < c->nq; q++) {
                i64 k = ks[a + q];
                c->pools[q].k = k;
                c->pools[q].d = (double *)malloc(sizeof(double) * (size_t)k);
                c->pools[q].row = (i64 *)malloc(sizeof(i64) * (size_t)k);
            }
        }
        if (c->nq > 0) {
            if (!pruning) scan_all(c); else search_slice(c);
        }
        slice_peak[w] = c->peak;
    }
    /* collect (search.py:298-314) */
    i64 total = 0;
    for (int w = 0; w < threads; w++) {
        ctx_t *c = &cs[w];
        for (i64 q = 0; q < c->nq; q++)
            total += mode == MODE_KNN ? c->pools[q].cnt : c->acc_row[q].n;
        if (c->status) { res->status = c->status; }
        if (slice_peak[w] > res->peak) res->peak = slice_peak[w];
        for (int l = 0; l < MAX_LAYERS; l++) if (lim[w][l]) res->limits[l] = lim[w][l];
    }
    res->total = total;
    res->ids = (i64 *)malloc(sizeof(i64) * (size_t)(total + 1));
    res->dis = (double *)malloc(sizeof(double) * (size_t)(total + 1));
    i64 o = 0;
    cand_t *tmp = NULL; i64 tcap = 0;
    for (int w = 0; w < threads; w++) {
        ctx_t *c = &cs[w];
        for (i64 q = 0; q < c->nq; q++) {
            i64 qa = c->q0 + q;
            if (mode == MODE_KNN) {
                pool_t *p = &c->pools[q];
                res->counts[qa] = p->cnt;
                for (i64 u = 0; u < p->cnt; u++) { res->ids[o] = ds->ids[p->row[u]]; res->dis[o] = p->d[u]; o++; }
                free(p->d); free(p->row);
            } else {
                i64 m = c->acc_row[q].n;
                if (m > tcap) { tcap = m * 2; tmp = (cand_t *)realloc(tmp, sizeof(cand_t) * (size_t)tcap); }
                for (i64 u = 0; u < m; u++) {
                    tmp[u].d = c->acc_dis[q].v[u]; tmp[u].row = c->acc_row[q].v[u]; tmp[u].id = ds->ids[tmp[u].row];
                }
                qsort(tmp, (size_t)m, sizeof(cand_t), cand_cmp);
                res->counts[qa] = m;
                for (i64 u = 0; u < m; u++) { res->ids[o] = tmp[u].id; res->dis[o] = tmp[u].d; o++; }
                free(c->acc_row[q].v); free(c->acc_dis[q].v);
            }
        }
        free(c->acc_row); free(c->acc_dis); free(c->pools); free(c->cbuf);
        scratch_free(&c->s);
    }
    free(tmp); free(cs); free(slice_peak); free(lim); free(row_dead);
    return res;
}

void orc_result_free(orc_result *r)
{
    if (!r) return;
    free(r->counts); free(r->ids); free(r->dis); free(r->verified); free(r->pruned);
    free(r);
}

/* ------------------------------------------------------------------ */
/* brute force (oracle.py:19-47): scan every live object in id order    */
/* ------------------------------------------------------------------ */

orc_result *orc_brute(const orc_ds *ds, const uint8_t *row_dead, const orc_ds *qs, int mode,
                      const double *radii, const i64 *ks, int threads)
{
    i64 nq = qs->n;
    orc_result *res = (orc_result *)calloc(1, sizeof(orc_result));
    res->nq = nq;
    res->counts = (i64 *)calloc((size_t)(nq + 1), sizeof(i64));
    res->verified = (i64 *)calloc((size_t)(nq + 1), sizeof(i64));
    res->pruned = (i64 *)calloc((size_t)(nq + 1), sizeof(i64));
    cand_t **per = (cand_t **)calloc((size_t)(nq + 1), sizeof(cand_t *));
    i64 ml = max_len(ds), mq = max_len(qs);
    if (mq > ml) ml = mq;
    if (threads < 1) threads = 1;
#ifdef _OPENMP
    #pragma omp parallel num_threads(threads)
#endif
    {
        scratch s;
        scratch_init(&s, ml, ds->dim);
        cand_t *all = (cand_t *)malloc(sizeof(cand_t) * (size_t)(ds->n + 1));
#ifdef _OPENMP
        #pragma omp for schedule(dynamic, 1)
#endif
        for (i64 q = 0; q < nq; q++) {
            i64 m = 0;
            for (i64 r = 0; r < ds->n; r++) {
                if (row_dead && row_dead[r]) continue;
                double d = dist_rq(ds, r, qs, q, &s);
                if (mode == MODE_RANGE && !(d <= radii[q])) continue;
                all[m].d = d; all[m].id = ds->ids[r]; all[m].row = r; m++;
            }
            qsort(all, (size_t)m, sizeof(cand_t), cand_cmp);
            if (mode == MODE_KNN && m > ks[q]) m = ks[q];
            per[q] = (cand_t *)malloc(sizeof(cand_t) * (size_t)(m + 1));
            memcpy(per[q], all, sizeof(cand_t) * (size_t)m);
            res->counts[q] = m;
        }
        free(all);
        scratch_free(&s);
    }
    i64 total = 0;
    for (i64 q = 0; q < nq; q++) total += res->counts[q];
    res->total = total;
    res->ids = (i64 *)malloc(sizeof(i64) * (size_t)(total + 1));
    res->dis = (double *)malloc(sizeof(double) * (size_t)(total + 1));
    i64 o = 0;
    for (i64 q = 0; q < nq; q++) {
        for (i64 u = 0; u < res->counts[q]; u++) { res->ids[o] = per[q][u].id; res->dis[o] = per[q][u].d; o++; }
        free(per[q]);
    }
    free(per);
    return res;
}
