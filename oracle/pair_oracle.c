/*
 * pair_oracle.c — plain-C scalar oracle for the distance-threshold search.
 *
 * TEST INFRASTRUCTURE ONLY.  Loaded with ctypes by tests/ (and nothing in
 * the product package) as an independent checker of the CUDA path.
 * Compiled with -ffp-contract=off so every + - * / sqrt is one IEEE-754
 * binary64 operation, exactly like the numpy/Python reference.
 *
 * Restates, operation for operation:
 *   orc_pair            core.py:334-438  temporal_intersection + threshold_interval
 *   orc_floor_divide    numpy npy_divmod / npy_floor_divide (used at index.py:110)
 *   orc_brute_force     oracle.py:23-41  (query-major order)
 *   orc_search_spans    engine.py:97-204 over explicit candidate spans
 *                       (batch order, row-major (entry, query) within a batch)
 * Non-finite intermediates (overflow at |coordinate| ~ 1e154 and above)
 * follow the vectorized pair_intervals (core.py:536-553), the engine's path.
 * where core.py/index.py/oracle.py live under
 * /root/reference/pkg/src/trajseek/.
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by the reference itself (tests/golden/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* A segment is 8 doubles: xs ys zs ts xe ye ze te. */
enum { XS, YS, ZS, TS, XE, YE, ZE, TE };

/* position_at (core.py:309-331) */
static void at_time(const double *s, double t, double p[3]) {
    if (s[TE] == s[TS] || t == s[TS]) {
        p[0] = s[XS]; p[1] = s[YS]; p[2] = s[ZS];
        return;
    }
    if (t == s[TE]) {
        p[0] = s[XE]; p[1] = s[YE]; p[2] = s[ZE];
        return;
    }
    double f = (t - s[TS]) / (s[TE] - s[TS]);
    p[0] = s[XS] + f * (s[XE] - s[XS]);
    p[1] = s[YS] + f * (s[YE] - s[YS]);
    p[2] = s[ZS] + f * (s[ZE] - s[ZS]);
}

/* clip (core.py:350-359): returns start/end positions on [ta, tb] */
static void clip(const double *s, double ta, double tb, double a[3], double b[3]) {
    if (s[TS] == ta && s[TE] == tb) {
        a[0] = s[XS]; a[1] = s[YS]; a[2] = s[ZS];
        b[0] = s[XE]; b[1] = s[YE]; b[2] = s[ZE];
        return;
    }
    at_time(s, ta, a);
    at_time(s, tb, b);
}

/* Returns 1 and the closed proximity interval, or 0 (no hit).  *tmiss is
 * set when the extents do not overlap. */
int orc_pair(const double *A, const double *B, double d, double *begin, double *end,
             int *tmiss) {
    double ta = A[TS] > B[TS] ? A[TS] : B[TS];
    double tb = A[TE] < B[TE] ? A[TE] : B[TE];
    *tmiss = 0;
    if (ta > tb) {
        *tmiss = 1;
        return 0;
    }
    double pa[3], qa[3], pb[3], qb[3];
    clip(A, ta, tb, pa, qa);
    clip(B, ta, tb, pb, qb);
    double span = tb - ta;
    double d2 = d * d;
    double ux = pa[0] - pb[0], uy = pa[1] - pb[1], uz = pa[2] - pb[2];
    double cc = ux * ux + uy * uy + uz * uz;
    if (span == 0.0) {
        if (cc <= d2) { *begin = ta; *end = tb; return 1; }
        return 0;
    }
    double wx = (qa[0] - pa[0]) - (qb[0] - pb[0]);
    double wy = (qa[1] - pa[1]) - (qb[1] - pb[1]);
    double wz = (qa[2] - pa[2]) - (qb[2] - pb[2]);
    double aa = wx * wx + wy * wy + wz * wz;
    double bb = 2.0 * (ux * wx + uy * wy + uz * wz);
    if (aa == 0.0) {
        if (cc <= d2) { *begin = ta; *end = tb; return 1; }
        return 0;
    }
    double disc = bb * bb - 4.0 * aa * (cc - d2);
    /* has_root = disc >= 0.0 (core.py:538): a NaN discriminant is a miss */
    if (!(disc >= 0.0)) return 0;
    double sd = sqrt(disc);
    double qq = bb >= 0.0 ? -0.5 * (bb + sd) : -0.5 * (bb - sd);
    double r1 = qq / aa;
    double r2 = qq != 0.0 ? (cc - d2) / qq : r1;
    /* np.minimum / np.maximum propagate NaN (core.py:545-546), and the hit
     * test (lo <= 1) & (hi >= 0) (core.py:553) then fails; the engine path
     * is the vectorized one, so that is the semantics restated here (the
     * scalar threshold_interval would return a NaN interval instead) */
    double lo, hi;
    if (isnan(r1) || isnan(r2)) {
        lo = hi = NAN;
    } else {
        lo = r1 < r2 ? r1 : r2;
        hi = r1 > r2 ? r1 : r2;
    }
    if (!(lo <= 1.0 && hi >= 0.0)) return 0;
    *begin = lo <= 0.0 ? ta : ta + lo * span;
    *end = hi >= 1.0 ? tb : ta + hi * span;
    return 1;
}

/* numpy floor_divide for float64 (npy_divmod), as used by index.py:110. */
double orc_floor_divide(double a, double b) {
    if (b == 0.0) return a / b;
    double mod = fmod(a, b);
    double div = (a - mod) / b;
    if (mod != 0.0) {
        if ((b < 0.0) != (mod < 0.0)) {
            mod += b;
            div -= 1.0;
        }
    }
    double fl;
    if (div != 0.0) {
        fl = floor(div);
        if (div - fl > 0.5) fl += 1.0;
    } else {
        fl = copysign(0.0, a / b);
    }
    return fl;
}

void orc_floor_divide_many(int64_t n, const double *a, double b, double *out) {
    for (int64_t i = 0; i < n; ++i) out[i] = orc_floor_divide(a[i], b);
}

/* ── brute force, multi-threaded over query ranges ─────────────────────── */

typedef struct {
    const double *const *e; /* 8 column pointers */
    const double *const *q;
    int64_t ne, q_lo, q_hi;
    double d;
    int64_t n, cap;
    int64_t *qi, *ei;
    double *tb, *te;
    int64_t tmiss, smiss;
} bf_task;

static void bf_push(bf_task *t, int64_t qi, int64_t ei, double b, double e) {
    if (t->n == t->cap) {
        t->cap = t->cap ? 2 * t->cap : 1024;
        t->qi = realloc(t->qi, t->cap * sizeof(int64_t));
        t->ei = realloc(t->ei, t->cap * sizeof(int64_t));
        t->tb = realloc(t->tb, t->cap * sizeof(double));
        t->te = realloc(t->te, t->cap * sizeof(double));
    }
    t->qi[t->n] = qi; t->ei[t->n] = ei; t->tb[t->n] = b; t->te[t->n] = e;
    t->n++;
}

static void *bf_run(void *arg) {
    bf_task *t = arg;
    double A[8], B[8];
    for (int64_t i = t->q_lo; i < t->q_hi; ++i) {
        for (int k = 0; k < 8; ++k) A[k] = t->q[k][i];
        for (int64_t j = 0; j < t->ne; ++j) {
            for (int k = 0; k < 8; ++k) B[k] = t->e[k][j];
            double b, e;
            int tm;
            /* oracle.py:35 — the query is the row ("a") operand */
            if (orc_pair(A, B, t->d, &b, &e, &tm)) bf_push(t, i, j, b, e);
            else if (tm) t->tmiss++;
            else t->smiss++;
        }
    }
    return NULL;
}

/* Query-major brute force.  Columns are passed as 8 pointers each
 * (xs ys zs ts xe ye ze te).  Results are returned in malloc'd arrays the
 * caller frees with orc_free.  Returns the hit count. */
int64_t orc_brute_force(int64_t ne, const double *const *ecols, int64_t nq,
                        const double *const *qcols, double d, int nthreads,
                        int64_t **q_ord, int64_t **e_ord, double **t_begin, double **t_end,
                        int64_t *tmiss, int64_t *smiss) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > nq && nq > 0) nthreads = (int)nq;
    bf_task *tasks = calloc(nthreads, sizeof(bf_task));
    pthread_t *th = calloc(nthreads, sizeof(pthread_t));
    for (int k = 0; k < nthreads; ++k) {
        tasks[k].e = ecols; tasks[k].q = qcols; tasks[k].ne = ne; tasks[k].d = d;
        tasks[k].q_lo = nq * k / nthreads;
        tasks[k].q_hi = nq * (k + 1) / nthreads;
        pthread_create(&th[k], NULL, bf_run, &tasks[k]);
    }
    int64_t total = 0;
    *tmiss = *smiss = 0;
    for (int k = 0; k < nthreads; ++k) {
        pthread_join(th[k], NULL);
        total += tasks[k].n;
        *tmiss += tasks[k].tmiss;
        *smiss += tasks[k].smiss;
    }
    *q_ord = malloc((total + 1) * sizeof(int64_t));
    *e_ord = malloc((total + 1) * sizeof(int64_t));
    *t_begin = malloc((total + 1) * sizeof(double));
    *t_end = malloc((total + 1) * sizeof(double));
    int64_t at = 0;
    for (int k = 0; k < nthreads; ++k) {
        bf_task *t = &tasks[k];
        if (t->n) {
            memcpy(*q_ord + at, t->qi, t->n * sizeof(int64_t));
            memcpy(*e_ord + at, t->ei, t->n * sizeof(int64_t));
            memcpy(*t_begin + at, t->tb, t->n * sizeof(double));
            memcpy(*t_end + at, t->te, t->n * sizeof(double));
        }
        at += t->n;
        free(t->qi); free(t->ei); free(t->tb); free(t->te);
    }
    free(tasks);
    free(th);
    return total;
}

void orc_free(void *p) { free(p); }

/* ── engine over explicit spans (engine.py:97-204), multi-threaded ──────────
 *
 * Batch b holds query ordinals lo[b]..hi[b] and candidate entry ordinals
 * first[b]..last[b] (first < 0: no candidates, engine.py:180-182).  Each
 * batch is the reference mesh pair_intervals(rows = its candidates,
 * cols = its queries) (engine.py:89, core.py:464): hits come back per
 * batch in row-major (entry, query) order, batches in the given order —
 * the reference engine's item order.  Work is cut into (batch, entry
 * chunk) units claimed by nthreads workers; results are concatenated in
 * unit order, which keeps that order.  Per batch: hits, temporal misses,
 * spatial misses (core.py:489-496, 560). */

typedef struct {
    int64_t b, e0, e1; /* batch, entry range [e0, e1) */
    int64_t n, cap;
    int64_t *qi, *ei;
    double *tb, *te;
    int64_t tmiss, smiss;
} os_unit;

typedef struct {
    const double *const *e;
    const double *const *q;
    const int64_t *lo, *hi;
    double d;
    os_unit *units;
    int64_t nunits;
    int64_t next; /* claimed with __atomic_fetch_add */
} os_job;

static void os_push(os_unit *u, int64_t qi, int64_t ei, double b, double e) {
    if (u->n == u->cap) {
        u->cap = u->cap ? 2 * u->cap : 256;
        u->qi = realloc(u->qi, u->cap * sizeof(int64_t));
        u->ei = realloc(u->ei, u->cap * sizeof(int64_t));
        u->tb = realloc(u->tb, u->cap * sizeof(double));
        u->te = realloc(u->te, u->cap * sizeof(double));
    }
    u->qi[u->n] = qi; u->ei[u->n] = ei; u->tb[u->n] = b; u->te[u->n] = e;
    u->n++;
}

static void *os_run(void *arg) {
    os_job *J = arg;
    double A[8], B[8];
    for (;;) {
        int64_t k = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
        if (k >= J->nunits) break;
        os_unit *u = &J->units[k];
        const int64_t qlo = J->lo[u->b], qhi = J->hi[u->b];
        for (int64_t j = u->e0; j < u->e1; ++j) {
            for (int c = 0; c < 8; ++c) A[c] = J->e[c][j];
            for (int64_t i = qlo; i <= qhi; ++i) {
                for (int c = 0; c < 8; ++c) B[c] = J->q[c][i];
                double tb, te;
                int tm;
                /* the entry is the row ("a") operand, engine.py:89 */
                if (orc_pair(A, B, J->d, &tb, &te, &tm)) os_push(u, i, j, tb, te);
                else if (tm) u->tmiss++;
                else u->smiss++;
            }
        }
    }
    return NULL;
}

/* Returns the total hit count; per_batch receives nb x 3 (hits, temporal
 * misses, spatial misses); result arrays are malloc'd (orc_free). */
int64_t orc_search_spans(const double *const *ecols, const double *const *qcols, int64_t nb,
                         const int64_t *lo, const int64_t *hi, const int64_t *first,
                         const int64_t *last, double d, int nthreads, int64_t chunk_pairs,
                         int64_t *per_batch, int64_t **q_ord, int64_t **e_ord, double **t_begin,
                         double **t_end) {
    if (nthreads < 1) nthreads = 1;
    if (chunk_pairs < 1) chunk_pairs = 1 << 20;
    int64_t nunits = 0;
    for (int64_t b = 0; b < nb; ++b) {
        if (first[b] < 0) continue;
        const int64_t s = hi[b] - lo[b] + 1, c = last[b] - first[b] + 1;
        int64_t step = chunk_pairs / s;
        if (step < 1) step = 1;
        nunits += (c + step - 1) / step;
    }
    os_unit *units = calloc(nunits + 1, sizeof(os_unit));
    int64_t k = 0;
    for (int64_t b = 0; b < nb; ++b) {
        if (first[b] < 0) continue;
        const int64_t s = hi[b] - lo[b] + 1;
        int64_t step = chunk_pairs / s;
        if (step < 1) step = 1;
        for (int64_t e0 = first[b]; e0 <= last[b]; e0 += step) {
            units[k].b = b;
            units[k].e0 = e0;
            units[k].e1 = e0 + step <= last[b] + 1 ? e0 + step : last[b] + 1;
            ++k;
        }
    }
    os_job J = {ecols, qcols, lo, hi, d, units, nunits, 0};
    if (nthreads > nunits) nthreads = nunits > 0 ? (int)nunits : 1;
    pthread_t *th = calloc(nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, os_run, &J);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    memset(per_batch, 0, (size_t)nb * 3 * sizeof(int64_t));
    int64_t total = 0;
    for (k = 0; k < nunits; ++k) {
        per_batch[units[k].b * 3 + 0] += units[k].n;
        per_batch[units[k].b * 3 + 1] += units[k].tmiss;
        per_batch[units[k].b * 3 + 2] += units[k].smiss;
        total += units[k].n;
    }
    *q_ord = malloc((total + 1) * sizeof(int64_t));
    *e_ord = malloc((total + 1) * sizeof(int64_t));
    *t_begin = malloc((total + 1) * sizeof(double));
    *t_end = malloc((total + 1) * sizeof(double));
    int64_t at = 0;
    for (k = 0; k < nunits; ++k) {
        os_unit *u = &units[k];
        if (u->n) {
            memcpy(*q_ord + at, u->qi, u->n * sizeof(int64_t));
            memcpy(*e_ord + at, u->ei, u->n * sizeof(int64_t));
            memcpy(*t_begin + at, u->tb, u->n * sizeof(double));
            memcpy(*t_end + at, u->te, u->n * sizeof(double));
        }
        at += u->n;
        free(u->qi); free(u->ei); free(u->tb); free(u->te);
    }
    free(units);
    return total;
}
