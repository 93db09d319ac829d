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
    if (disc < 0.0) return 0;
    double sd = sqrt(disc);
    double qq = bb >= 0.0 ? -0.5 * (bb + sd) : -0.5 * (bb - sd);
    double r1 = qq / aa;
    double r2 = qq != 0.0 ? (cc - d2) / qq : r1;
    double lo = r1 < r2 ? r1 : r2;
    double hi = r1 > r2 ? r1 : r2;
    if (lo > 1.0 || hi < 0.0) return 0;
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
