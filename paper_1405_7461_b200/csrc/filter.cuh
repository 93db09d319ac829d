// filter.cuh — K1's conservative FP64 pair filter (host + device).
//
// The common path of K1 only has to decide which (candidate, query) pairs
// could have a non-negative reference discriminant (core.py:533-537); the
// flagged ones are recomputed with the reference's exact operation sequence
// (pair_eval in k1_pairs.cu).  This header holds the filter arithmetic as a
// pure function so tools/filter_check.cu can test it on the CPU against the
// exact restatement (oracle/pair_oracle.c) on adversarial pairs.
//
// Velocity form.  Each segment carries v = RN(d * RN(1/ext)) (0 for a
// waypoint).  With delta = cts - r.ts and the shared span [ta, tb]:
//   u = (r.s - c.s) + delta * v_late      (separation at ta; v_late is the
//                                          velocity of the earlier starter)
//   w = (tb - ta) * (r.v - c.v)           (change of separation over the span)
// and for a query inside every candidate's span (TA_R/TB_R)
//   w = c.ext * r.v - c.d                 (query endpoints taken verbatim).
// A zero-length span gives w = 0 exactly, hence aa = dot = 0 and the test
// below passes: flat pairs are flagged with no separate time comparison,
// except in TA_R/TB_R, where the query's own ext == 0 is tested.
//
// Error bound.  For overlapping pairs of a launch with C = max |coordinate|
// (C <= 2^250, d <= 2^250, C == 0 or C >= 2^-200; otherwise K1 runs the
// exact path everywhere) and segments inside the exponent window of
// seg_unsafe() (db.cu), the filter's u and w are within eu <= 23 ulp(C)
// ~ 2^-48.5 C and ew <= 64 ulp(C) ~ 2^-47 C per component of the
// reference's U and W.  Writing D(U,W) = (U.W)^2 - |W|^2 (|U|^2 - d^2)
// = d^2 |W|^2 - |U x W|^2:
//   |D(u,w) - D(U,W)| <= 2|U||W|^2 |a| + (|U|^2 + d^2) 2|W||b| + h.o.
//                     <= 2^-45 C^2 aa + (cc + d^2)(2^-35 aa + 2^-57.4 C^2)
// (|a| <= sqrt3 eu, |b| <= sqrt3 ew, 2|W||b| <= 2^-35 |W|^2 + 2^35 |b|^2),
// and both roundings of the discriminant (the reference's and ours) are
// below 2^-48 aa (cc + d^2).  The test
//   t = dot^2 - aa e + 2^-35 aa s + KA aa + KC s >= 0,   s = cc + d^2,
//   KA = 2^-40 C^2,  KC = 2^-54 C^2
// therefore holds whenever the reference's discriminant is >= 0.  It is
// evaluated as
//   x  = fma(e, 2^-35 - 1, 2^-34 d^2 + KA)          (= 2^-35 s - e + KA)
//   t  = fma(aa, x, dot^2)
//   t2 = fma(KC, e, t)  >=  -2 KC d^2
// whose own roundings are below 2^-50 aa s + 2^-52 |t|, inside the slack.
#pragma once

#include <math.h>
#include <cfenv>

#ifdef __CUDACC__
#define TSK_HD __host__ __device__ __forceinline__
#else
#define TSK_HD inline
#endif

namespace tsk {

// Clip-at-ta cases of a query against a warp's candidates.  Queries in a
// tile are sorted by start time, so each case is a contiguous j range:
//   TA_C    cts <  every candidate's ts: the query started first
//   TA_R    cts >  every candidate's ts: the entry started first
//   TA_BOTH otherwise (decided per pair)
enum { TA_C = 0, TA_R = 1, TA_BOTH = 2 };
// Clip-at-tb cases; TB_R / TB_C are proven for a whole j range from the
// tile's running max / suffix min of query end times, TB_DYN decides per
// query (cte < min te: TB_R, cte > max te: TB_C, else per pair).
enum { TB_R = 0, TB_C = 1, TB_DYN = 2 };

// Filter view of a candidate (held in registers).
struct CandF {
    double ts, te, ext, sx, sy, sz, vx, vy, vz;
};

// Filter view of a query (read from its shared-memory record).
struct QF {
    double ts, te, sx, sy, sz, ext, vx, vy, vz, dx, dy, dz;
};

struct FilterK {
    double d2, k5, kc, t0, km;  // km = 2^-35 - 1
};

TSK_HD FilterK filter_consts(double cmax, double d2) {
    const double c2 = cmax * cmax;
    FilterK k;
    k.d2 = d2;
    const double ka = 0x1p-40 * c2;
    k.kc = 0x1p-54 * c2;
    k.k5 = fma(0x1p-34, d2, ka);
    k.t0 = -2.0 * k.kc * d2;
    k.km = 0x1p-35 - 1.0;
    return k;
}

// Launch-level validity of the filter's error bound (else: exact path only).
// a >= b as its own compare: keeps the per-candidate tests separate (the
// compiler otherwise merges `x >= t || y >= t` into a max + compare)
TSK_HD bool ge_sep(double a, double b) {
#ifdef __CUDA_ARCH__
    unsigned r;
    asm("{.reg .pred p; setp.ge.f64 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(r) : "d"(a), "d"(b));
    return r != 0;
#else
    return a >= b;
#endif
}

TSK_HD bool filter_ok(double cmax, double d2) {
    return cmax <= 0x1p250 && d2 <= 0x1p500 && (cmax == 0.0 || cmax >= 0x1p-200);
}

// Launch-level validity of K1's FP32 path: |coordinates| and d below 2^60
// inside the FP64 filter's window.  The box-cull fast path and the external
// overlap count (layout.cu) run exactly when this holds.
TSK_HD bool k1f_launch_ok(double cmax, double d2) {
    return filter_ok(cmax, d2) && d2 <= 0x1p120 && cmax <= 0x1p60;
}

// velocity component of a hoisted segment: RN(d * rcp), rcp = RN(1/ext) or 0
TSK_HD double seg_velocity(double d, double rcp) { return d * rcp; }

template <int TA, int TB>
TSK_HD bool pair_filter(const CandF &r, const QF &Q, double wmin_te, double wmax_te, const FilterK &K) {
    const double rv[3] = {r.vx, r.vy, r.vz}, qv[3] = {Q.vx, Q.vy, Q.vz};
    const double ds[3] = {r.sx - Q.sx, r.sy - Q.sy, r.sz - Q.sz};
    const double dl = Q.ts - r.ts;
    double u[3], ta;
    if (TA == TA_R) {
        ta = Q.ts;
        for (int i = 0; i < 3; ++i) u[i] = fma(dl, rv[i], ds[i]);
    } else if (TA == TA_C) {
        ta = r.ts;
        for (int i = 0; i < 3; ++i) u[i] = fma(dl, qv[i], ds[i]);
    } else {
        const bool qlate = dl >= 0.0;
        ta = qlate ? Q.ts : r.ts;
        for (int i = 0; i < 3; ++i) u[i] = fma(dl, qlate ? rv[i] : qv[i], ds[i]);
    }
    const bool tb_r = TB == TB_R || (TB == TB_DYN && Q.te < wmin_te);
    const bool tb_c = !tb_r && (TB == TB_C || (TB == TB_DYN && Q.te > wmax_te));
    double w[3];
    bool flat = false;
    if (TA == TA_R && tb_r) {
        const double qd[3] = {Q.dx, Q.dy, Q.dz};
        for (int i = 0; i < 3; ++i) w[i] = fma(Q.ext, rv[i], -qd[i]);
        flat = Q.ext == 0.0;
    } else {
        double span;
        if (tb_r) span = Q.te - ta;
        else if (tb_c) span = TA == TA_C ? r.ext : r.te - ta;
        else span = (r.te < Q.te ? r.te : Q.te) - ta;
        for (int i = 0; i < 3; ++i) w[i] = span * (rv[i] - qv[i]);
    }
    const double e = fma(u[0], u[0], fma(u[1], u[1], fma(u[2], u[2], -K.d2)));
    const double aa = fma(w[0], w[0], fma(w[1], w[1], w[2] * w[2]));
    const double dot = fma(u[0], w[0], fma(u[1], w[1], u[2] * w[2]));
    const double x = fma(e, K.km, K.k5);
    const double t = fma(aa, x, dot * dot);
    const double t2 = fma(K.kc, e, t);
    return flat || ge_sep(t2, K.t0);
}


// ── FP32 pre-filter (K1's common path) ─────────────────────────────────────
//
// Per work item, positions and times are taken relative to an origin
// (O, T0) = the first staged query's start.  A candidate holds
//   p  = RN32((r.s - O) - (r.ts - T0) v_r)   (its line at time T0)
//   v  = RN32(v_r),  sr >= |v_r| (rounded up)
// and a query
//   ts = RN32(q.ts - T0), s = RN32(q.s - O),
//   a >= (1 + 2^-8) ext_q,  b >= (1 + 2^-8)(d + |q.e - q.s|) + delta.
// Then u = (p + ts v) - s approximates u* = r.s + (q.ts - r.ts) V_r - q.s,
// the separation of the candidate's line from the query's start at q.ts.
//
// Why |u| > a sr + b implies a reference miss.  On the shared span
// [ta, tb] (inside [q.ts, q.te]) both segments are linear, so the true
// separation s(t) = u* + (t - q.ts)(V_r - V_q) and
//   |s(t)| >= |u*| - ext_q |V_r| - |q.e - q.s|.
// A reference hit needs some lambda in [0, 1] with its computed quadratic
// q(lambda) = |U + lambda W|^2 - d^2 <= mu (d^2 + (|U| + |W|)^2), mu = 2^-20
// far above the roundings of its coefficients, discriminant and roots (the
// rare path's second filter rests on the same fact with mu = 2^-30), with
// U, W the reference's separation at ta and change over the span, within
// 2^-48 C of the true ones.  That gives
//   (1 - 2^-10)|U| <= (1 + 2^-20) d + (1 + 2^-10)|W|,
// so a hit is impossible once |u*| > (1 + 2^-8)(d + ext_q|V_r| + |q.e - q.s|)
// + 2^-38 C.  FP32 error: every magnitude the FP32 path forms is, per
// component, at most M = A_r + TV_r + T_q V_r + A_q (A: max |s - O| of the
// item's candidates / queries, TV_r: max |r.ts - T0| |v_r|, T_q: max
// |q.ts - T0|, V_r: max |v_r| component) and each of p, ts*v, t, s, u is
// rounded once, so |u - u*| <= 7 * 2^-24 M < 2^-18 M.  delta adds 2^-18 M
// + 2^-38 C + 2^-100 (underflow).  The test itself uses |u|^2 rounded down
// and (a sr + b)^2 rounded up.  Items with M, V_r or ext_q above 2^60 (or
// d above 2^60) are evaluated exactly instead.
struct CandF32 {
    float px, py, pz, vx, vy, vz, sr;
};

struct F32Item {
    double ox, oy, oz, t0, delta;
    bool ok;
    float sep_rb;  // the separating-axis stage's per-item radius (f32_sep_rbase; set by K1)
};

#ifndef __CUDA_ARCH__
inline float tsk_f2f_ru(double x) {
    float f = (float)x;
    if ((double)f < x) f = nextafterf(f, INFINITY);
    return f;
}
#endif
#ifdef __CUDA_ARCH__
#define TSK_F2F_RN(x) __double2float_rn(x)
#define TSK_F2F_RU(x) __double2float_ru(x)
#else
#define TSK_F2F_RN(x) ((float)(x))
#define TSK_F2F_RU(x) tsk_f2f_ru(x)
#endif

// Item bounds (see above): ar = A_r, tvr = TV_r, vr = V_r, aq = A_q,
// tq = T_q, eq = max ext_q, cmax = max |coordinate| of the launch.
// tr = max |r.ts - T0| of the candidates (the K1 layout's group origins
// are candidates' starts: their FP32 records are re-based per item).
TSK_HD F32Item f32_item(double ox, double oy, double oz, double t0, double ar, double tvr, double vr,
                        double aq, double tq, double eq, double cmax, double tr = 0.0) {
    F32Item it;
    it.ox = ox; it.oy = oy; it.oz = oz; it.t0 = t0;
    const double M = ar + tvr + tq * vr + aq + tr * vr;
    it.ok = M <= 0x1p60 && vr <= 0x1p60 && eq <= 0x1p60;  // false for NaN
    it.delta = 0x1p-18 * M + 0x1p-38 * cmax + 0x1p-100;
    it.sep_rb = INFINITY;  // no separating-axis rejections until K1 sets it
    return it;
}

// FP32 view of a query (sx.. its start, ext = RN(te - ts), dx.. = RN(e - s));
// dthr = d.
TSK_HD void f32_query(double ts, double sx, double sy, double sz, double ext, double dx, double dy,
                      double dz, const F32Item &it, double dthr, float out[6]) {
    const double lq = sqrt(dx * dx + dy * dy + dz * dz) * (1.0 + 0x1p-40);
    out[0] = TSK_F2F_RN(ts - it.t0);
    out[1] = TSK_F2F_RN(sx - it.ox);
    out[2] = TSK_F2F_RN(sy - it.oy);
    out[3] = TSK_F2F_RN(sz - it.oz);
    out[4] = TSK_F2F_RU(ext * (1.0 + 0x1p-8));
    out[5] = TSK_F2F_RU((1.0 + 0x1p-8) * (dthr + lq) + it.delta);
}

// sr >= |v| in FP32 (rounded up); hoisted per entry at upload.
TSK_HD float f32_speed(double vx, double vy, double vz) {
    return TSK_F2F_RU(sqrt(vx * vx + vy * vy + vz * vz) * (1.0 + 0x1p-40));
}

// FP32 view of a candidate (its start, start time and hoisted velocity;
// sr = f32_speed of the velocity).
TSK_HD CandF32 f32_cand_sr(double ts, double sx, double sy, double sz, double vx, double vy, double vz, float sr,
                           const F32Item &it) {
    CandF32 c;
    const double dt = ts - it.t0;
    c.px = TSK_F2F_RN(fma(-dt, vx, sx - it.ox));
    c.py = TSK_F2F_RN(fma(-dt, vy, sy - it.oy));
    c.pz = TSK_F2F_RN(fma(-dt, vz, sz - it.oz));
    c.vx = TSK_F2F_RN(vx);
    c.vy = TSK_F2F_RN(vy);
    c.vz = TSK_F2F_RN(vz);
    c.sr = sr;
    return c;
}

// The K1 layout stores every candidate's FP32 view once, relative to its
// BOX_GROUP's origin (O_g, T_g) = the start of the group's first entry
// (f32_cand_sr with that origin: pg, v, sr).  An item re-bases it to its own
// origin (O, T0):
//   p = RN32(RN32(pg + dO) - dT v),  dO = RN32(O_g - O), dT = RN32(T_g - T0)
// (one FFMA), for the line (r.s - O) - (r.ts - T0) v_r of the direct form.
// Error: pg, dO, the sum, dT, v and the FFMA are each rounded once, on
// magnitudes at most |r.s - O_g| + |r.ts - T_g| V_r, A_r, A_r + |r.ts - T_g|
// V_r, T_r V_r and A_r + TV_r (O_g is a candidate's start, so |O_g - O| <=
// A_r and |T_g - T0| <= T_r = max |r.ts - T0|), so |p - p*| <= 16 2^-24 M
// with M += T_r V_r (f32_item's tr): inside delta = 2^-18 M, which the
// direct form (7 2^-24 M) left 9x slack for.  tools/filter_check.cpp runs
// the pre-filter and the separating-axis stage on re-based candidates.
TSK_HD CandF32 f32_cand_rebase(float pgx, float pgy, float pgz, float vx, float vy, float vz, float sr, float dox,
                               float doy, float doz, float dt) {
    CandF32 c;
#ifdef __CUDA_ARCH__
    c.px = __fmaf_rn(-dt, vx, __fadd_rn(pgx, dox));
    c.py = __fmaf_rn(-dt, vy, __fadd_rn(pgy, doy));
    c.pz = __fmaf_rn(-dt, vz, __fadd_rn(pgz, doz));
#else
    c.px = fmaf(-dt, vx, pgx + dox);
    c.py = fmaf(-dt, vy, pgy + doy);
    c.pz = fmaf(-dt, vz, pgz + doz);
#endif
    c.vx = vx; c.vy = vy; c.vz = vz;
    c.sr = sr;
    return c;
}

// FP32 view of a candidate (its start, start time and hoisted velocity).
TSK_HD CandF32 f32_cand(double ts, double sx, double sy, double sz, double vx, double vy, double vz,
                        const F32Item &it) {
    CandF32 c;
    const double dt = ts - it.t0;
    c.px = TSK_F2F_RN(fma(-dt, vx, sx - it.ox));
    c.py = TSK_F2F_RN(fma(-dt, vy, sy - it.oy));
    c.pz = TSK_F2F_RN(fma(-dt, vz, sz - it.oz));
    c.vx = TSK_F2F_RN(vx);
    c.vy = TSK_F2F_RN(vy);
    c.vz = TSK_F2F_RN(vz);
    c.sr = f32_speed(vx, vy, vz);
    return c;
}

#ifndef __CUDA_ARCH__
inline float tsk_fma_dir(float a, float b, float c, int mode) {
    const int m = fegetround();
    fesetround(mode);
    volatile float r = fmaf(a, b, c);
    fesetround(m);
    return r;
}
#endif

// |u|^2 of the pre-filter test, rounded down.
TSK_HD float f32_n2(const CandF32 &c, float qts, float qx, float qy, float qz) {
#ifdef __CUDA_ARCH__
    const float ux = __fsub_rn(__fmaf_rn(qts, c.vx, c.px), qx);
    const float uy = __fsub_rn(__fmaf_rn(qts, c.vy, c.py), qy);
    const float uz = __fsub_rn(__fmaf_rn(qts, c.vz, c.pz), qz);
    return __fmaf_rd(uz, uz, __fmaf_rd(uy, uy, __fmul_rd(ux, ux)));
#else
    const float ux = fmaf(qts, c.vx, c.px) - qx;
    const float uy = fmaf(qts, c.vy, c.py) - qy;
    const float uz = fmaf(qts, c.vz, c.pz) - qz;
    return tsk_fma_dir(uz, uz, tsk_fma_dir(uy, uy, tsk_fma_dir(ux, ux, 0.f, FE_DOWNWARD), FE_DOWNWARD),
                       FE_DOWNWARD);
#endif
}

// ── box cull (K1 layout) ───────────────────────────────────────────────────
//
// While both segments of a pair are active each moving point lies on its own
// segment, so the pair's separation h(t) is at least the gap G between the
// two segments' bounding boxes.  A reference hit needs some lambda in [0, 1]
// with |U + lambda W|^2 <= d^2 + mu (d^2 + (|U| + |W|)^2), mu = 2^-24 (U, W:
// separation at ta and its change over the span; mu is far above the
// reference's roundings, see the FP32 pre-filter below), so
//   G <= h <= (1 + 2^-11) d + 2^-12 (|U| + |W|) + 2^-40 C.
// The error term grows with |U| + |W|, not with d: long motion crossing the
// query with a perpendicular offset h below the rounding of |U|^2 is a
// reference hit at any d (cc = |U|^2 absorbs h^2; tools/filter_check.cpp
// mode 8).  Both ends of U and U + W lie in the boxes, so |U| + |W| <=
// 3 (G + D), D = the sum of the two boxes' diagonals, and a hit needs
//   G <= R = (1 + 2^-8) d + 2^-10 D + 2^-29 C      (C: max |coordinate|).
// Boxes are rounded outward to FP32; the gap, its square and sum are rounded
// down, so the tested value never exceeds the true G^2; R and R^2 are rounded
// up.  tools/filter_check.cpp checks this on the adversarial pairs (no
// reference hit is ever culled) and that dropping the D term misses.
//
// The launch-level part of R: (1 + 2^-8) d + 2^-29 C, rounded up.
TSK_HD float box_cull_rbase(double d, double cmax) {
    const double r = (1.0 + 0x1p-8) * d + 0x1p-29 * cmax + 0x1p-100;
    return TSK_F2F_RU(r * (1.0 + 0x1p-40));
}

#ifndef __CUDA_ARCH__
inline float tsk_add_dir(float a, float b, int mode) { return tsk_fma_dir(1.0f, a, b, mode); }
#endif

// A box's share of R: 2^-10 of its diagonal, rounded up.
TSK_HD float box_cull_dterm(float lx, float ly, float lz, float hx, float hy, float hz) {
#ifdef __CUDA_ARCH__
    const float dx = __fsub_ru(hx, lx), dy = __fsub_ru(hy, ly), dz = __fsub_ru(hz, lz);
    return __fmul_ru(0x1p-10f, __fsqrt_ru(__fmaf_ru(dz, dz, __fmaf_ru(dy, dy, __fmul_ru(dx, dx)))));
#else
    const float dx = tsk_add_dir(hx, -lx, FE_UPWARD), dy = tsk_add_dir(hy, -ly, FE_UPWARD),
                dz = tsk_add_dir(hz, -lz, FE_UPWARD);
    const float s = tsk_fma_dir(dz, dz, tsk_fma_dir(dy, dy, tsk_fma_dir(dx, dx, 0.f, FE_UPWARD), FE_UPWARD),
                                FE_UPWARD);
    float r = std::sqrt(s);
    if ((double)r * (double)r < (double)s) r = nextafterf(r, INFINITY);
    return tsk_fma_dir(0x1p-10f, r, 0.f, FE_UPWARD);
#endif
}

// R^2 of one (candidate box, query box) test, rounded up.
TSK_HD float box_cull_r2(float rbase, float dterm_a, float dterm_b) {
#ifdef __CUDA_ARCH__
    const float R = __fadd_ru(__fadd_ru(rbase, dterm_a), dterm_b);
    return __fmul_ru(R, R);
#else
    const float R = tsk_add_dir(tsk_add_dir(rbase, dterm_a, FE_UPWARD), dterm_b, FE_UPWARD);
    return tsk_fma_dir(R, R, 0.f, FE_UPWARD);
#endif
}

#ifndef __CUDA_ARCH__
inline float tsk_f2f_rd(double x) {
    float f = (float)x;
    if ((double)f > x) f = nextafterf(f, -INFINITY);
    return f;
}
#endif
#ifdef __CUDA_ARCH__
#define TSK_F2F_RD(x) __double2float_rd(x)
#else
#define TSK_F2F_RD(x) tsk_f2f_rd(x)
#endif

// squared gap between boxes [gl, gh] and [ql, qh] (per axis), rounded down
TSK_HD float box_gap2(float glx, float gly, float glz, float ghx, float ghy, float ghz, float qlx, float qly,
                      float qlz, float qhx, float qhy, float qhz) {
#ifdef __CUDA_ARCH__
    const float gx = fmaxf(fmaxf(__fsub_rd(glx, qhx), __fsub_rd(qlx, ghx)), 0.f);
    const float gy = fmaxf(fmaxf(__fsub_rd(gly, qhy), __fsub_rd(qly, ghy)), 0.f);
    const float gz = fmaxf(fmaxf(__fsub_rd(glz, qhz), __fsub_rd(qlz, ghz)), 0.f);
    return __fmaf_rd(gz, gz, __fmaf_rd(gy, gy, __fmul_rd(gx, gx)));
#else
    auto sub = [](float a, float b) { return tsk_fma_dir(1.0f, a, -b, FE_DOWNWARD); };
    const float gx = std::fmax(std::fmax(sub(glx, qhx), sub(qlx, ghx)), 0.f);
    const float gy = std::fmax(std::fmax(sub(gly, qhy), sub(qly, ghy)), 0.f);
    const float gz = std::fmax(std::fmax(sub(glz, qhz), sub(qlz, ghz)), 0.f);
    return tsk_fma_dir(gz, gz, tsk_fma_dir(gy, gy, tsk_fma_dir(gx, gx, 0.f, FE_DOWNWARD), FE_DOWNWARD),
                       FE_DOWNWARD);
#endif
}

#ifdef __CUDACC__
// box_gap2 of one box [g] against two query boxes at once (FADD2 / FFMA2 /
// FMUL2 with the same directed roundings per element: each half equals the
// scalar form bit for bit, so the cull's proof is unchanged).
__device__ __forceinline__ float2 box_gap2_x2(float glx, float gly, float glz, float ghx, float ghy, float ghz,
                                              float2 qlx, float2 qly, float2 qlz, float2 qhx, float2 qhy, float2 qhz) {
    const float2 a0 = __fadd2_rd(make_float2(glx, glx), make_float2(-qhx.x, -qhx.y));
    const float2 a1 = __fadd2_rd(qlx, make_float2(-ghx, -ghx));
    const float2 b0 = __fadd2_rd(make_float2(gly, gly), make_float2(-qhy.x, -qhy.y));
    const float2 b1 = __fadd2_rd(qly, make_float2(-ghy, -ghy));
    const float2 c0 = __fadd2_rd(make_float2(glz, glz), make_float2(-qhz.x, -qhz.y));
    const float2 c1 = __fadd2_rd(qlz, make_float2(-ghz, -ghz));
    const float2 gx = make_float2(fmaxf(fmaxf(a0.x, a1.x), 0.f), fmaxf(fmaxf(a0.y, a1.y), 0.f));
    const float2 gy = make_float2(fmaxf(fmaxf(b0.x, b1.x), 0.f), fmaxf(fmaxf(b0.y, b1.y), 0.f));
    const float2 gz = make_float2(fmaxf(fmaxf(c0.x, c1.x), 0.f), fmaxf(fmaxf(c0.y, c1.y), 0.f));
    return __ffma2_rd(gz, gz, __ffma2_rd(gy, gy, __fmul2_rd(gx, gx)));
}
#endif

// Two candidates of a lane in packed form: component c of candidates k0/k1
// in one float2 (sm_100's FFMA2 / FADD2 / FMUL2 then issue one instruction
// for both, the query's scalar broadcast as the .F32 operand).
#ifdef __CUDACC__
struct CandF32x2 {
    float2 px, py, pz, vx, vy, vz;
};

// f32_n2 of two candidates at once: the same IEEE operations, per half, in
// the same order and rounding (u = RN(RN(ts v + p) - s); |u|^2 rounded
// down), so every flag equals the scalar form's (and the margin proof,
// which is about that operation sequence, is unchanged).
__device__ __forceinline__ float2 f32_n2x2(const CandF32x2 &c, float qts, float qx, float qy, float qz) {
    const float2 t = make_float2(qts, qts);
    const float2 ux = __fadd2_rn(__ffma2_rn(t, c.vx, c.px), make_float2(-qx, -qx));
    const float2 uy = __fadd2_rn(__ffma2_rn(t, c.vy, c.py), make_float2(-qy, -qy));
    const float2 uz = __fadd2_rn(__ffma2_rn(t, c.vz, c.pz), make_float2(-qz, -qz));
    return __ffma2_rd(uz, uz, __ffma2_rd(uy, uy, __fmul2_rd(ux, ux)));
}
#endif

// n > R2: the pair cannot hit (false for NaN, so NaN flags).
TSK_HD bool f32_far(float n, float R2) {
#ifdef __CUDA_ARCH__
    unsigned far;
    asm("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(far) : "f"(n), "f"(R2));
    return far != 0u;
#else
    return n > R2;
#endif
}

// min that propagates NaN (a NaN norm must keep its query flagged).
TSK_HD float f32_min_nan(float a, float b) {
#ifdef __CUDA_ARCH__
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
#else
    return (a != a || b != b) ? NAN : (a < b ? a : b);
#endif
}

// The pre-filter test against a given R2 >= (a sr + b)^2 (rounded up):
// true = the pair may hit (NaN flags).  K1 passes one R2 per (query, lane),
// computed with the largest sr of the lane's candidates (R grows with sr,
// so each pair's own test below is implied).
TSK_HD bool f32_flag_r2(const CandF32 &c, float qts, float qx, float qy, float qz, float R2) {
    return !f32_far(f32_n2(c, qts, qx, qy, qz), R2);
}

// (a sr + b)^2 rounded up
TSK_HD float f32_r2(float qa, float sr, float qb) {
#ifdef __CUDA_ARCH__
    const float R = __fmaf_ru(qa, sr, qb);
    return __fmul_ru(R, R);
#else
    const float R = tsk_fma_dir(qa, sr, qb, FE_UPWARD);
    return tsk_fma_dir(R, R, 0.f, FE_UPWARD);
#endif
}

// ── FP32 separating-axis test (second stage of the pre-filter) ───────────
//
// The pre-filter's triangle bound flags every pair whose candidate line
// passes within ext_q |V_r| + |q.e - q.s| + d of the query's start; with
// segments much longer than d most flagged pairs are misses.  Before a
// flagged pair reaches the exact path this test follows both motions over
// the query's whole span [q.ts, q.te] (a superset of the shared span; the
// candidate's line is extended): the relative position runs along the
// segment from D(q.ts) = u to D(q.te) = e, with
//   u = (p + ts v) - s      (the pre-filter's own u, same operations)
//   e = (p + te v) - e_q    (te = RN32(q.te - T0), e_q = RN32(q.e - O)).
// For any direction n, n . D(t) >= min(n . u, n . e) on the segment (it is
// linear in t), so min(n . u, n . e) > R |n| proves |D(t)| > R throughout.
// n = u + lambda w (w = e - u, lambda ~ the closest point, any value is
// valid) makes the test tight.
//
// Why R suffices.  A reference hit needs some instant of the shared span
// with separation h <= (1 + 2^-11) d + 2^-12 (|U| + |W|) + 2^-40 C (the
// mu = 2^-24 statement of the box cull), and |U| + |W| <= 3 max(|D(q.ts)|,
// |D(q.te)|) by convexity.  FP32 error: every value formed is, per
// component, at most M2 = A_r + TV_r + (T_q + E_q + T_r) V_r + A_q + D_q
// (D_q: max |q.e - q.s| component, E_q: max ext_q; T_r V_r covers the
// re-based candidate records) and each of p, v, ts,
// te, s, e_q, the products and sums is rounded once, so u and e are within
// 2^-19 M2 (Euclidean) of the exact D; the dot products n . u, n . e are
// within 2^-22 |n| m (m: the larger Euclidean norm of u, e, bounded by
// 2 max |component|).  Hence with
//   R = RU((1 + 2^-8) d + 2^-29 C + 2^-14 M2) + 2^-9 max|u_i, e_i|
// (the first term per item, f32_sep_rbase), nn >= |n| (rounded up) and
// rhs = RU(R nn), min(n . u, n . e) > rhs proves a reference miss.  NaN
// anywhere keeps the pair (the compare is false).  Checked by
// tools/filter_check.cpp on the adversarial pairs (no reference hit is
// rejected; a mutated, margin-free R does reject hits).
TSK_HD float f32_sep_rbase(double d, double cmax, double M2) {
    const double r = (1.0 + 0x1p-8) * d + 0x1p-29 * cmax + 0x1p-14 * M2 + 0x1p-100;
    return TSK_F2F_RU(r * (1.0 + 0x1p-40));
}

// FP32 view of a query's end: RN32(q.te - T0), RN32(q.e - O).
TSK_HD void f32_query_end(double te, double ex, double ey, double ez, const F32Item &it, float out[4]) {
    out[0] = TSK_F2F_RN(te - it.t0);
    out[1] = TSK_F2F_RN(ex - it.ox);
    out[2] = TSK_F2F_RN(ey - it.oy);
    out[3] = TSK_F2F_RN(ez - it.oz);
}

#ifndef __CUDA_ARCH__
inline float tsk_sqrt_ru(float x) {
    float r = std::sqrt(x);
    if ((double)r * (double)r < (double)x) r = nextafterf(r, INFINITY);
    return r;
}
#endif

// true = the pair provably cannot hit (false for NaN: the pair is kept).
TSK_HD bool f32_sep_far(float px, float py, float pz, float vx, float vy, float vz, float qts, float qx,
                        float qy, float qz, float qte, float qex, float qey, float qez, float rbase,
                        float mcoef = 0x1p-9f) {
#ifdef __CUDA_ARCH__
    const float ux = __fsub_rn(__fmaf_rn(qts, vx, px), qx);
    const float uy = __fsub_rn(__fmaf_rn(qts, vy, py), qy);
    const float uz = __fsub_rn(__fmaf_rn(qts, vz, pz), qz);
    const float ex = __fsub_rn(__fmaf_rn(qte, vx, px), qex);
    const float ey = __fsub_rn(__fmaf_rn(qte, vy, py), qey);
    const float ez = __fsub_rn(__fmaf_rn(qte, vz, pz), qez);
    const float wx = ex - ux, wy = ey - uy, wz = ez - uz;
    const float ww = __fmaf_rn(wz, wz, __fmaf_rn(wy, wy, wx * wx));
    const float uw = __fmaf_rn(uz, wz, __fmaf_rn(uy, wy, ux * wx));
    // any lambda is valid; the closest point's makes the test tight
    const float lam = ww > 0.f ? fminf(fmaxf(__fdividef(-uw, ww), 0.f), 1.f) : 0.f;
    const float nx = __fmaf_rn(lam, wx, ux), ny = __fmaf_rn(lam, wy, uy), nz = __fmaf_rn(lam, wz, uz);
    const float a1 = __fmaf_rn(nz, uz, __fmaf_rn(ny, uy, nx * ux));
    const float a2 = __fmaf_rn(nz, ez, __fmaf_rn(ny, ey, nx * ex));
    const float nn = __fsqrt_ru(__fmaf_ru(nz, nz, __fmaf_ru(ny, ny, __fmul_ru(nx, nx))));
    const float m = fmaxf(fmaxf(fmaxf(fabsf(ux), fabsf(uy)), fmaxf(fabsf(uz), fabsf(ex))),
                          fmaxf(fabsf(ey), fabsf(ez)));
    const float rhs = __fmul_ru(__fmaf_ru(m, mcoef, rbase), nn);
    const float lo = f32_min_nan(a1, a2);
    unsigned far;
    asm("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(far) : "f"(lo), "f"(rhs));
    return far != 0u;
#else
    const float ux = fmaf(qts, vx, px) - qx, uy = fmaf(qts, vy, py) - qy, uz = fmaf(qts, vz, pz) - qz;
    const float ex = fmaf(qte, vx, px) - qex, ey = fmaf(qte, vy, py) - qey, ez = fmaf(qte, vz, pz) - qez;
    const float wx = ex - ux, wy = ey - uy, wz = ez - uz;
    const float ww = fmaf(wz, wz, fmaf(wy, wy, wx * wx));
    const float uw = fmaf(uz, wz, fmaf(uy, wy, ux * wx));
    const float lam = ww > 0.f ? std::fmin(std::fmax(-uw / ww, 0.f), 1.f) : 0.f;
    const float nx = fmaf(lam, wx, ux), ny = fmaf(lam, wy, uy), nz = fmaf(lam, wz, uz);
    const float a1 = fmaf(nz, uz, fmaf(ny, uy, nx * ux));
    const float a2 = fmaf(nz, ez, fmaf(ny, ey, nx * ex));
    const float nn = tsk_sqrt_ru(tsk_fma_dir(nz, nz, tsk_fma_dir(ny, ny, tsk_fma_dir(nx, nx, 0.f, FE_UPWARD),
                                                               FE_UPWARD), FE_UPWARD));
    const float m = std::fmax(std::fmax(std::fmax(std::fabs(ux), std::fabs(uy)), std::fmax(std::fabs(uz), std::fabs(ex))),
                              std::fmax(std::fabs(ey), std::fabs(ez)));
    const float rhs = tsk_fma_dir(tsk_fma_dir(m, mcoef, rbase, FE_UPWARD), nn, 0.f, FE_UPWARD);
    const float lo = (a1 != a1 || a2 != a2) ? NAN : std::fmin(a1, a2);
    return lo > rhs;
#endif
}

// The pre-filter test: true = the pair may hit (NaN flags).
TSK_HD bool f32_flag(const CandF32 &c, float qts, float qx, float qy, float qz, float qa, float qb) {
#ifdef __CUDA_ARCH__
    const float ux = __fsub_rn(__fmaf_rn(qts, c.vx, c.px), qx);
    const float uy = __fsub_rn(__fmaf_rn(qts, c.vy, c.py), qy);
    const float uz = __fsub_rn(__fmaf_rn(qts, c.vz, c.pz), qz);
    const float n = __fmaf_rd(uz, uz, __fmaf_rd(uy, uy, __fmul_rd(ux, ux)));
    const float R = __fmaf_ru(qa, c.sr, qb);
    const float R2 = __fmul_ru(R, R);
    unsigned far;
    asm("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(far) : "f"(n), "f"(R2));
    return far == 0u;
#else
    const float ux = fmaf(qts, c.vx, c.px) - qx;
    const float uy = fmaf(qts, c.vy, c.py) - qy;
    const float uz = fmaf(qts, c.vz, c.pz) - qz;
    const float n = tsk_fma_dir(uz, uz, tsk_fma_dir(uy, uy, tsk_fma_dir(ux, ux, 0.f, FE_DOWNWARD), FE_DOWNWARD),
                                FE_DOWNWARD);
    const float R = tsk_fma_dir(qa, c.sr, qb, FE_UPWARD);
    const float R2 = tsk_fma_dir(R, R, 0.f, FE_UPWARD);
    return !(n > R2);
#endif
}

}  // namespace tsk
