// filter_check.cpp — CPU check of K1's conservative filter (csrc/filter.cuh).
//
// TEST INFRASTRUCTURE (run by tests/test_filter_bound.py).  For adversarial
// (candidate, query) pairs it evaluates the reference's discriminant with the
// vectorised pair arithmetic of core.py:490-537 (one IEEE op per numpy op,
// built with -ffp-contract=off) and checks that every pair whose reference
// discriminant is >= 0 is flagged by pair_filter<TA, TB> in every clip case
// K1 could route it through.  Prints one JSON line of counts; exit 1 on a
// miss.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_1405_7461_b200/csrc/filter.cuh"

using namespace tsk;

struct Seg {
    double ts, te, s[3], e[3];
};

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t next_u64() {
    uint64_t z = (rng_state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static double unif() { return (double)(next_u64() >> 11) * 0x1p-53; }
static double unif(double a, double b) { return a + (b - a) * unif(); }

// clipped() of core.py:503-514 for one segment at time t
static void clipped(const Seg &g, double t, double p[3]) {
    const double ext = g.te - g.ts;
    const double denom = ext == 0.0 ? 1.0 : ext;
    const double f = (t - g.ts) / denom;
    for (int i = 0; i < 3; ++i) {
        double v = g.s[i] + f * (g.e[i] - g.s[i]);
        if (ext == 0.0 || t == g.ts) v = g.s[i];
        else if (t == g.te) v = g.e[i];
        p[i] = v;
    }
}

// reference discriminant (core.py:523-537); returns false when no overlap
static bool ref_disc(const Seg &r, const Seg &c, double d, double &disc, double &cc_out) {
    const double ta = r.ts > c.ts ? r.ts : c.ts;
    const double tb = r.te < c.te ? r.te : c.te;
    if (!(ta <= tb)) return false;
    double ra[3], rb[3], ca[3], cb[3];
    clipped(r, ta, ra);
    clipped(r, tb, rb);
    clipped(c, ta, ca);
    clipped(c, tb, cb);
    const double ux = ra[0] - ca[0], uy = ra[1] - ca[1], uz = ra[2] - ca[2];
    const double cc = ux * ux + uy * uy + uz * uz;
    const double d2 = d * d;
    const double wx = (rb[0] - ra[0]) - (cb[0] - ca[0]);
    const double wy = (rb[1] - ra[1]) - (cb[1] - ca[1]);
    const double wz = (rb[2] - ra[2]) - (cb[2] - ca[2]);
    const double aa = wx * wx + wy * wy + wz * wz;
    const double bb = 2.0 * (ux * wx + uy * wy + uz * wz);
    disc = bb * bb - 4.0 * aa * (cc - d2);
    cc_out = cc;
    return true;
}

// hoisting of db.cu (k_hoist / k_qprep) and its exponent window
static bool mag_ok(double v) {
    const double a = std::fabs(v);
    return a == 0.0 || (a >= 0x1p-900 && a <= 0x1p1000);
}
static bool vel_ok(double v) {
    const double a = std::fabs(v);
    return a == 0.0 || (a >= 0x1p-1000 && a <= 0x1p1000);
}
static bool hoist(const Seg &g, double &ext, double v[3], double dd[3]) {
    ext = g.te - g.ts;
    const double rcp = ext > 0.0 ? 1.0 / ext : 0.0;
    bool ok = mag_ok(g.ts) && mag_ok(g.te) && mag_ok(ext);
    for (int i = 0; i < 3; ++i) {
        dd[i] = g.e[i] - g.s[i];
        v[i] = seg_velocity(dd[i], rcp);
        ok = ok && std::fabs(g.s[i]) <= 0x1p1000 && std::fabs(g.e[i]) <= 0x1p1000 && vel_ok(v[i]);
    }
    return ok;
}

struct Counts {
    long pairs = 0, overlapping = 0, disc_pos = 0, checks = 0, flagged = 0, misses = 0, skipped = 0;
    long hits = 0, f32_checks = 0, f32_flagged = 0, f32_misses = 0, f32_skipped = 0, box_checks = 0;
    long box_misses = 0, box_mut_misses = 0, sep_checks = 0, sep_rejected = 0, sep_misses = 0, sep_mut_misses = 0,
         sep_only = 0, rebase_checks = 0, rebase_misses = 0;
};

// the reference's hit decision for an overlapping pair (core.py:523-551)
static bool ref_hit(const Seg &r, const Seg &c, double d) {
    const double ta = r.ts > c.ts ? r.ts : c.ts;
    const double tb = r.te < c.te ? r.te : c.te;
    if (!(ta <= tb)) return false;
    double ra[3], rb[3], ca[3], cb[3];
    clipped(r, ta, ra);
    clipped(r, tb, rb);
    clipped(c, ta, ca);
    clipped(c, tb, cb);
    const double ux = ra[0] - ca[0], uy = ra[1] - ca[1], uz = ra[2] - ca[2];
    const double cc = ux * ux + uy * uy + uz * uz;
    const double d2 = d * d;
    const double wx = (rb[0] - ra[0]) - (cb[0] - ca[0]);
    const double wy = (rb[1] - ra[1]) - (cb[1] - ca[1]);
    const double wz = (rb[2] - ra[2]) - (cb[2] - ca[2]);
    const double aa = wx * wx + wy * wy + wz * wz;
    const double bb = 2.0 * (ux * wx + uy * wy + uz * wz);
    if (aa == 0.0) return cc <= d2;
    const double disc = bb * bb - 4.0 * aa * (cc - d2);
    if (!(disc >= 0.0)) return false;
    const double sd = std::sqrt(disc);
    const double qq = bb >= 0.0 ? -0.5 * (bb + sd) : -0.5 * (bb - sd);
    const double r1 = qq / aa;
    const double r2 = qq == 0.0 ? r1 : (cc - d2) / qq;
    const bool nan_root = std::isnan(r1) || std::isnan(r2);  // np.minimum/maximum propagate NaN
    const double lo = nan_root ? NAN : (r1 < r2 ? r1 : r2), hi = nan_root ? NAN : (r1 > r2 ? r1 : r2);
    return lo <= 1.0 && hi >= 0.0;
}

// K1's FP32 pre-filter for candidate r and query c, with the item origin at
// (O, T0) and the item bounds taken from this pair alone (the tightest
// bounds any item containing the pair can have).
static void check_f32(const Seg &r, const Seg &c, double d, const double O[3], double T0, double cmax,
                      Counts &n, const char *tag) {
    double rext, rv[3], rd[3], cext, cv[3], cd[3];
    const bool ok = hoist(r, rext, rv, rd) & hoist(c, cext, cv, cd);
    if (!ok || !filter_ok(cmax, d * d) || !(d * d <= 0x1p120) || !(cmax <= 0x1p60)) {
        ++n.f32_skipped;
        return;
    }
    double ar = 0, aq = 0, vr = 0;
    for (int i = 0; i < 3; ++i) {
        ar = std::fmax(ar, std::fabs(r.s[i] - O[i]));
        aq = std::fmax(aq, std::fabs(c.s[i] - O[i]));
        vr = std::fmax(vr, std::fabs(rv[i]));
    }
    const double tvr = std::fabs(r.ts - T0) * vr, tq = std::fabs(c.ts - T0);
    const F32Item it = f32_item(O[0], O[1], O[2], T0, ar, tvr, vr, aq, tq, cext, cmax);
    if (!it.ok) {
        ++n.f32_skipped;
        return;
    }
    float q[6];
    f32_query(c.ts, c.s[0], c.s[1], c.s[2], cext, cd[0], cd[1], cd[2], it, std::sqrt(d * d), q);
    const CandF32 cf = f32_cand(r.ts, r.s[0], r.s[1], r.s[2], rv[0], rv[1], rv[2], it);
    const bool f = f32_flag(cf, q[0], q[1], q[2], q[3], q[4], q[5]);
    // K1's lane form (f32_scan2): one threshold from the largest speed bound
    // of the lane's four candidates, the query passes when the NaN-propagating
    // min of the four norms is not far, then each candidate's own compare
    // against that threshold.  Companions: random speeds and norms (some NaN).
    float srl = cf.sr, nmin = f32_n2(cf, q[0], q[1], q[2], q[3]);
    const float nown = nmin;
    for (int k = 0; k < 3; ++k) {
        srl = std::fmax(srl, (float)unif(0.0, 2.0 * cf.sr + 1.0));
        const float nk = next_u64() % 8 == 0 ? NAN : (float)unif(0.0, 1e6);
        nmin = f32_min_nan(nmin, nk);
    }
    const float R2 = f32_r2(q[4], srl, q[5]);
    const bool lane_flag = !f32_far(nmin, R2) && !f32_far(nown, R2);
    if (f && !lane_flag) {
        ++n.f32_misses;
        if (n.f32_misses <= 5) std::fprintf(stderr, "F32 LANE MISS %s\n", tag);
    }
    const bool need = ref_hit(r, c, d);
    // the K1 layout's re-based records: the candidate's FP32 view relative to
    // a group origin (O_g, T_g) (another candidate's start), re-based to the
    // item origin (f32_cand_rebase); the item bounds then cover O_g and T_g
    {
        double Og[3];
        for (int i = 0; i < 3; ++i) Og[i] = r.s[i] + unif(-1, 1) * (std::fabs(r.e[i] - r.s[i]) + std::fabs(r.s[i]) * 1e-3 + 1.0);
        const double Tg = r.ts + unif(-3, 3) * (std::fabs(r.te - r.ts) + 1.0);
        double ar2 = ar, tr2 = std::fmax(std::fabs(r.ts - T0), std::fabs(Tg - T0));
        for (int i = 0; i < 3; ++i) ar2 = std::fmax(ar2, std::fabs(Og[i] - O[i]));
        const double tvr2 = std::fmax(tvr, std::fabs(Tg - T0) * vr);  // the group's own start at T_g
        const F32Item it2 = f32_item(O[0], O[1], O[2], T0, ar2, tvr2, vr, aq, tq, cext, cmax, tr2);
        if (it2.ok) {
            F32Item go;
            go.ox = Og[0]; go.oy = Og[1]; go.oz = Og[2]; go.t0 = Tg;
            const CandF32 pg = f32_cand(r.ts, r.s[0], r.s[1], r.s[2], rv[0], rv[1], rv[2], go);
            const CandF32 rb = f32_cand_rebase(pg.px, pg.py, pg.pz, pg.vx, pg.vy, pg.vz, pg.sr,
                                               TSK_F2F_RN(Og[0] - O[0]), TSK_F2F_RN(Og[1] - O[1]),
                                               TSK_F2F_RN(Og[2] - O[2]), TSK_F2F_RN(Tg - T0));
            float q2[6];
            f32_query(c.ts, c.s[0], c.s[1], c.s[2], cext, cd[0], cd[1], cd[2], it2, std::sqrt(d * d), q2);
            const bool f2 = f32_flag(rb, q2[0], q2[1], q2[2], q2[3], q2[4], q2[5]);
            double dq = 0;
            for (int i = 0; i < 3; ++i) dq = std::fmax(dq, std::fabs(c.e[i] - c.s[i]));
            const double M2 = ar2 + tvr2 + (tq + cext + tr2) * vr + aq + dq;
            float qe[4];
            f32_query_end(c.te, c.e[0], c.e[1], c.e[2], it2, qe);
            const bool far2 = f32_sep_far(rb.px, rb.py, rb.pz, rb.vx, rb.vy, rb.vz, q2[0], q2[1], q2[2], q2[3], qe[0],
                                          qe[1], qe[2], qe[3], f32_sep_rbase(std::sqrt(d * d), cmax, M2));
            ++n.rebase_checks;
            if (need && (!f2 || far2)) {
                ++n.rebase_misses;
                if (n.rebase_misses <= 5) std::fprintf(stderr, "REBASE MISS %s d=%.17g flag=%d far=%d\n", tag, d, f2, far2);
            }
        }
    }
    // the separating-axis second stage over the query's span (f32_sep_far)
    {
        double dq = 0;
        for (int i = 0; i < 3; ++i) dq = std::fmax(dq, std::fabs(c.e[i] - c.s[i]));
        const double M2 = ar + tvr + (tq + cext) * vr + aq + dq;
        float qe[4];
        f32_query_end(c.te, c.e[0], c.e[1], c.e[2], it, qe);
        const float rb = f32_sep_rbase(std::sqrt(d * d), cmax, M2);
        const bool far = f32_sep_far(cf.px, cf.py, cf.pz, cf.vx, cf.vy, cf.vz, q[0], q[1], q[2], q[3], qe[0], qe[1],
                                     qe[2], qe[3], rb);
        ++n.sep_checks;
        n.sep_rejected += far;
        if (need && far) {
            ++n.sep_misses;
            if (n.sep_misses <= 5)
                std::fprintf(stderr, "SEP MISS %s d=%.17g r=[%.17g %.17g (%.17g %.17g %.17g)->(%.17g %.17g %.17g)] "
                             "c=[%.17g %.17g (%.17g %.17g %.17g)->(%.17g %.17g %.17g)]\n",
                             tag, d, r.ts, r.te, r.s[0], r.s[1], r.s[2], r.e[0], r.e[1], r.e[2], c.ts, c.te,
                             c.s[0], c.s[1], c.s[2], c.e[0], c.e[1], c.e[2]);
        }
        // mutation: margin-free radius (d itself, no m term) must reject hits
        const float rb0 = TSK_F2F_RN(std::sqrt(d * d));
        if (need && f32_sep_far(cf.px, cf.py, cf.pz, cf.vx, cf.vy, cf.vz, q[0], q[1], q[2], q[3], qe[0], qe[1],
                                qe[2], qe[3], rb0, 0.f))
            ++n.sep_mut_misses;
        // every pair the second stage keeps is flagged by the first
        if (!far && !f) ++n.sep_only;
    }
    // the box cull (K1 layout): segment boxes rounded outward to FP32
    {
        float bl[2][3], bh[2][3];
        const Seg *sg[2] = {&r, &c};
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < 3; ++i) {
                bl[k][i] = tsk_f2f_rd(std::fmin(sg[k]->s[i], sg[k]->e[i]));
                bh[k][i] = tsk_f2f_ru(std::fmax(sg[k]->s[i], sg[k]->e[i]));
            }
        const float g2 = box_gap2(bl[0][0], bl[0][1], bl[0][2], bh[0][0], bh[0][1], bh[0][2], bl[1][0], bl[1][1],
                                  bl[1][2], bh[1][0], bh[1][1], bh[1][2]);
        const float rb = box_cull_rbase(std::sqrt(d * d), cmax);
        const float dr = box_cull_dterm(bl[0][0], bl[0][1], bl[0][2], bh[0][0], bh[0][1], bh[0][2]);
        const float dq = box_cull_dterm(bl[1][0], bl[1][1], bl[1][2], bh[1][0], bh[1][1], bh[1][2]);
        const bool pass = !(g2 > box_cull_r2(rb, dr, dq));
        ++n.box_checks;
        if (need && !pass) {
            ++n.box_misses;
            if (n.box_misses <= 5) std::fprintf(stderr, "BOX MISS %s d=%.17g\n", tag, d);
        }
        // mutation: without the diagonal term the cull must miss (mode 8)
        if (need && g2 > box_cull_r2(rb, 0.f, 0.f)) ++n.box_mut_misses;
    }
    ++n.f32_checks;
    n.hits += need;
    n.f32_flagged += f;
    if (need && !f) {
        ++n.f32_misses;
        if (n.f32_misses <= 5)
            std::fprintf(stderr,
                         "F32 MISS %s d=%.17g r=[%.17g %.17g (%.17g %.17g %.17g)->(%.17g %.17g %.17g)] "
                         "c=[%.17g %.17g (%.17g %.17g %.17g)->(%.17g %.17g %.17g)] O=(%g %g %g) T0=%.17g\n",
                         tag, d, r.ts, r.te, r.s[0], r.s[1], r.s[2], r.e[0], r.e[1], r.e[2], c.ts, c.te,
                         c.s[0], c.s[1], c.s[2], c.e[0], c.e[1], c.e[2], O[0], O[1], O[2], T0);
    }
}

template <int TA, int TB>
static void check_case(const CandF &cf, const QF &qf, double wmin, double wmax, const FilterK &K,
                       bool need, Counts &n, const Seg &r, const Seg &c, double d, const char *tag) {
    const bool f = pair_filter<TA, TB>(cf, qf, wmin, wmax, K);
    ++n.checks;
    n.flagged += f;
    if (need && !f) {
        ++n.misses;
        if (n.misses <= 5)
            std::fprintf(stderr,
                         "MISS %s TA=%d TB=%d d=%.17g r=[%.17g %.17g (%.17g %.17g %.17g)->(%.17g %.17g %.17g)] "
                         "c=[%.17g %.17g (%.17g %.17g %.17g)->(%.17g %.17g %.17g)]\n",
                         tag, TA, TB, d, r.ts, r.te, r.s[0], r.s[1], r.s[2], r.e[0], r.e[1], r.e[2], c.ts, c.te,
                         c.s[0], c.s[1], c.s[2], c.e[0], c.e[1], c.e[2]);
    }
}

static void check_pair(const Seg &r, const Seg &c, double d, Counts &n, const char *tag) {
    ++n.pairs;
    double disc, cc;
    if (!ref_disc(r, c, d, disc, cc)) return;
    ++n.overlapping;
    CandF cf;
    QF qf;
    double rv[3], rd[3], qv[3], qd[3];
    const bool ok = hoist(r, cf.ext, rv, rd) & hoist(c, qf.ext, qv, qd);
    double cmax = 0.0;
    for (int i = 0; i < 3; ++i)
        cmax = std::fmax(cmax, std::fmax(std::fmax(std::fabs(r.s[i]), std::fabs(r.e[i])),
                                         std::fmax(std::fabs(c.s[i]), std::fabs(c.e[i]))));
    if (!ok || !filter_ok(cmax, d * d)) {
        ++n.skipped;  // K1 evaluates these exactly (unsafe tile / launch)
        return;
    }
    const bool need = disc >= 0.0;
    n.disc_pos += need;
    {
        // FP32 pre-filter, origin at the query's start and at a shifted point
        const double O0[3] = {c.s[0], c.s[1], c.s[2]};
        check_f32(r, c, d, O0, c.ts, cmax, n, tag);
        double O1[3];
        for (int i = 0; i < 3; ++i) O1[i] = c.s[i] + unif(-1, 1) * (std::fabs(c.s[i]) + 1.0);
        check_f32(r, c, d, O1, c.ts - unif(0, 5) * (std::fabs(c.te - c.ts) + 1.0), cmax, n, tag);
    }
    cf.ts = r.ts; cf.te = r.te;
    cf.sx = r.s[0]; cf.sy = r.s[1]; cf.sz = r.s[2];
    cf.vx = rv[0]; cf.vy = rv[1]; cf.vz = rv[2];
    qf.ts = c.ts; qf.te = c.te;
    qf.sx = c.s[0]; qf.sy = c.s[1]; qf.sz = c.s[2];
    qf.vx = qv[0]; qf.vy = qv[1]; qf.vz = qv[2];
    qf.dx = qd[0]; qf.dy = qd[1]; qf.dz = qd[2];
    const FilterK K = filter_consts(cmax, d * d);
    const double inf = INFINITY;
    // every route K1 can take for this pair
    const bool ta_r = c.ts > r.ts, ta_c = c.ts < r.ts;
    const bool tb_r = c.te < r.te, tb_c = c.te > r.te;
    // generic per-pair tb, and the dynamic split around this candidate's te
    check_case<TA_BOTH, TB_DYN>(cf, qf, -inf, inf, K, need, n, r, c, d, tag);
    check_case<TA_BOTH, TB_DYN>(cf, qf, r.te, r.te, K, need, n, r, c, d, tag);
    if (ta_r) {
        check_case<TA_R, TB_DYN>(cf, qf, -inf, inf, K, need, n, r, c, d, tag);
        check_case<TA_R, TB_DYN>(cf, qf, r.te, r.te, K, need, n, r, c, d, tag);
        if (tb_c) check_case<TA_R, TB_C>(cf, qf, r.te, r.te, K, need, n, r, c, d, tag);
    }
    if (ta_c) {
        check_case<TA_C, TB_DYN>(cf, qf, -inf, inf, K, need, n, r, c, d, tag);
        check_case<TA_C, TB_DYN>(cf, qf, r.te, r.te, K, need, n, r, c, d, tag);
        if (tb_r) check_case<TA_C, TB_R>(cf, qf, r.te, r.te, K, need, n, r, c, d, tag);
    }
    (void)tb_r;
}

// closest approach of the two (linear) motions over the shared span, in
// long double: the threshold at which the pair flips between hit and miss
static double min_dist(const Seg &r, const Seg &c, bool clamp = false) {
    const long double ta = r.ts > c.ts ? r.ts : c.ts, tb = r.te < c.te ? r.te : c.te;
    auto pos = [](const Seg &g, long double t, long double p[3]) {
        const long double ext = (long double)g.te - g.ts;
        const long double f = ext == 0 ? 0 : (t - g.ts) / ext;
        for (int i = 0; i < 3; ++i) p[i] = g.s[i] + f * ((long double)g.e[i] - g.s[i]);
    };
    long double ra[3], rb[3], ca[3], cb[3];
    pos(r, ta, ra); pos(r, tb, rb); pos(c, ta, ca); pos(c, tb, cb);
    long double u[3], w[3], uu = 0, ww = 0, uw = 0;
    for (int i = 0; i < 3; ++i) {
        u[i] = ra[i] - ca[i];
        w[i] = (rb[i] - ra[i]) - (cb[i] - ca[i]);
        uu += u[i] * u[i]; ww += w[i] * w[i]; uw += u[i] * w[i];
    }
    long double lam = ww > 0 ? -uw / ww : 0;
    // the line distance (the discriminant's root), or with clamp = true the
    // segment distance (lambda clamped to [0, 1]: where hits flip)
    if (clamp) lam = lam < 0 ? 0 : (lam > 1 ? 1 : lam);
    long double m2 = uu + 2 * lam * uw + lam * lam * ww;
    return (double)std::sqrt(m2 > 0 ? m2 : 0);
}

static Seg rand_seg(double L, double t0, double t1, double speed) {
    Seg g;
    g.ts = t0; g.te = t1;
    for (int i = 0; i < 3; ++i) {
        g.s[i] = unif(-L, L);
        g.e[i] = g.s[i] + speed * unif(-1, 1);
    }
    return g;
}

int main(int argc, char **argv) {
    long iters = argc > 1 ? std::atol(argv[1]) : 200000;
    Counts n, nrand;
    const double scales[] = {1e-3, 1.0, 100.0, 1e4, 1e6};
    const double tbase[] = {0.0, 1e3, 1.7e9};
    for (long it = 0; it < iters; ++it) {
        const double L = scales[next_u64() % 5];
        const double T = tbase[next_u64() % 3];
        const double sp = L * (next_u64() % 2 ? 1.0 : 1e-3);
        // overlapping spans with random alignment
        const double a0 = T + unif(0, 10), a1 = a0 + unif(0.01, 10);
        double b0 = T + unif(0, 10), b1 = b0 + unif(0.01, 10);
        const int mode = (int)(next_u64() % 10);
        if (mode == 1) b0 = a0;                         // equal starts (TA_BOTH)
        if (mode == 2) b1 = a1;                         // equal ends
        if (mode == 3) { b0 = a1; b1 = a1 + 1.0; }      // touching: zero-length span
        if (mode == 4) b1 = b0;                         // zero-ext query (waypoint)
        Seg r = rand_seg(L, a0, a1, sp), c = rand_seg(L, b0, b1, sp);
        if (mode == 5) {  // near-parallel motion
            const double eps = std::ldexp(1.0, -(int)(next_u64() % 50));
            for (int i = 0; i < 3; ++i) {
                c.s[i] = r.s[i] + unif(-1, 1) * L * 1e-3;
                c.e[i] = c.s[i] + (r.e[i] - r.s[i]) * (1 + eps * unif(-1, 1));
            }
            c.ts = r.ts; c.te = r.te;
        }
        if (mode == 6) {  // identical motion offset by a constant
            for (int i = 0; i < 3; ++i) {
                const double off = unif(-1, 1) * L;
                c.s[i] = r.s[i] + off;
                c.e[i] = r.e[i] + off;
            }
            c.ts = r.ts; c.te = r.te;
        }
        if (mode == 7) {
            // head-on: the query sits inside the candidate's span and the
            // candidate moves straight at the query's start point, so the
            // FP32 pre-filter's triangle bound is tight at the flip point
            r.ts = a0; r.te = a0 + 10.0;
            c.ts = a0 + unif(0.5, 4.0); c.te = c.ts + unif(0.01, 4.0);
            double dir[3], nrm = 0;
            for (int i = 0; i < 3; ++i) { dir[i] = unif(-1, 1); nrm += dir[i] * dir[i]; }
            nrm = std::sqrt(nrm);
            const double dist0 = L * unif(0.5, 1.0), speed = dist0 / unif(12.0, 40.0);
            for (int i = 0; i < 3; ++i) {
                c.s[i] = unif(-L, L);
                c.e[i] = next_u64() % 2 ? c.s[i] : c.s[i] + dir[i] / nrm * speed * (c.te - c.ts) * unif(-1, 1);
                r.s[i] = c.s[i] + dir[i] / nrm * dist0;
                r.e[i] = r.s[i] - dir[i] / nrm * speed * (r.te - r.ts);
            }
        }
        if (mode == 8) {
            // absorbed offset: long motion along one axis crossing the
            // query, a perpendicular offset h below the rounding of |U|^2
            // (h ~ 2^-26 |U| and less), so the reference's cc = |U|^2
            // loses it and reports a hit at a separation far above a tiny d
            const int ax = (int)(next_u64() % 3), px = (ax + 1 + (int)(next_u64() % 2)) % 3;
            const double h = L * std::ldexp(unif(0.5, 1.0), -(int)(18 + next_u64() % 20));
            c.ts = r.ts; c.te = r.te;
            for (int i = 0; i < 3; ++i) {
                c.s[i] = c.e[i] = unif(-L, L) * (next_u64() % 2);
                r.s[i] = r.e[i] = c.s[i];
            }
            r.s[ax] = c.s[ax] + L * unif(0.5, 1.0);
            r.e[ax] = c.s[ax] - L * unif(0.5, 1.0);
            r.s[px] += h; r.e[px] += h;
            if (next_u64() % 2) {  // the query moves too (same offset kept)
                const double m = L * unif(-1, 1);
                c.e[ax] += m; r.e[ax] += m;
            }
        }
        if (mode != 7 && mode != 8 && next_u64() % 3 == 0) { r.s[2] = r.e[2] = 0.0; c.s[2] = c.e[2] = 0.0; }  // planar data
        nrand.pairs++;
        check_pair(r, c, L * 0.01, nrand, "rand");
        if (mode == 8)  // thresholds far below the offset
            for (int k = 0; k < 4; ++k) check_pair(r, c, L * std::ldexp(1.0, -(int)(30 + next_u64() % 40)), n, "absorbed");
        // thresholds straddling the pair's own flip point
        const double md = min_dist(r, c);
        if (md > 0 && std::isfinite(md)) {
            for (int k = 0; k < 6; ++k) {
                const double rel = std::ldexp(1.0, -(int)(next_u64() % 52)) * (next_u64() % 2 ? 1 : -1);
                check_pair(r, c, md * (1 + rel), n, "edge");
            }
            check_pair(r, c, md, n, "edge0");
            check_pair(r, c, std::nextafter(md, 0.0), n, "edge-");
            check_pair(r, c, std::nextafter(md, INFINITY), n, "edge+");
        } else {
            check_pair(r, c, 0.0, n, "zero");
        }
        // thresholds straddling the segment distance (hit/miss flip point)
        const double ms = min_dist(r, c, true);
        if (ms > 0 && std::isfinite(ms)) {
            for (int k = 0; k < 4; ++k) {
                const double rel = std::ldexp(1.0, -(int)(next_u64() % 52)) * (next_u64() % 2 ? 1 : -1);
                check_pair(r, c, ms * (1 + rel), n, "seg");
            }
            check_pair(r, c, ms, n, "seg0");
            check_pair(r, c, std::nextafter(ms, INFINITY), n, "seg+");
        }
    }
    std::printf("{\"edge\": {\"pairs\": %ld, \"overlapping\": %ld, \"disc_pos\": %ld, \"checks\": %ld, "
                "\"flagged\": %ld, \"skipped\": %ld, \"misses\": %ld, \"hits\": %ld, \"f32_checks\": %ld, "
                "\"f32_flagged\": %ld, \"f32_skipped\": %ld, \"f32_misses\": %ld, \"box_checks\": %ld, "
                "\"box_misses\": %ld, \"box_mutation_misses\": %ld, \"sep_checks\": %ld, \"sep_rejected\": %ld, "
                "\"sep_misses\": %ld, \"sep_mutation_misses\": %ld, \"rebase_checks\": %ld, \"rebase_misses\": %ld}, "
                "\"random\": {\"pairs\": %ld, \"overlapping\": %ld, \"disc_pos\": %ld, \"checks\": %ld, "
                "\"flagged\": %ld, \"misses\": %ld, \"hits\": %ld, \"f32_checks\": %ld, \"f32_flagged\": %ld, "
                "\"f32_misses\": %ld}}\n",
                n.pairs, n.overlapping, n.disc_pos, n.checks, n.flagged, n.skipped, n.misses, n.hits,
                n.f32_checks, n.f32_flagged, n.f32_skipped, n.f32_misses, n.box_checks, n.box_misses + nrand.box_misses,
                n.box_mut_misses + nrand.box_mut_misses, n.sep_checks + nrand.sep_checks, n.sep_rejected + nrand.sep_rejected,
                n.sep_misses + nrand.sep_misses, n.sep_mut_misses + nrand.sep_mut_misses,
                n.rebase_checks + nrand.rebase_checks, n.rebase_misses + nrand.rebase_misses, nrand.pairs, nrand.overlapping,
                nrand.disc_pos, nrand.checks, nrand.flagged, nrand.misses, nrand.hits, nrand.f32_checks,
                nrand.f32_flagged, nrand.f32_misses);
    return (n.misses || nrand.misses || n.f32_misses || nrand.f32_misses || n.box_misses || nrand.box_misses ||
            n.sep_misses || nrand.sep_misses || n.rebase_misses || nrand.rebase_misses) ? 1 : 0;
}
