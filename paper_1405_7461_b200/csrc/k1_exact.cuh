// k1_exact.cuh — K1's exact rare path, shared by both pair kernels.
//
// Pairs flagged by a kernel's filter are queued per warp and evaluated here
// 32 at a time, one per lane: the reference's operation sequence for the
// clipped positions and quadratic coefficients (core.py:503-537,
// /root/reference/pkg/src/trajseek/), a second filter, and the exact root
// solve (core.py:536-558).  Candidates are re-read from global memory and
// queries from the kernel's tile (shared or global), so the kernels stage
// nothing for it.
#pragma once

#include "filter.cuh"
#include <math_constants.h>

#include "tsk_internal.cuh"

namespace tsk {

// Shared-memory loads through an explicit 32-bit shared-window address, so
// the loop carries one address register instead of re-deriving the window
// base every iteration.
__device__ __forceinline__ void lds2(uint32_t a, double &x, double &y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

// Exact view of a query record (rare path); RN(1/ext) as the hoist computes it.
struct QVals {
    double ts, te, sx, sy, sz, ext, dx, dy, dz, rcp;
};

__device__ __forceinline__ QVals load_q(const QRec *rec) {
    QVals q;
    q.ts = rec->ts; q.te = rec->te;
    q.sx = rec->sx; q.sy = rec->sy; q.sz = rec->sz; q.ext = rec->ext;
    q.dx = rec->dx; q.dy = rec->dy; q.dz = rec->dz;
    q.rcp = q.ext > 0.0 ? __drcp_rn(q.ext) : 0.0;
    return q;
}

struct Cand {
    double ts, te, ext, rcp, sx, sy, sz, dx, dy, dz, ex, ey, ez;
};

template <bool SLOW>
__device__ __forceinline__ double quot(double a, double b, double y) {
    return SLOW ? __ddiv_rn(a, b) : qdiv(a, b, y);
}

// p = s + ((t - ts) / ext) * (e - s), the non-verbatim branch of core.py:508-513
template <bool SLOW>
__device__ __forceinline__ void lerp(double t, double ts, double ext, double rcp, double sx, double sy,
                                     double sz, double dx, double dy, double dz, double &px,
                                     double &py, double &pz) {
    double f = quot<SLOW>(__dsub_rn(t, ts), ext, rcp);
    px = __dadd_rn(sx, __dmul_rn(f, dx));
    py = __dadd_rn(sy, __dmul_rn(f, dy));
    pz = __dadd_rn(sz, __dmul_rn(f, dz));
}

// position_at with every verbatim rule (core.py:309-331 / 503-521); used on
// the zero-span path only.
__device__ __forceinline__ void position_exact(double t, double ts, double te, double sx, double sy,
                                               double sz, double ex, double ey, double ez,
                                               double dx, double dy, double dz, double &px,
                                               double &py, double &pz) {
    double ext = __dsub_rn(te, ts);
    if (ext == 0.0 || t == ts) {
        px = sx; py = sy; pz = sz;
    } else if (t == te) {
        px = ex; py = ey; pz = ez;
    } else {
        double f = __ddiv_rn(__dsub_rn(t, ts), ext);
        px = __dadd_rn(sx, __dmul_rn(f, dx));
        py = __dadd_rn(sy, __dmul_rn(f, dy));
        pz = __dadd_rn(sz, __dmul_rn(f, dz));
    }
}

struct Hit {
    bool hit;
    double tb, te;
};

// Exact root solve (core.py:536-558) for one pair with span > 0.
__device__ __forceinline__ Hit solve_exact(double ta, double tb, double cc, double aa, double dot,
                                           double e, double d2) {
    Hit h;
    double bb = __dmul_rn(2.0, dot);
    double lo, hi;
    if (aa == 0.0) {  // constant separation
        h.hit = cc <= d2;
        lo = 0.0;
        hi = 1.0;
    } else {
        double disc = __dsub_rn(__dmul_rn(bb, bb), __dmul_rn(__dmul_rn(4.0, aa), e));
        if (!(disc >= 0.0)) {
            h.hit = false;
            h.tb = h.te = 0.0;
            return h;
        }
        double sd = __dsqrt_rn(disc);
        double qq = bb >= 0.0 ? __dmul_rn(-0.5, __dadd_rn(bb, sd)) : __dmul_rn(-0.5, __dsub_rn(bb, sd));
        double r1 = __ddiv_rn(qq, aa);
        double r2 = qq == 0.0 ? r1 : __ddiv_rn(e, qq);
        // np.minimum / np.maximum propagate NaN (core.py:545-546): a NaN root
        // (aa = inf from |w| above ~1e154) makes the hit test below fail
        const bool nan_root = isnan(r1) || isnan(r2);
        lo = nan_root ? CUDART_NAN : (r1 < r2 ? r1 : r2);
        hi = nan_root ? CUDART_NAN : (r1 > r2 ? r1 : r2);
        h.hit = lo <= 1.0 && hi >= 0.0;
    }
    double span = __dsub_rn(tb, ta);
    h.tb = lo <= 0.0 ? ta : __dadd_rn(ta, __dmul_rn(lo, span));
    h.te = hi >= 1.0 ? tb : __dadd_rn(ta, __dmul_rn(hi, span));
    return h;
}

// Flat (zero-length shared span) pairs, quadratic-root candidates and lanes
// at a window edge: exact recomputation with every verbatim rule.
__device__ __forceinline__ Hit rare_pair(const Cand &r, const QRec &Q, double cc, double aa, double dot,
                                         double e, double d2) {
    Hit h;
    h.hit = false;
    h.tb = h.te = 0.0;
    const double ta = r.ts > Q.ts ? r.ts : Q.ts;
    const double tb = r.te < Q.te ? r.te : Q.te;
    if (!(ta <= tb)) return h;  // no temporal overlap
    if (ta == tb) {
        // positions at the shared instant, constant separation (core.py:376-378)
        double rx, ry, rz, qx, qy, qz;
        position_exact(ta, r.ts, r.te, r.sx, r.sy, r.sz, r.ex, r.ey, r.ez, r.dx, r.dy, r.dz, rx, ry, rz);
        position_exact(ta, Q.ts, Q.te, Q.sx, Q.sy, Q.sz, Q.ex, Q.ey, Q.ez, Q.dx, Q.dy, Q.dz, qx, qy, qz);
        const double ux = __dsub_rn(rx, qx), uy = __dsub_rn(ry, qy), uz = __dsub_rn(rz, qz);
        const double c2 = __dadd_rn(__dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy)), __dmul_rn(uz, uz));
        h.hit = c2 <= d2;
        h.tb = ta;
        h.te = tb;
        return h;
    }
    return solve_exact(ta, tb, cc, aa, dot, e, d2);
}

struct ItemCtx {
    int64_t b, lo_q, first_c, c_hi;  // batch, tile's first query ordinal, tile's candidate range
    int64_t c_lo;                    // first valid candidate (first_c may be aligned below it)
    int64_t q0;                      // first query offset within batch b (tile)
    int64_t b1;                      // shared unit: the second batch (queries js..), else -1
    int nt, js;                      // staged queries; queries of batch b (nt when single)
    int jx[K1_GMAX - 2];             // groups: tile offsets of batches b + 2 .. (nt when absent)
};

// Batches in an item's tile (1 .. K1_GMAX).
__device__ __forceinline__ int item_batches(const ItemCtx &it) {
    if (it.b1 < 0) return 1;
    int n = 2;
#pragma unroll
    for (int i = 0; i < K1_GMAX - 2; ++i) n += it.jx[i] < it.nt;
    return n;
}

// Per-item counters are kept per batch in one 64-bit word: the low half
// for batch b, the high half for b1 (a warp's counts in one item are far
// below 2^32).
constexpr unsigned long long CNT_B1 = 1ull << 32;

__device__ __forceinline__ uint64_t make_key(const K1Launch &L, int64_t b, int64_t e_off,
                                             int64_t q_off) {
    uint64_t major = L.query_major ? (uint64_t)q_off : (uint64_t)e_off;
    uint64_t minor = L.query_major ? (uint64_t)e_off : (uint64_t)q_off;
    return ((uint64_t)b << (L.major_bits + L.minor_bits)) | (major << L.minor_bits) | minor;
}

// True when bb^2 = 4 dot^2 and 4 aa e of the reference's discriminant are
// finite (core.py:537); false for NaN.
__device__ __forceinline__ bool no_overflow(double aa, double dot, double e) {
    return fabs(dot) <= 0x1p510 && aa <= 0x1p500 && fabs(e) <= 0x1p500;
}

// The common-path arithmetic of one (candidate, query) pair up to the hit
// test.  Returns whether the pair needs the exact rare path.
template <int TA, int TB, bool SLOW>
__device__ __forceinline__ bool pair_eval(const Cand &r, const QVals &Q, const QRec *qrec, double wmin_te,
                                          double wmax_te, double d2, double &cc, double &aa,
                                          double &dot, double &e) {
    const double cts = Q.ts, cte = Q.te;
    // ── clip at ta (core.py:503-516) ──
    double ta, rax, ray, raz, cax, cay, caz;
    if (TA == TA_R) {
        ta = cts;
        lerp<SLOW>(cts, r.ts, r.ext, r.rcp, r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, rax, ray, raz);
        cax = Q.sx; cay = Q.sy; caz = Q.sz;
    } else if (TA == TA_C) {
        ta = r.ts;
        rax = r.sx; ray = r.sy; raz = r.sz;
        lerp<SLOW>(r.ts, cts, Q.ext, Q.rcp, Q.sx, Q.sy, Q.sz, Q.dx, Q.dy, Q.dz, cax, cay, caz);
    } else {
        ta = r.ts > cts ? r.ts : cts;
        lerp<SLOW>(ta, r.ts, r.ext, r.rcp, r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, rax, ray, raz);
        lerp<SLOW>(ta, cts, Q.ext, Q.rcp, Q.sx, Q.sy, Q.sz, Q.dx, Q.dy, Q.dz, cax, cay, caz);
    }
    // ── clip at tb: interpolate the later ender ──
    double tb, rbx, rby, rbz, cbx, cby, cbz;
    if (TB == TB_R || (TB == TB_DYN && cte < wmin_te)) {  // every candidate ends after the query
        tb = cte;
        lerp<SLOW>(cte, r.ts, r.ext, r.rcp, r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, rbx, rby, rbz);
        cbx = qrec->ex; cby = qrec->ey; cbz = qrec->ez;
    } else if (TB == TB_C || (TB == TB_DYN && cte > wmax_te)) {  // the query ends after every candidate
        tb = r.te;
        rbx = r.ex; rby = r.ey; rbz = r.ez;
        lerp<SLOW>(r.te, cts, Q.ext, Q.rcp, Q.sx, Q.sy, Q.sz, Q.dx, Q.dy, Q.dz, cbx, cby, cbz);
    } else {
        tb = r.te < cte ? r.te : cte;
        double px, py, pz, qx, qy, qz;
        lerp<SLOW>(tb, r.ts, r.ext, r.rcp, r.sx, r.sy, r.sz, r.dx, r.dy, r.dz, px, py, pz);
        lerp<SLOW>(tb, cts, Q.ext, Q.rcp, Q.sx, Q.sy, Q.sz, Q.dx, Q.dy, Q.dz, qx, qy, qz);
        const bool zr = r.te > cte, zc = cte > r.te;
        const double qex = qrec->ex, qey = qrec->ey, qez = qrec->ez;
        rbx = zr ? px : r.ex; rby = zr ? py : r.ey; rbz = zr ? pz : r.ez;
        cbx = zc ? qx : qex; cby = zc ? qy : qey; cbz = zc ? qz : qez;
    }
    // ── quadratic coefficients (core.py:523-537) ──
    const double ux = __dsub_rn(rax, cax), uy = __dsub_rn(ray, cay), uz = __dsub_rn(raz, caz);
    cc = __dadd_rn(__dadd_rn(__dmul_rn(ux, ux), __dmul_rn(uy, uy)), __dmul_rn(uz, uz));
    const double wx = __dsub_rn(__dsub_rn(rbx, rax), __dsub_rn(cbx, cax));
    const double wy = __dsub_rn(__dsub_rn(rby, ray), __dsub_rn(cby, cay));
    const double wz = __dsub_rn(__dsub_rn(rbz, raz), __dsub_rn(cbz, caz));
    aa = __dadd_rn(__dadd_rn(__dmul_rn(wx, wx), __dmul_rn(wy, wy)), __dmul_rn(wz, wz));
    dot = __dadd_rn(__dadd_rn(__dmul_rn(ux, wx), __dmul_rn(uy, wy)), __dmul_rn(uz, wz));
    e = __dsub_rn(cc, d2);
    // disc / 4 (exact scaling); the margin keeps the test a superset under
    // underflow, and pairs whose reference discriminant could overflow
    // (bb^2 or 4 aa e beyond 2^1022: disc = +-inf or NaN) go to the exact solve
    const double dq = __dsub_rn(__dmul_rn(dot, dot), __dmul_rn(aa, e));
    return ta == tb || dq >= -0x1p-1000 || !no_overflow(aa, dot, e);
}

constexpr int K1_WARPS = K1_THREADS / 32;

// Output and key layout for the (non-inlined) flush, kept in shared memory
// so the hot loop does not hold them in registers.
struct FlushCfg {
    // entry columns the exact path reads (queued candidates are re-read from
    // global memory / L2: the rare path is rare)
    const double *ts, *te, *rcp, *sx, *sy, *sz, *dx, *dy, *dz, *ex, *ey, *ez;
    unsigned long long *hit_count;
    uint64_t *keys;
    double *tbeg, *tend;
    uint64_t cap;
    double d2;
    int minor_bits, query_major;
    const int64_t *orig;  // K1 layout position -> start-sorted ordinal (nullptr: identity)
};

__device__ __forceinline__ Cand cand_exact(const FlushCfg &C, int64_t e) {
    Cand r;
    r.ts = C.ts[e]; r.te = C.te[e]; r.rcp = C.rcp[e]; r.ext = __dsub_rn(r.te, r.ts);
    r.sx = C.sx[e]; r.sy = C.sy[e]; r.sz = C.sz[e]; r.dx = C.dx[e]; r.dy = C.dy[e]; r.dz = C.dz[e];
    r.ex = C.ex[e]; r.ey = C.ey[e]; r.ez = C.ez[e];
    return r;
}

// Query record of the FP32 pre-filter (64 B): filter view (start, the
// triangle bound's a and b), the query's end for the separating-axis stage
// (filter.cuh f32_sep_far), and the exact times for windows and per-pair
// overlap counting.
struct __align__(16) QF32 {
    float ts, x, y, z;
    float a, b, te, ex;
    float ey, ez, pad0, pad1;
    double ts64, te64;
};

// Per-warp context of the current sub-tile, read by the flush.
struct WarpCtx {
    uint64_t key_base[K1_GMAX];  // key of (b + g, e_off of candidate 0, query offset 0) without the j term
                            // (g = 0: it.q0; g >= 1: the batch's first query at tile index js_g)
    int64_t f[K1_GMAX];     // first candidate ordinal of batch b + g (K1 layout: e_off = orig - f)
    int js;                 // tile index of batch b + 1's first query (nt when single)
    int jx[K1_GMAX - 2];    // ... of b + 2 .. (groups; nt when absent)
    double wmin_te, wmax;   // min te / max te of the warp's candidates (tb cases)
    int64_t wbase;          // entry ordinal of the warp's candidate 0
    int nvalid;             // valid candidates of the warp (the rest are past the item)
    int nlo;                // ... from this index on (the masked head of a tile aligned below c_lo)
};

// Block-shared state of K1 (both kernels): the flush configuration and the
// per-warp contexts.  The rare path reaches them from the warp index, so the
// hot loops carry none of it in registers.
__shared__ FlushCfg k1_fcfg;
__shared__ WarpCtx k1_wctx[K1_WARPS];
__shared__ unsigned long long k1_hitsx[K1_GMAX - 2];  // per item: hits of batches b + 2 .. (groups)

__device__ __forceinline__ void append_hit_w(const FlushCfg &C, bool hit, uint64_t key, double tb,
                                             double te, int lane) {
    unsigned hm = __ballot_sync(0xffffffffu, hit);
    if (!hm) return;
    int leader = __ffs(hm) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(C.hit_count, (unsigned long long)__popc(hm));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) {
        unsigned long long idx = base + __popc(hm & ((1u << lane) - 1u));
        if (idx < C.cap) {
            C.keys[idx] = key;
            C.tbeg[idx] = tb;
            C.tend[idx] = te;
        }
    }
}

// Exact evaluation of up to 32 queued pairs, one per lane, converged:
// the reference's arithmetic (pair_eval), the second filter and the exact
// solve (core.py:503-558), then the warp-aggregated append.
template <int TA, int TB, bool SLOW>
__device__ __noinline__ void rare_flush(const QRec *__restrict__ qt, const uint32_t *wq, int warp, int n_items,
                                        int lane, unsigned long long &n_hit) {
    const FlushCfg &C = k1_fcfg;
    const double d2 = C.d2;
    const double wmin_te = k1_wctx[warp].wmin_te, wmax_te = k1_wctx[warp].wmax;
    Hit h;
    h.hit = false;
    h.tb = h.te = 0.0;
    uint64_t key = 0;
    int g = 0;
    const uint32_t ent = lane < n_items ? wq[lane] : 0u;
    const int ci = (int)(ent >> 16), j = (int)(ent & 0xffffu);
    // candidates past the item's range can be queued (flagged with a huge
    // threshold) but are not pairs of this item
    if (lane < n_items && ci < k1_wctx[warp].nvalid) {
        const Cand r = cand_exact(C, k1_wctx[warp].wbase + ci);
        const QRec *qrec = qt + j;
        const QVals Q = load_q(qrec);
        double cc, aa, dot, e;
        const bool ex = pair_eval<TA, TB, SLOW>(r, Q, qrec, wmin_te, wmax_te, d2, cc, aa, dot, e);
        // Second filter: q(λ) = aa λ² + 2 dot λ + e can reach 0 on [0, 1] only if
        // q(0) <= 0, q(1) <= 0 or the vertex -dot/aa lies in [0, 1].  Outside all
        // three by m = 2^-30 (cc + d² + aa + 2|dot|) — far above the rounding of
        // these tests — both roots lie strictly outside [0, 1] beyond their own
        // rounding and the reference's solve reports a miss.  Flat spans always
        // go to the exact solve.
        // (only where the reference's discriminant neither overflows nor has
        // a subnormal scale: exact-path tiles can hold any finite input)
        const double mag = __dadd_rn(__dadd_rn(cc, d2), __dadd_rn(aa, 2.0 * fabs(dot)));
        const double m = mag * 0x1p-30;
        const double q1 = __dadd_rn(__dadd_rn(e, dot), __dadd_rn(dot, aa));
        const bool vertex_in = dot <= m && __dadd_rn(dot, aa) >= -m;
        const bool flat = Q.ts == r.te || r.ts == Q.te || Q.ts == Q.te || r.ts == r.te;
        const bool plain = no_overflow(aa, dot, e) && mag >= 0x1p-900;
        if (ex && (flat || !plain || !(e > m) || !(q1 > m) || vertex_in))
            h = rare_pair(r, *qrec, cc, aa, dot, e, d2);
        // candidate ci shifts the entry offset, query j the query offset,
        // within the batch the query belongs to (g: which of the tile's
        // batches, from the tile offsets where they start)
        const int js = k1_wctx[warp].js;
        g = j >= js;
        int jb = g ? js : 0;
#pragma unroll
        for (int i = 0; i < K1_GMAX - 2; ++i) {
            const int ji = k1_wctx[warp].jx[i];
            if (j >= ji) {
                g = i + 2;
                jb = ji;
            }
        }
        const uint64_t jj = (uint64_t)(j - jb);
        // the entry term: the candidate's offset in the warp, or in the K1
        // layout its start-sorted ordinal's offset within the batch's range
        const uint64_t et = C.orig ? (uint64_t)(C.orig[k1_wctx[warp].wbase + ci] - k1_wctx[warp].f[g]) : (uint64_t)ci;
        key = k1_wctx[warp].key_base[g] + (C.query_major ? (jj << C.minor_bits) + et : (et << C.minor_bits) + jj);
    }
    // batches b and b + 1 count in the halves of the lane's counter; b + 2
    // on (groups) in block counters (hits are rare)
    n_hit += h.hit && g < 2 ? (g ? CNT_B1 : 1ull) : 0ull;
    if (h.hit && g >= 2) atomicAdd(&k1_hitsx[g - 2], 1ull);
    append_hit_w(C, h.hit, key, h.tb, h.te, lane);
}


// ── shared kernel helpers ───────────────────────────────────────────────────

// exact start / end time of a staged query record
__device__ __forceinline__ double rec_ts(const QRec &r) { return r.ts; }
__device__ __forceinline__ double rec_te(const QRec &r) { return r.te; }
__device__ __forceinline__ double rec_ts(const QF32 &r) { return r.ts64; }
__device__ __forceinline__ double rec_te(const QF32 &r) { return r.te64; }

__device__ __forceinline__ int lower_bound_pm(const double *pm, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (pm[m] >= v) b = m;
        else a = m + 1;
    }
    return a;
}

// first index with a[m] > v in a non-decreasing array
__device__ __forceinline__ int upper_bound_arr(const double *a_, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (a_[m] <= v) a = m + 1;
        else b = m;
    }
    return a;
}

template <class R>
__device__ __forceinline__ int lower_bound_ts(const R *q, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (rec_ts(q[m]) < v) a = m + 1;
        else b = m;
    }
    return a;
}

template <class R>
__device__ __forceinline__ int lower_bound_te(const R *q, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (rec_te(q[m]) < v) a = m + 1;
        else b = m;
    }
    return a;
}

template <class R>
__device__ __forceinline__ int upper_bound_ts(const R *q, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (rec_ts(q[m]) <= v) a = m + 1;
        else b = m;
    }
    return a;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// lo[k] = #{j : te_j < ts[k]} and hi[k] = #{j : ts_j <= te[k]} over a tile
// whose start and end times both ascend, given as plain arrays padded with
// +inf up to twice the next power of two >= nt: all 2 CPT searches advance
// together by binary lifting, so each step issues 2 CPT independent shared
// loads and no bounds checks.
// Entries of the FP32 kernel's window arrays (running max / suffix min of
// the tile's end / start times, +inf padded).  Binary lifting over nt
// entries (tile_bounds) reads below 2 pow2(nt), window_bounds below
// K1_TQ + 64; the wide build (1,024-query tiles, where 2 K1_TQ would not
// fit beside 16 warps' shared memory) pads to K1_TQ + 64 and clamps
// tile_bounds' reads.
#ifdef K1_WIDE
constexpr int K1_PMN = K1_TQ + 64;
#else
constexpr int K1_PMN = 2 * K1_TQ;
#endif

template <int CPT>
__device__ __forceinline__ void tile_bounds(const double *qts, const double *qte, int nt, const double (&ts)[CPT],
                                            const double (&te)[CPT], int (&lo)[CPT], int (&hi)[CPT]) {
    // positions kept as shared-window byte addresses of the next unread record
    const uint32_t bs = (uint32_t)__cvta_generic_to_shared(qts), be = (uint32_t)__cvta_generic_to_shared(qte);
    uint32_t pl[CPT], ph[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        pl[k] = be;
        ph[k] = bs;
    }
    if (nt > 0) {
        for (uint32_t sb = 8u * (nt > 1 ? 1u << (32 - __clz(nt - 1)) : 1u); sb >= 8u; sb >>= 1) {
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                double vl, vh;
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(vl) : "r"(pl[k] + sb - 8u));
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(vh) : "r"(ph[k] + sb - 8u));
                if (K1_PMN < 2 * K1_TQ) {  // wide build: past the padding reads +inf
                    if (pl[k] + sb - 8u >= be + 8u * K1_PMN) vl = INFINITY;
                    if (ph[k] + sb - 8u >= bs + 8u * K1_PMN) vh = INFINITY;
                }
                pl[k] += vl < ts[k] ? sb : 0u;
                ph[k] += vh <= te[k] ? sb : 0u;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        lo[k] = (int)((pl[k] - be) >> 3);
        hi[k] = (int)((ph[k] - bs) >> 3);
    }
}

__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Decode work item `item` of the plan (k_plan_items: per work unit,
// candidate tiles of ct entries times query tiles of tqs queries; a shared
// unit has one tile holding both batches' queries).
__device__ __forceinline__ ItemCtx decode_item(const K1Launch &L, int64_t item, int64_t ct, int64_t tqs) {
    // unit = last u with item_off[u] <= item (a non-empty unit)
    const int mode = (int)L.plan.meta[3];
    int64_t a = 0, z = plan_units_mode(L.plan.nb, mode);
    while (z - a > 1) {
        int64_t m = (a + z) >> 1;
        if (L.plan.item_off[m] <= item) a = m;
        else z = m;
    }
    const UnitT<K1_GMAX> U = plan_unit<K1_GMAX>(L.plan, a, tqs, mode);  // (the host launches octets in the wide build only)
    const int64_t local = item - L.plan.item_off[a];
    ItemCtx c;
    c.b = U.b;
    c.b1 = U.b1;
    int64_t tc;
    if (U.b1 >= 0) {  // shared: one tile with all the group's queries
        tc = local;
        c.q0 = 0;
        c.nt = (int)U.s;
        c.js = (int)U.js;
#pragma unroll
        for (int i = 0; i < K1_GMAX - 2; ++i) c.jx[i] = (int)U.jx[i];
    } else {
        const int64_t tq_n = (U.s + tqs - 1) / tqs;
        const int64_t tq = local % tq_n;
        tc = local / tq_n;
        c.q0 = tq * tqs;
        c.nt = (int)(U.s - c.q0 < tqs ? U.s - c.q0 : tqs);
        c.js = c.nt;
#pragma unroll
        for (int i = 0; i < K1_GMAX - 2; ++i) c.jx[i] = c.nt;
    }
    c.lo_q = U.lo_q + c.q0;
    // K1 layout (L.cull): tiles start at a BOX_GROUP multiple (k_plan_items
    // counts them the same way); candidates before U.f are masked
    const int64_t f0 = L.cull ? (U.f / BOX_GROUP) * BOX_GROUP : U.f;
    c.first_c = f0 + tc * ct;
    c.c_lo = U.f;
    c.c_hi = c.first_c + ct - 1 < U.l ? c.first_c + ct - 1 : U.l;
    return c;
}

__device__ __forceinline__ void fill_flush_cfg(const K1Launch &L) {
    FlushCfg &f = k1_fcfg;
    f.ts = L.e.ts; f.te = L.e.te; f.rcp = L.e.rcp;
    f.sx = L.e.sx; f.sy = L.e.sy; f.sz = L.e.sz;
    f.dx = L.e.dx; f.dy = L.e.dy; f.dz = L.e.dz;
    f.ex = L.e.ex; f.ey = L.e.ey; f.ez = L.e.ez;
    f.hit_count = L.hit_count;
    f.keys = L.keys;
    f.tbeg = L.tbeg;
    f.tend = L.tend;
    f.cap = L.cap;
    f.d2 = L.d2;
    f.minor_bits = L.minor_bits;
    f.query_major = L.query_major;
    f.orig = L.orig;
}

// Key bases of a warp's sub-tile (lane 0): without a K1 layout the entry
// offset of candidate 0 is folded in; with one each hit adds its own
// (orig - f).
__device__ __forceinline__ void set_key_bases(const K1Launch &L, const ItemCtx &it, int64_t wbase, int warp) {
    const int nb = item_batches(it);
    for (int g = 0; g < K1_GMAX; ++g) {
        const int64_t b = it.b + g;
        const int64_t f = g < nb ? L.plan.first[b] : 0;
        const int64_t q0 = g == 0 ? it.q0 : 0;
        k1_wctx[warp].f[g] = f;
        k1_wctx[warp].key_base[g] = g >= nb ? 0 : (L.orig ? make_key(L, b, 0, q0) : make_key(L, b, wbase - f, q0));
    }
    k1_wctx[warp].js = it.js;
#pragma unroll
    for (int i = 0; i < K1_GMAX - 2; ++i) k1_wctx[warp].jx[i] = it.jx[i];
}

// Running max (warp 0) / suffix min (warp 1) of the tile's end times.
template <class R>
__device__ __forceinline__ void te_scans(const R *q, int nt, double *pm, double *sm, int warp, int lane) {
    if (warp == 1) {
        double carry = INFINITY;
        for (int base = ((nt - 1) & ~31); base >= 0; base -= 32) {
            int j = base + lane;
            double v = j < nt ? rec_te(q[j]) : INFINITY;
            for (int o = 1; o < 32; o <<= 1) {
                double t = __shfl_down_sync(0xffffffffu, v, o);
                if (lane + o < 32) v = fmin(v, t);
            }
            v = fmin(v, carry);
            if (j < nt) sm[j] = v;
            carry = __shfl_sync(0xffffffffu, v, 0);
        }
    }
    if (warp == 0) {
        double carry = -INFINITY;
        for (int base = 0; base < nt; base += 32) {
            int j = base + lane;
            double v = j < nt ? rec_te(q[j]) : -INFINITY;
            for (int o = 1; o < 32; o <<= 1) {
                double t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v = fmax(v, t);
            }
            v = fmax(v, carry);
            if (j < nt) pm[j] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
}

// Window of the staged queries that can overlap a warp's candidates and its
// start-time case ranges [jlo, ja) TA_C, [ja, jb) TA_BOTH, [jb, jhi) TA_R;
// the four searches run on lanes 0..3 in parallel.
template <class R>
__device__ __forceinline__ int4 warp_window(const R *q, const double *pm, int nt, bool unsorted, double wmin,
                                            double wmax, double wmax_ts, int lane) {
    if (unsorted) return make_int4(0, 0, nt, nt);  // everything in the mixed range
    int v = 0;
    if (lane == 0) v = lower_bound_pm(pm, nt, wmin);        // running max te >= min ts
    else if (lane == 1) v = upper_bound_ts(q, nt, wmax);    // first query starting after max te
    else if (lane == 2) v = lower_bound_ts(q, nt, wmin);    // first cts >= min ts
    else if (lane == 3) v = upper_bound_ts(q, nt, wmax_ts); // first cts >  max ts
    const int jlo = __shfl_sync(0xffffffffu, v, 0);
    int jhi = __shfl_sync(0xffffffffu, v, 1);
    const int ja0 = __shfl_sync(0xffffffffu, v, 2), jb0 = __shfl_sync(0xffffffffu, v, 3);
    if (jhi < jlo) jhi = jlo;
    const int ja = clampi(ja0, jlo, jhi);
    const int jb = clampi(jb0, ja, jhi);
    return make_int4(jlo, ja, jb, jhi);
}


// Flush the warp's queue 32 pairs at a time while 32 or more are waiting,
// and the last partial batch when the range is done (qn: warp-uniform).
template <int TA, int TB, bool SLOW, int CPT>
__device__ __forceinline__ void flush_queue(const QRec *__restrict__ qt, uint32_t *wq, int warp, int lane, int &qn,
                                            bool done, unsigned long long &n_hit) {
    while (qn >= 32 || (done && qn > 0)) {
        const int nf = qn < 32 ? qn : 32;
        __syncwarp();
        rare_flush<TA, TB, SLOW>(qt, wq, warp, nf, lane, n_hit);
        __syncwarp();
        uint32_t mv[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) mv[k] = lane + 32 * (k + 1) < qn ? wq[lane + 32 * (k + 1)] : 0u;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < CPT; ++k)
            if (lane + 32 * (k + 1) < qn) wq[lane + 32 * k] = mv[k];
        qn -= nf;
    }
}

// Per-batch 64-bit counters: warp sums → block sums → atomics per item
// (low halves to batch b, high halves to b1).
// red_ev (optional): the block's evaluated-pair sum, added to L.eval_count.
__device__ __forceinline__ void item_counters(const K1Launch &L, const ItemCtx &it, unsigned long long n_ov,
                                              unsigned long long n_hit, int lane, int tid,
                                              unsigned long long *red, const unsigned long long *red_ev = nullptr) {
    for (int o = 16; o; o >>= 1) {
        n_ov += __shfl_xor_sync(0xffffffffu, n_ov, o);
        n_hit += __shfl_xor_sync(0xffffffffu, n_hit, o);
    }
    if (lane == 0 && (n_ov | n_hit)) {
        atomicAdd(&red[0], n_ov & 0xffffffffull);
        atomicAdd(&red[1], n_hit & 0xffffffffull);
        atomicAdd(&red[2], n_ov >> 32);
        atomicAdd(&red[3], n_hit >> 32);
    }
    __syncthreads();
    if (tid == 0) {
        if (red[0]) atomicAdd(&L.plan.ovl[it.b], red[0]);
        if (red[1]) atomicAdd(&L.plan.hits[it.b], red[1]);
        if (it.b1 >= 0 && red[2]) atomicAdd(&L.plan.ovl[it.b1], red[2]);
        if (it.b1 >= 0 && red[3]) atomicAdd(&L.plan.hits[it.b1], red[3]);
        if (it.b1 >= 0) {  // groups: batches b + 2 .. (rare_flush counted them)
            for (int i = 0; i < K1_GMAX - 2; ++i)
                if (it.jx[i] < it.nt && k1_hitsx[i]) atomicAdd(&L.plan.hits[it.b + 2 + i], k1_hitsx[i]);
        }
        for (int i = 0; i < K1_GMAX - 2; ++i) k1_hitsx[i] = 0;  // for the next item (the barrier below orders it)
        if (red_ev && *red_ev) atomicAdd(L.eval_count, *red_ev);
    }
    __syncthreads();
}

// Temporal overlaps of a lane's candidates with staged queries j0..j1-1
// (TSK_OVERLAPS_ONLY: the perfmodel's temporal-miss fractions).
template <int CPT, class R>
__device__ __forceinline__ unsigned long long count_overlaps(const R *q, int j0, int j1, int js, const double (&ts)[CPT],
                                                             const double (&te)[CPT]) {
    unsigned long long n = 0;
    for (int j = j0; j < j1; ++j) {
        const double cts = rec_ts(q[j]), cte = rec_te(q[j]);
        const unsigned long long inc = j >= js ? CNT_B1 : 1ull;
#pragma unroll
        for (int k = 0; k < CPT; ++k) n += (ts[k] <= cte && cts <= te[k]) ? inc : 0ull;
    }
    return n;
}

// Overlaps of index range [a, b) split at js into the two batch halves.
__device__ __forceinline__ unsigned long long split_count(int a, int b, int js) {
    if (b <= a) return 0ull;
    const int lo = b < js ? b : js;   // [a, min(b, js)) in batch b
    const int hi = a > js ? a : js;   // [max(a, js), b) in batch b1
    return (unsigned long long)(lo > a ? lo - a : 0) + (unsigned long long)(b > hi ? b - hi : 0) * CNT_B1;
}

}  // namespace tsk
