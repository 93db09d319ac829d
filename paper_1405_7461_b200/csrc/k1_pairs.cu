// k1_pairs.cu — K1, the moving-distance pair kernel (GPUTrajDistSearch).
//
// Replaces core.pair_intervals (/root/reference/pkg/src/trajseek/core.py:464-565)
// driven by engine.execute_batch/_run_chunks (engine.py:78-148) for every
// batch of a plan at once.
//
// Work decomposition.  A work item is (batch b, candidate tile, query tile):
// up to K1_TQ queries of the batch are staged in shared memory as 112-byte
// records, each thread holds K1_CPT candidate entry segments in registers
// (lane l of a warp holds candidates l, l+32, ... of the warp's 32*K1_CPT
// consecutive ones; sub-tiles of 256*K1_CPT candidates are walked in turn),
// and every warp loops over the window of staged queries that can overlap
// any of its candidates (entries and queries are both start-time sorted, so
// the window is two binary searches).  Items are claimed from a global
// atomic counter by a persistent grid.
//
// Arithmetic.  For an overlapping pair the reference clips both segments
// to [ta, tb] and solves the quadratic (core.py:503-565).  With span > 0,
// only the earlier-starting segment is interpolated at ta and only the
// later-ending one at tb; the other endpoint is taken verbatim, which is
// what the np.where selections of core.py:514 produce.  Each warp splits
// its query window into the three start-time cases (query first / entry
// first / mixed); in the mixed range both are interpolated at ta, exact
// because the later starter has f == 0.  The end-time case is proven for a
// whole range from the tile's running max / suffix min of end times, else
// decided per query.  Zero-length shared spans (touching extents,
// waypoints) take the exact rare path.  The hit test uses
// dq = dot^2 - aa*(cc - d^2) (= disc/4, exact scaling) with a tiny negative
// margin; the few candidates that pass are re-solved with the reference's
// exact root formula.  All ops are binary64 with explicit rounding;
// divisions use qdiv() with a per-segment RN(1/ext).
#include <atomic>

#include "filter.cuh"
#include "tsk_internal.cuh"

#ifndef K1_CPT
#define K1_CPT 2
#endif
#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS (K1_CPT == 1 ? 3 : 2)
#endif
#ifndef K1_MIN_BLOCKS_F32
#define K1_MIN_BLOCKS_F32 3
#endif

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

__device__ __forceinline__ QVals load_q(uint32_t a) {
    QVals q;
    double vz_unused;
    lds2(a + 0, q.ts, q.te);
    lds2(a + 16, q.sx, q.sy);
    lds2(a + 32, q.sz, q.ext);
    lds2(a + 64, vz_unused, q.dz);
    lds2(a + 80, q.dx, q.dy);
    q.rcp = q.ext > 0.0 ? __drcp_rn(q.ext) : 0.0;
    return q;
}

// Filter view of a query record (QRec bytes 0..95).
__device__ __forceinline__ QF load_qf(uint32_t a) {
    QF q;
    lds2(a + 0, q.ts, q.te);
    lds2(a + 16, q.sx, q.sy);
    lds2(a + 32, q.sz, q.ext);
    lds2(a + 48, q.vx, q.vy);
    lds2(a + 64, q.vz, q.dz);
    lds2(a + 80, q.dx, q.dy);
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
        lo = r1 < r2 ? r1 : r2;
        hi = r1 > r2 ? r1 : r2;
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
    int64_t q0;                      // first query offset within batch (tile)
    int nt;                          // staged queries
};

__device__ __forceinline__ void append_hit(const K1Launch &L, bool hit, uint64_t key, double tb,
                                           double te, int lane) {
    unsigned hm = __ballot_sync(0xffffffffu, hit);
    if (!hm) return;
    int leader = __ffs(hm) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(L.hit_count, (unsigned long long)__popc(hm));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) {
        unsigned long long idx = base + __popc(hm & ((1u << lane) - 1u));
        if (idx < L.cap) {
            L.keys[idx] = key;
            L.tbeg[idx] = tb;
            L.tend[idx] = te;
        }
    }
}

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
__device__ __forceinline__ bool pair_eval(const Cand &r, const QVals &Q, uint32_t qa, double wmin_te,
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
        double flag_unused;
        lds2(qa + 96, cbx, cby);
        lds2(qa + 112, cbz, flag_unused);
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
        double qex, qey, qez, flag_unused;
        lds2(qa + 96, qex, qey);
        lds2(qa + 112, qez, flag_unused);
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

// Per-warp shared state for the rare path: a queue of flagged
// (candidate, query) pairs.
constexpr int K1_WARPS = K1_THREADS / 32;
// Queue entries per warp.  A query iteration starts with fewer than 32
// queued and appends at most 32 * K1_CPT.
constexpr int K1_QCAP = 32 * (K1_CPT + 1);

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
};

__device__ __forceinline__ Cand cand_exact(const FlushCfg &C, int64_t e) {
    Cand r;
    r.ts = C.ts[e]; r.te = C.te[e]; r.rcp = C.rcp[e]; r.ext = __dsub_rn(r.te, r.ts);
    r.sx = C.sx[e]; r.sy = C.sy[e]; r.sz = C.sz[e]; r.dx = C.dx[e]; r.dy = C.dy[e]; r.dz = C.dz[e];
    r.ex = C.ex[e]; r.ey = C.ey[e]; r.ez = C.ez[e];
    return r;
}

// Query record of the FP32 pre-filter (48 B): filter view + exact times
// for per-pair overlap counting.
struct __align__(16) QF32 {
    float ts, x, y, z;
    float a, b, pad0, pad1;
    double ts64, te64;
};

// Per-warp context of the current sub-tile, read by the flush.
struct WarpCtx {
    uint64_t key_base0;     // key of (b, e_off of candidate 0, it.q0) without the j term
    double wmin_te, wmax;   // min te / max te of the warp's candidates (tb cases)
    int64_t wbase;          // entry ordinal of the warp's candidate 0
    int nvalid;             // valid candidates of the warp (the rest are past the item)
};

// Block-shared state of K1 (both kernels): the flush configuration, the
// per-warp contexts, and the dynamic region (FP32 query records, then the
// per-warp staged candidates and queues).  The rare path reaches all of it
// from the warp index, so the hot loops carry none of it in registers.
__shared__ FlushCfg k1_fcfg;
__shared__ WarpCtx k1_wctx[K1_WARPS];
extern __shared__ __align__(16) unsigned char k1_dyn[];

__device__ __forceinline__ QF32 *k1_sqf() { return reinterpret_cast<QF32 *>(k1_dyn); }
__device__ __forceinline__ uint32_t *warp_q(int warp) {
    return reinterpret_cast<uint32_t *>(k1_dyn + sizeof(QF32) * K1_TQ) + warp * K1_QCAP;
}

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
__device__ __noinline__ void rare_flush(const QRec *__restrict__ sq, int warp, int n_items, int lane,
                                        unsigned &n_hit) {
    const FlushCfg &C = k1_fcfg;
    const double d2 = C.d2;
    const uint32_t *wq = warp_q(warp);
    const double wmin_te = k1_wctx[warp].wmin_te, wmax_te = k1_wctx[warp].wmax;
    Hit h;
    h.hit = false;
    h.tb = h.te = 0.0;
    uint64_t key = 0;
    const uint32_t ent = lane < n_items ? wq[lane] : 0u;
    const int ci = (int)(ent >> 16), j = (int)(ent & 0xffffu);
    // candidates past the item's range can be queued (flagged with a huge
    // threshold) but are not pairs of this item
    if (lane < n_items && ci < k1_wctx[warp].nvalid) {
        const Cand r = cand_exact(C, k1_wctx[warp].wbase + ci);
        const uint32_t qa = (uint32_t)__cvta_generic_to_shared(sq) + (uint32_t)j * (uint32_t)sizeof(QRec);
        const QVals Q = load_q(qa);
        double cc, aa, dot, e;
        const bool ex = pair_eval<TA, TB, SLOW>(r, Q, qa, wmin_te, wmax_te, d2, cc, aa, dot, e);
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
            h = rare_pair(r, sq[j], cc, aa, dot, e, d2);
        // candidate ci shifts the entry offset, query j the query offset
        key = k1_wctx[warp].key_base0 + (C.query_major ? ((uint64_t)j << C.minor_bits) + (uint64_t)ci
                                           : ((uint64_t)ci << C.minor_bits) + (uint64_t)j);
    }
    n_hit += h.hit ? 1u : 0u;
    append_hit_w(C, h.hit, key, h.tb, h.te, lane);
}

// Evaluation modes of the common loop (per item / warp sub-tile):
//   K1_F32  FP32 pre-filter (below); survivors are re-evaluated exactly
//   K1_F64  the FP64 filter of filter.cuh (items whose magnitudes are
//           outside the FP32 pre-filter's validity)
//   K1_ALL  every overlapping pair is queued for the exact IEEE path
//           (extreme-exponent tiles, launches outside the filter bounds)
enum { K1_F32 = 0, K1_F64 = 1, K1_ALL = 2 };

// FP32 pre-filter: filter.cuh (f32_item / f32_query / f32_cand / f32_flag).

__device__ __forceinline__ void lds4f(uint32_t a, float &x, float &y, float &z, float &w) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
}

// One warp, K1_CPT candidates per lane, staged queries j0..j1-1 of one
// (TA, TB) case.  CNT: count overlaps per iteration; otherwise the caller
// counts them for the whole range by binary search and lanes that do not
// overlap a query are rejected on the rare path (window edges only).
// Flagged pairs are queued and evaluated exactly 32 at a time (rare_flush),
// so hit-dense workloads do not serialise the warp on divergent code.
template <int TA, int TB, int MODE, bool CNT>
__device__ __forceinline__ void pair_run(const QRec *__restrict__ sq,
                                         const QF32 *__restrict__ sqf, int j0, int j1,
                                         const CandF (&r)[K1_CPT], const CandF32 (&c32)[K1_CPT],
                                         double wmin_te, double wmax_te, int warp, int lane,
                                         unsigned &n_ov, unsigned &n_hit, const FilterK &K) {
    constexpr bool SLOW = MODE == K1_ALL;
    uint32_t *const wq = warp_q(warp);
    constexpr uint32_t STRIDE = MODE == K1_F32 ? (uint32_t)sizeof(QF32) : (uint32_t)sizeof(QRec);
    const uint32_t base = MODE == K1_F32 ? (uint32_t)__cvta_generic_to_shared(sqf)
                                         : (uint32_t)__cvta_generic_to_shared(sq);
    int qn = 0;  // queued entries (warp-uniform)
    const uint32_t qa0 = base + (uint32_t)j0 * STRIDE;
    const uint32_t qa_end = qa0 + (uint32_t)(j1 - j0) * STRIDE;
    uint32_t qa = qa0;
    for (;;) {
        // Inner loop, driven by the record address alone and free of calls
        // (the flush is called outside it, so nothing it holds needs saving
        // around a call): loads, math, one vote, one branch per query.  Flags
        // are queued; it exits when 32 or more are waiting.
        for (; qa < qa_end; qa += STRIDE) {
            bool cand[K1_CPT];
            if (MODE == K1_F32) {
                float qts, qx, qy, qz, qa4, qb4, p0, p1;
                lds4f(qa, qts, qx, qy, qz);
                lds4f(qa + 16, qa4, qb4, p0, p1);
                double cts = 0.0, cte = 0.0;
                if (CNT) lds2(qa + 32, cts, cte);
#pragma unroll
                for (int k = 0; k < K1_CPT; ++k) {
                    bool ov = true;
                    if (CNT) {
                        if (TA == TA_C) ov = r[k].ts <= cte;
                        else if (TA == TA_R) ov = cts <= r[k].te;
                        else ov = r[k].ts <= cte && cts <= r[k].te;
                        n_ov += ov ? 1u : 0u;
                    }
                    cand[k] = f32_flag(c32[k], qts, qx, qy, qz, qa4, qb4) && ov;
                }
            } else if (MODE == K1_ALL) {
                double cts, cte;
                lds2(qa, cts, cte);
#pragma unroll
                for (int k = 0; k < K1_CPT; ++k) {
                    const bool ov = r[k].ts <= cte && cts <= r[k].te;  // invalid lanes: ts = +inf
                    if (CNT) n_ov += ov ? 1u : 0u;
                    cand[k] = ov;
                }
            } else {
                const QF Q = load_qf(qa);
#pragma unroll
                for (int k = 0; k < K1_CPT; ++k) {
                    bool ov = true;
                    if (CNT) {
                        // TA_C: the query started first, so it overlaps iff it ends
                        // at or after r.ts; TA_R: iff it starts at or before r.te
                        // (invalid lanes: ts = +inf, te = -inf)
                        if (TA == TA_C) ov = r[k].ts <= Q.te;
                        else if (TA == TA_R) ov = Q.ts <= r[k].te;
                        else ov = r[k].ts <= Q.te && Q.ts <= r[k].te;
                        n_ov += ov ? 1u : 0u;
                    }
                    cand[k] = pair_filter<TA, TB>(r[k], Q, wmin_te, wmax_te, K) && ov;
                }
            }
            bool any = false;
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k) any |= cand[k];
            if (!__any_sync(0xffffffffu, any)) continue;
            // rare: queue the flagged pairs of this query (qn < 32 on entry)
            const uint32_t j = (qa - base) / STRIDE;
            unsigned lt;
            asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k) {
                const unsigned m = __ballot_sync(0xffffffffu, cand[k]);
                if (cand[k]) wq[qn + __popc(m & lt)] = ((uint32_t)(k * 32 + lane) << 16) | j;
                qn += __popc(m);
            }
            if (qn >= 32) {
                qa += STRIDE;
                break;
            }
        }
        // flush 32 at a time; the last partial batch at the end of the range
        const bool done = qa >= qa_end;
        while (qn >= 32 || (done && qn > 0)) {
            const int nf = qn < 32 ? qn : 32;
            __syncwarp();
            rare_flush<TA, TB, SLOW>(sq, warp, nf, lane, n_hit);
            __syncwarp();
            uint32_t mv[K1_CPT];
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k) mv[k] = lane + 32 * (k + 1) < qn ? wq[lane + 32 * (k + 1)] : 0u;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k)
                if (lane + 32 * (k + 1) < qn) wq[lane + 32 * k] = mv[k];
            qn -= nf;
        }
        if (done) break;
    }
}

__device__ __forceinline__ int lower_bound_pm(const double *pm, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (pm[m] >= v) b = m;
        else a = m + 1;
    }
    return a;
}

__device__ __forceinline__ int lower_bound_ts(const QRec *q, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (q[m].ts < v) a = m + 1;
        else b = m;
    }
    return a;
}

__device__ __forceinline__ int lower_bound_te(const QRec *q, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (q[m].te < v) a = m + 1;
        else b = m;
    }
    return a;
}

__device__ __forceinline__ int upper_bound_ts(const QRec *q, int n, double v) {
    int a = 0, b = n;
    while (a < b) {
        int m = (a + b) >> 1;
        if (q[m].ts <= v) a = m + 1;
        else b = m;
    }
    return a;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// The FP32 inner loop is a leaf function (no calls, so nothing has to be
// saved around one and it gets clean registers): it scans queries from qa
// until 32 or more flags are queued or the range ends, and returns
// (qa, queued, overlaps).  The caller flushes and resumes.
static_assert(K1_CPT == 2, "f32_scan takes two candidates by value");
template <int TA, bool CNT>
__device__ __noinline__ uint4 f32_scan(uint32_t qa, uint32_t qa_end, uint32_t base, int qn, CandF32 c0,
                                       CandF32 c1, double ts0, double te0, double ts1, double te1, int warp,
                                       int lane) {
    uint32_t *const wq = warp_q(warp);
    const CandF32 c32[K1_CPT] = {c0, c1};
    const double rts[K1_CPT] = {ts0, ts1}, rte[K1_CPT] = {te0, te1};
    unsigned n_ov = 0;
    for (; qa < qa_end; qa += (uint32_t)sizeof(QF32)) {
        float qts, qx, qy, qz, qa4, qb4, p0, p1;
        lds4f(qa, qts, qx, qy, qz);
        lds4f(qa + 16, qa4, qb4, p0, p1);
        double cts = 0.0, cte = 0.0;
        if (CNT) lds2(qa + 32, cts, cte);
        bool cand[K1_CPT];
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k) {
            bool ov = true;
            if (CNT) {
                if (TA == TA_C) ov = rts[k] <= cte;
                else if (TA == TA_R) ov = cts <= rte[k];
                else ov = rts[k] <= cte && cts <= rte[k];
                n_ov += ov ? 1u : 0u;
            }
            cand[k] = f32_flag(c32[k], qts, qx, qy, qz, qa4, qb4) && ov;
        }
        bool any = false;
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k) any |= cand[k];
        if (!__any_sync(0xffffffffu, any)) continue;
        const uint32_t j = (qa - base) / (uint32_t)sizeof(QF32);
        unsigned lt;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, cand[k]);
            if (cand[k]) wq[qn + __popc(m & lt)] = ((uint32_t)(k * 32 + lane) << 16) | j;
            qn += __popc(m);
        }
        if (qn >= 32) {
            qa += (uint32_t)sizeof(QF32);
            break;
        }
    }
    return make_uint4(qa, (unsigned)qn, n_ov, 0u);
}

// FP32 range: scan, flush 32 at a time, resume.
template <int TA, int TB, bool CNT>
__device__ __forceinline__ void f32_range(const QRec *__restrict__ sq, const QF32 *__restrict__ sqf, int j0,
                                          int j1, const CandF (&r)[K1_CPT], const CandF32 (&c32)[K1_CPT],
                                          int warp, int lane, unsigned &n_ov, unsigned &n_hit) {
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sqf);
    uint32_t qa = base + (uint32_t)j0 * (uint32_t)sizeof(QF32);
    const uint32_t qa_end = base + (uint32_t)j1 * (uint32_t)sizeof(QF32);
    uint32_t *const wq = warp_q(warp);
    int qn = 0;
    for (;;) {
        const uint4 o = f32_scan<TA, CNT>(qa, qa_end, base, qn, c32[0], c32[1], r[0].ts, r[0].te, r[1].ts,
                                          r[1].te, warp, lane);
        qa = o.x;
        qn = (int)o.y;
        n_ov += o.z;
        const bool done = qa >= qa_end;
        while (qn >= 32 || (done && qn > 0)) {
            const int nf = qn < 32 ? qn : 32;
            __syncwarp();
            rare_flush<TA, TB, false>(sq, warp, nf, lane, n_hit);
            __syncwarp();
            uint32_t mv[K1_CPT];
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k) mv[k] = lane + 32 * (k + 1) < qn ? wq[lane + 32 * (k + 1)] : 0u;
            __syncwarp();
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k)
                if (lane + 32 * (k + 1) < qn) wq[lane + 32 * k] = mv[k];
            qn -= nf;
        }
        if (done) break;
    }
}

template <int TA, int TB, int MODE, bool CNT>
__device__ __forceinline__ void range_run(const QRec *__restrict__ sq, const QF32 *__restrict__ sqf, int j0,
                                          int j1, const CandF (&r)[K1_CPT], const CandF32 (&c32)[K1_CPT],
                                          double wmin_te, double wmax, int warp, int lane,
                                          unsigned &n_ov, unsigned &n_hit, const FilterK &K) {
    if (MODE == K1_F32) {
        if (j0 < j1) f32_range<TA, TB, CNT>(sq, sqf, j0, j1, r, c32, warp, lane, n_ov, n_hit);
    } else {
        pair_run<TA, TB, MODE, CNT>(sq, sqf, j0, j1, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    }
}

// The three start-time ranges of a warp's window in one mode.  C_BISECT:
// every query of the TA_C range ends before all candidates and te is
// sorted, so overlaps are counted by bisection; R_BISECT likewise for the
// TA_R range (every query ends after all candidates).
template <int MODE>
__device__ __forceinline__ void run_cases(const K1Launch &L, const QRec *__restrict__ sq,
                                          const QF32 *__restrict__ sqf, int nt, int jlo, int ja, int jb,
                                          int jhi, bool c_bisect, bool r_bisect,
                                          const CandF (&r)[K1_CPT], const CandF32 (&c32)[K1_CPT],
                                          double wmin_te, double wmax, int warp, int lane,
                                          unsigned &n_ov, unsigned &n_hit, const FilterK &K) {
    if (c_bisect) {
        // overlap <=> r.ts <= cte; cte ascending over the tile
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k)
            n_ov += (unsigned)(ja - clampi(lower_bound_te(sq, nt, r[k].ts), jlo, ja));
        range_run<TA_C, TB_R, MODE, false>(sq, sqf, jlo, ja, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    } else {
        range_run<TA_C, TB_DYN, MODE, true>(sq, sqf, jlo, ja, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    }
    range_run<TA_BOTH, TB_DYN, MODE, true>(sq, sqf, ja, jb, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    if (r_bisect) {
        // overlap <=> cts <= r.te; cts ascending over the tile
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k)
            n_ov += (unsigned)(clampi(upper_bound_ts(sq, nt, r[k].te), jb, jhi) - jb);
        range_run<TA_R, TB_C, MODE, false>(sq, sqf, jb, jhi, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    } else {
        range_run<TA_R, TB_DYN, MODE, true>(sq, sqf, jb, jhi, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    }
}

// F32: the FP32 pre-filter kernel (items outside its validity take the
// exact path); otherwise the FP64-filter kernel.  Two kernels, so that each
// gets its own register allocation.
template <bool F32>
__global__ void __launch_bounds__(K1_THREADS, F32 ? K1_MIN_BLOCKS_F32 : K1_MIN_BLOCKS) k1_pairs(K1Launch L) {
    __shared__ QRec sq[K1_TQ];
    __shared__ double f32b[8];    // per-item magnitude bounds (FP32 pre-filter)
    __shared__ F32Item fi_sh;     // the item's FP32 origin and error bound
    __shared__ double pm[K1_TQ];  // running max of te over the tile
    __shared__ double sm[K1_TQ];  // suffix min of te over the tile
    __shared__ ItemCtx it_sh;
    __shared__ int64_t item_sh;
    __shared__ unsigned long long red_ov, red_hit;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        k1_fcfg.ts = L.e.ts; k1_fcfg.te = L.e.te; k1_fcfg.rcp = L.e.rcp;
        k1_fcfg.sx = L.e.sx; k1_fcfg.sy = L.e.sy; k1_fcfg.sz = L.e.sz;
        k1_fcfg.dx = L.e.dx; k1_fcfg.dy = L.e.dy; k1_fcfg.dz = L.e.dz;
        k1_fcfg.ex = L.e.ex; k1_fcfg.ey = L.e.ey; k1_fcfg.ez = L.e.ez;
        k1_fcfg.hit_count = L.hit_count;
        k1_fcfg.keys = L.keys;
        k1_fcfg.tbeg = L.tbeg;
        k1_fcfg.tend = L.tend;
        k1_fcfg.cap = L.cap;
        k1_fcfg.d2 = L.d2;
        k1_fcfg.minor_bits = L.minor_bits;
        k1_fcfg.query_major = L.query_major;
    }
    QF32 *const sqf = k1_sqf();
    const int64_t total = L.plan.meta[0];
    const int sub = (int)L.plan.meta[1];
    const int64_t tqs = L.plan.meta[2];  // query tile size chosen by k_plan_items (<= K1_TQ)
    constexpr int64_t STRIDE = (int64_t)K1_THREADS * K1_CPT;  // candidates per sub-tile
    const int64_t ct = STRIDE * sub;
    const int64_t nb = L.plan.nb;
    // filter constants (filter.cuh); C = max |coordinate| of entries and queries
    const double cq = __longlong_as_double((long long)*L.q_cmax_bits);
    const double cmax = L.db_cmax > cq ? L.db_cmax : cq;
    FilterK K = filter_consts(cmax, L.d2);
    K.km = L.filter_km;
    const bool launch_exact = !filter_ok(cmax, L.d2);
    const double dthr = sqrt(L.d2);  // d (RN(d*d) rounds; sqrt(RN(d^2)) >= d (1 - 2^-52))
    const bool launch_f32 = F32 && !launch_exact && L.d2 <= 0x1p120 && cmax <= 0x1p60;

    for (;;) {
        if (tid == 0) {
            int64_t item = (int64_t)atomicAdd(L.item_counter, 1ull);
            item_sh = item;
            if (item < total) {
                // batch = last b with item_off[b] <= item (a non-empty batch)
                int64_t a = 0, z = nb;
                while (z - a > 1) {
                    int64_t m = (a + z) >> 1;
                    if (L.plan.item_off[m] <= item) a = m;
                    else z = m;
                }
                const int64_t b = a;
                const int64_t local = item - L.plan.item_off[b];
                const int64_t s_b = L.plan.hi[b] - L.plan.lo[b] + 1;
                const int64_t tq_n = (s_b + tqs - 1) / tqs;
                const int64_t tq = local % tq_n, tc = local / tq_n;
                ItemCtx c;
                c.b = b;
                c.q0 = tq * tqs;
                c.lo_q = L.plan.lo[b] + c.q0;
                c.nt = (int)(s_b - c.q0 < tqs ? s_b - c.q0 : tqs);
                c.first_c = L.plan.first[b] + tc * ct;
                c.c_hi = c.first_c + ct - 1 < L.plan.last[b] ? c.first_c + ct - 1 : L.plan.last[b];
                it_sh = c;
            }
            red_ov = 0;
            red_hit = 0;
        }
        __syncthreads();
        if (item_sh >= total) break;
        const ItemCtx it = it_sh;

        // stage the query tile
        int unsafe_q = 0;
        for (int j = tid; j < it.nt; j += K1_THREADS) {
            QRec rec = L.q[it.lo_q + j];
            sq[j] = rec;
            if (rec.flag != 0.0) unsafe_q = 1;
        }
        unsafe_q = __syncthreads_or(unsafe_q);
        int te_desc = 0;  // any adjacent pair with te decreasing?
        for (int j = tid; j + 1 < it.nt; j += K1_THREADS)
            if (sq[j + 1].te < sq[j].te) te_desc = 1;
        const bool te_sorted = !__syncthreads_or(te_desc);
        // running max of te (window lower bounds, TA_C range test) and
        // suffix min of te (TA_R range test) over the tile
        if (tid >= 32 && tid < 64) {
            double carry = INFINITY;
            for (int base = ((it.nt - 1) & ~31); base >= 0; base -= 32) {
                int j = base + lane;
                double v = j < it.nt ? sq[j].te : INFINITY;
                for (int o = 1; o < 32; o <<= 1) {
                    double t = __shfl_down_sync(0xffffffffu, v, o);
                    if (lane + o < 32) v = fmin(v, t);
                }
                v = fmin(v, carry);
                if (j < it.nt) sm[j] = v;
                carry = __shfl_sync(0xffffffffu, v, 0);
            }
        }
        // FP32 pre-filter bounds of this item relative to (O, T0) = the
        // first staged query's start: warp 2 over the candidate groups,
        // warp 3 over the staged queries
        if (launch_f32 && warp == 2) {
            const double ox = sq[0].sx, oy = sq[0].sy, oz = sq[0].sz, t0 = sq[0].ts;
            double ar = 0.0, tvr = 0.0, vr = 0.0;
            for (int64_t g = it.first_c / GB_SIZE + lane; g <= it.c_hi / GB_SIZE; g += 32) {
                const GBound gb = L.e.gb[g];
                ar = fmax(ar, fmax(fmax(fabs(gb.hi[0] - ox), fabs(ox - gb.lo[0])),
                                   fmax(fmax(fabs(gb.hi[1] - oy), fabs(oy - gb.lo[1])),
                                        fmax(fabs(gb.hi[2] - oz), fabs(oz - gb.lo[2])))));
                tvr = fmax(tvr, fmax(fabs(gb.ts_hi - t0), fabs(t0 - gb.ts_lo)) * gb.vmax);
                vr = fmax(vr, gb.vmax);
            }
            ar = warp_max(ar);
            tvr = warp_max(tvr);
            vr = warp_max(vr);
            if (lane == 0) {
                f32b[0] = ar;
                f32b[1] = tvr;
                f32b[2] = vr;
            }
        }
        if (launch_f32 && warp == 3) {
            const double ox = sq[0].sx, oy = sq[0].sy, oz = sq[0].sz, t0 = sq[0].ts;
            double aq = 0.0, tq = 0.0, eq = 0.0;
            for (int j = lane; j < it.nt; j += 32) {
                aq = fmax(aq, fmax(fabs(sq[j].sx - ox), fmax(fabs(sq[j].sy - oy), fabs(sq[j].sz - oz))));
                tq = fmax(tq, fabs(sq[j].ts - t0));
                eq = fmax(eq, sq[j].ext);
            }
            aq = warp_max(aq);
            tq = warp_max(tq);
            eq = warp_max(eq);
            if (lane == 0) {
                f32b[3] = aq;
                f32b[4] = tq;
                f32b[5] = eq;
            }
        }
        if (tid < 32) {
            double carry = -INFINITY;
            for (int base = 0; base < it.nt; base += 32) {
                int j = base + lane;
                double v = j < it.nt ? sq[j].te : -INFINITY;
                for (int o = 1; o < 32; o <<= 1) {
                    double t = __shfl_up_sync(0xffffffffu, v, o);
                    if (lane >= o) v = fmax(v, t);
                }
                v = fmax(v, carry);
                if (j < it.nt) pm[j] = v;
                carry = __shfl_sync(0xffffffffu, v, 31);
            }
        }
        __syncthreads();
        // FP32 pre-filter records; M bounds every magnitude the FP32 path
        // forms (per component), its error is <= 7 * 2^-24 M
        bool item_f32 = false;
        if (launch_f32 && !unsafe_q) {
            if (tid == 0)
                fi_sh = f32_item(sq[0].sx, sq[0].sy, sq[0].sz, sq[0].ts, f32b[0], f32b[1], f32b[2], f32b[3],
                                 f32b[4], f32b[5], cmax);
            __syncthreads();
            item_f32 = fi_sh.ok;
            if (item_f32) {
                for (int j = tid; j < it.nt; j += K1_THREADS) {
                    const QRec &q = sq[j];
                    float v[6];
                    f32_query(q.ts, q.sx, q.sy, q.sz, q.ext, q.dx, q.dy, q.dz, fi_sh, dthr, v);
                    QF32 f;
                    f.ts = v[0]; f.x = v[1]; f.y = v[2]; f.z = v[3]; f.a = v[4]; f.b = v[5];
                    f.pad0 = f.pad1 = 0.f;
                    f.ts64 = q.ts;
                    f.te64 = q.te;
                    sqf[j] = f;
                }
            }
            __syncthreads();
        }

        unsigned n_ov = 0, n_hit = 0;
        for (int s = 0; s < sub; ++s) {
            const int64_t base = it.first_c + (int64_t)s * STRIDE;
            if (base > it.c_hi) break;  // block-uniform
            const int64_t wbase = base + (int64_t)warp * 32 * K1_CPT;
            CandF r[K1_CPT];
            bool valid_any = false, unsafe_r = false;
            double wmin = INFINITY, wmax = -INFINITY, wmin_te = INFINITY, wmax_ts = -INFINITY;
#pragma unroll
            for (int k = 0; k < K1_CPT; ++k) {
                const int64_t e = wbase + (int64_t)k * 32 + lane;
                const bool valid = e <= it.c_hi;
                if (valid) {
                    r[k].ts = L.e.ts[e]; r[k].te = L.e.te[e];
                    r[k].sx = L.e.sx[e]; r[k].sy = L.e.sy[e]; r[k].sz = L.e.sz[e];
                    r[k].vx = L.e.vx[e]; r[k].vy = L.e.vy[e]; r[k].vz = L.e.vz[e];
                    r[k].ext = __dsub_rn(r[k].te, r[k].ts);
                    unsafe_r |= L.e.unsafe[e] != 0;
                    wmin = fmin(wmin, r[k].ts);
                    wmax = fmax(wmax, r[k].te);
                    wmin_te = fmin(wmin_te, r[k].te);
                    wmax_ts = fmax(wmax_ts, r[k].ts);
                } else {
                    r[k].ts = INFINITY; r[k].te = -INFINITY; r[k].ext = 1.0;
                    r[k].sx = r[k].sy = r[k].sz = 0.0;
                    r[k].vx = r[k].vy = r[k].vz = 0.0;
                }
                valid_any |= valid;
            }
            CandF32 c32[K1_CPT];
            if (item_f32) {
#pragma unroll
                for (int k = 0; k < K1_CPT; ++k) {
                    if (r[k].ts <= r[k].te) {  // valid lane
                        c32[k] = f32_cand(r[k].ts, r[k].sx, r[k].sy, r[k].sz, r[k].vx, r[k].vy, r[k].vz, fi_sh);
                    } else {  // far away: never flagged (and rejected exactly if it were)
                        c32[k].px = c32[k].py = c32[k].pz = 0x1p60f;
                        c32[k].vx = c32[k].vy = c32[k].vz = c32[k].sr = 0.f;
                    }
                }
            }
            // key of (b, e_off of the warp's candidate 0, q_off = it.q0) without the j term
            if (lane == 0) {
                k1_wctx[warp].key_base0 = make_key(L, it.b, wbase - L.plan.first[it.b], it.q0);
                k1_wctx[warp].wbase = wbase;
                const int64_t nv = it.c_hi - wbase + 1;
                k1_wctx[warp].nvalid = nv < 0 ? 0 : (nv > 32 * K1_CPT ? 32 * K1_CPT : (int)nv);
            }
            __syncwarp();
            if (L.noop) continue;
            if (!__any_sync(0xffffffffu, valid_any)) continue;
            // warp window over the staged queries and its start-time case ranges
            wmin = warp_min(wmin);
            wmax = warp_max(wmax);
            wmin_te = warp_min(wmin_te);
            wmax_ts = warp_max(wmax_ts);
            if (lane == 0) {
                k1_wctx[warp].wmin_te = wmin_te;
                k1_wctx[warp].wmax = wmax;
            }
            int jlo = 0, jhi = it.nt, ja = it.nt, jb = it.nt;
            if (!*L.q_unsorted) {
                jlo = lower_bound_pm(pm, it.nt, wmin);   // running max te >= min ts
                jhi = upper_bound_ts(sq, it.nt, wmax);   // first query starting after max te
                if (jhi < jlo) jhi = jlo;
                ja = clampi(lower_bound_ts(sq, it.nt, wmin), jlo, jhi);  // first cts >= min ts
                jb = clampi(upper_bound_ts(sq, it.nt, wmax_ts), ja, jhi); // first cts >  max ts
            } else {
                ja = jlo;
                jb = jhi;  // everything in the generic (mixed) range
            }
            const bool slow = launch_exact || unsafe_q || __any_sync(0xffffffffu, unsafe_r) || (F32 && !item_f32);
            // tb case of a whole range: every query of the TA_C range ends
            // before all candidates (running max < min te), or every query of
            // the TA_R range ends after all of them (suffix min > max te)
            const bool c_tb_r = jlo < ja && pm[ja - 1] < wmin_te;
            const bool r_tb_c = jb < jhi && sm[jb] > wmax;
            if (slow) {
                pair_run<TA_C, TB_DYN, K1_ALL, true>(sq, sqf, jlo, ja, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
                pair_run<TA_BOTH, TB_DYN, K1_ALL, true>(sq, sqf, ja, jb, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
                pair_run<TA_R, TB_DYN, K1_ALL, true>(sq, sqf, jb, jhi, r, c32, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
                continue;
            }
            if (F32)
                run_cases<K1_F32>(L, sq, sqf, it.nt, jlo, ja, jb, jhi, c_tb_r && te_sorted, r_tb_c, r, c32,
                                  wmin_te, wmax, warp, lane, n_ov, n_hit, K);
            else
                run_cases<K1_F64>(L, sq, sqf, it.nt, jlo, ja, jb, jhi, c_tb_r && te_sorted, r_tb_c, r, c32,
                                  wmin_te, wmax, warp, lane, n_ov, n_hit, K);
        }
        // per-batch counters (64-bit)
        for (int o = 16; o; o >>= 1) {
            n_ov += __shfl_xor_sync(0xffffffffu, n_ov, o);
            n_hit += __shfl_xor_sync(0xffffffffu, n_hit, o);
        }
        if (lane == 0 && (n_ov | n_hit)) {
            atomicAdd(&red_ov, (unsigned long long)n_ov);
            atomicAdd(&red_hit, (unsigned long long)n_hit);
        }
        __syncthreads();
        if (tid == 0) {
            if (red_ov) atomicAdd(&L.plan.ovl[it.b], red_ov);
            if (red_hit) atomicAdd(&L.plan.hits[it.b], red_hit);
        }
        __syncthreads();
    }
}

static size_t k1_dyn_smem() {
    return sizeof(QF32) * K1_TQ + sizeof(uint32_t) * K1_QCAP * K1_WARPS;
}

// The dynamic shared-memory limit is a per-device function attribute.
static void k1_set_attrs() {
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(done_mask.load() & bit)) {
        TSK_CUDA(cudaFuncSetAttribute(k1_pairs<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)k1_dyn_smem()));
        TSK_CUDA(cudaFuncSetAttribute(k1_pairs<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)k1_dyn_smem()));
        done_mask.fetch_or(bit);
    }
}

int k1_blocks_per_sm(bool f32) {
    k1_set_attrs();
    int n = 0;
    if (f32) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_pairs<true>, K1_THREADS, k1_dyn_smem());
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_pairs<false>, K1_THREADS, k1_dyn_smem());
    return n > 0 ? n : 1;
}

int k1_candidates_per_thread() { return K1_CPT; }

bool k1_use_f32(double d2, double db_cmax) { return d2 <= 0x1p120 && db_cmax <= 0x1p60; }

void launch_k1(const K1Launch &L, int grid, cudaStream_t st) {
    k1_set_attrs();
    if (k1_use_f32(L.d2, L.db_cmax)) k1_pairs<true><<<grid, K1_THREADS, k1_dyn_smem(), st>>>(L);
    else k1_pairs<false><<<grid, K1_THREADS, k1_dyn_smem(), st>>>(L);
    TSK_CUDA(cudaGetLastError());
}

}  // namespace tsk
