// tsk_internal.cuh — shared device layouts and helpers for libtrajseek.
//
// Arithmetic contract: every floating-point step of the pair evaluation is
// one IEEE-754 binary64 operation, in the reference's order
// (/root/reference/pkg/src/trajseek/core.py:490-565).  The library is
// compiled with -fmad=false and the explicit __d*_rn intrinsics below are
// used on the hot path so that no multiply-add is contracted.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <memory>
#include <vector>

#include "../../include/trajseek.h"

namespace tsk {

// ── error plumbing ──────────────────────────────────────────────────────────

void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

struct Error {
    int code;
    std::string msg;
};

#define TSK_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (call);                                                         \
        if (_e != cudaSuccess)                                                           \
            throw ::tsk::Error{_e == cudaErrorMemoryAllocation ? TSK_ENOMEM : TSK_ECUDA, \
                               std::string(#call) + ": " + cudaGetErrorString(_e)};      \
    } while (0)

#define TSK_REQUIRE(cond, msg)                                \
    do {                                                      \
        if (!(cond)) throw ::tsk::Error{TSK_EINVAL, (msg)};   \
    } while (0)

// ── device buffers ──────────────────────────────────────────────────────────

// Grow-only device buffer (stream-ordered allocations on the db's stream).
struct DBuf {
    void *p = nullptr;
    size_t bytes = 0;
    template <class T>
    T *as() const { return static_cast<T *>(p); }
    void reserve(size_t need, cudaStream_t s);
    void release(cudaStream_t s);
};

// Entry (or query) segments in device SoA form.  Hoisted invariants:
//   dx,dy,dz = xe-xs, ye-ys, ze-zs  (the (e - s) of core.py:512)
//   rcp      = RN(1/(te-ts)) for te > ts, else 0 (waypoint)
//   vx,vy,vz = RN(d * rcp)  (velocity, K1's filter; filter.cuh)
//   unsafe   = 1 when the segment is outside the exponent window in which
//              qdiv below is exact and the filter's error bound holds
//              (seg_unsafe in db.cu); such tiles are evaluated exactly
// Per-group bounds of GB_SIZE consecutive (start-sorted) segments: the
// magnitudes K1's FP32 pre-filter needs for its per-item error bound
// (k1_pairs.cu, "FP32 pre-filter").
constexpr int GB_SIZE = 256;
struct GBound {
    double lo[3], hi[3];  // bounding box of the start positions
    double ts_lo, ts_hi;  // start-time range
    double vmax;          // max |velocity component|
    double pad;
};

struct Soa {
    int64_t n = 0;
    GBound *gb = nullptr;  // (n + GB_SIZE - 1) / GB_SIZE groups (entry stores only)
    double *ts = nullptr, *te = nullptr, *sx = nullptr, *sy = nullptr, *sz = nullptr;
    double *ex = nullptr, *ey = nullptr, *ez = nullptr;
    double *dx = nullptr, *dy = nullptr, *dz = nullptr, *rcp = nullptr;
    double *vx = nullptr, *vy = nullptr, *vz = nullptr;
    int64_t *traj = nullptr, *seg = nullptr;
    float *sr32 = nullptr;  // FP32 pre-filter speed bound (filter.cuh f32_speed)
    uint8_t *unsafe = nullptr;
    int any_unsafe = 0;
    int sorted = 1;     // ts non-decreasing
    int te_sorted = 1;  // te non-decreasing too (external overlap counts, count_overlaps_ext)
    DBuf storage;
};

// Query record staged in shared memory: 8 × 16 B, laid out for 16-byte
// shared loads.  The filter reads the first 96 B (ts..dy), the exact path
// ts..ext, dx..dz and ex..ez; RN(1/ext) is recomputed there.
struct __align__(16) QRec {
    double ts, te;
    double sx, sy;
    double sz, ext;
    double vx, vy;
    double vz, dz;
    double dx, dy;
    double ex, ey;
    double ez, flag;  // flag: 1.0 when the segment is unsafe (seg_unsafe)
};
static_assert(sizeof(QRec) == 128, "QRec layout");

// K1's copy of an indexed store: the same columns, reordered inside each
// index bin by the Morton code of the segment midpoints (alternating
// direction bin by bin), so that 128 consecutive entries — one warp's
// candidates — lie close together in space as well as in time.  A batch's
// candidate range is a union of whole bins (index.py:160-173), so it is the
// same contiguous ordinal range in both orders; `orig` maps a K1 position
// back to its start-sorted ordinal (hit keys, and so the reference's item
// order, use that).  `box` holds per BOX_GROUP entries the bounding box of
// their segments, rounded outward to FP32 (lo.xyz, hi.xyz): K1 skips every
// (query, warp) pair whose boxes are farther apart than the threshold.
constexpr int BOX_GROUP = 128;
struct K1Layout {
    Soa s;
    int64_t *orig = nullptr;
    float4 *box = nullptr;  // 2 per group: (lo.x, lo.y, lo.z, 0), (hi.x, hi.y, hi.z, 0)
    double2 *gtime = nullptr;  // per group: (min ts, max te)
    // FP32 pre-filter records, 2 float4 per entry: (pgx, pgy, pgz, sr),
    // (vx, vy, vz, 0), relative to the group origin gorig = (O_g, T_g), the
    // start of the group's first entry (filter.cuh f32_cand_rebase)
    float4 *frec = nullptr;
    double4 *gorig = nullptr;
    int64_t ngroups = 0;
    DBuf aux;
    bool built = false;
};

struct Index {
    int64_t m = 0, n_ne = 0;
    int rule = 0;
    double width = 0, t0 = 0, t_max = 0;
    double *ne_start = nullptr, *ne_end = nullptr, *ne_endmax = nullptr;
    int64_t *ne_first = nullptr, *ne_last = nullptr, *ne_bin = nullptr;
    DBuf storage;
    bool built = false;
};

}  // namespace tsk

// The opaque handles of the C-ABI.
struct tsk_db {
    int device = 0;
    cudaStream_t stream = nullptr;
    tsk::Soa s;
    double cmax = 0;  // max |coordinate| of the entry store
    tsk::Index ix;
    tsk::K1Layout k;  // spatially ordered copy for K1 (built with the index)
    // search workspace (grow-only)
    tsk::DBuf q_rec, batches, counters, recs, sorted, cub_tmp, out_cols, canon_cols, canon_tmp;
    tsk::DBuf pipe;         // per-chunk item tables of the pipelined search
    int64_t last_hits = 0;  // hits of the previous search (sizes the pipeline's host block)
    double last_k1_ms = 0;  // and its K1 time (chooses the pipeline's chunk count)
    int ids32 = 0;          // every entry id fits in int32 (4-byte ids over PCIe)
    tsk::Soa q;  // device copy of the current query set
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_k0 = nullptr, ev_k1 = nullptr;
    cudaStream_t stream2 = nullptr;  // result copies of the compact pipeline
    // caller-owned host copies of the entry id columns (tsk_db_set_host_ids):
    // the compact result path expands ids from ordinals on the host
    const int64_t *host_etraj = nullptr, *host_eseg = nullptr;
};

struct tsk_result {
    int64_t n = 0, nb = 0;
    double device_ms = 0, k1_ms = 0;
    int64_t k1_evals = 0;  // pairs K1's FP32 pre-filter evaluated (last attempt)
    int64_t launches = 0;
    int64_t *pb_host = nullptr;      // pinned nb × 4 (first[], last[], ovl[], hits[])
    size_t pb_bytes = 0;
    void *host = nullptr;            // pinned block holding the columns
    size_t host_bytes = 0;
    int64_t *qtraj = nullptr, *qseg = nullptr, *etraj = nullptr, *eseg = nullptr;
    double *tbeg = nullptr, *tend = nullptr;
    int64_t *qord = nullptr, *eord = nullptr;
};

namespace tsk {

// ── exact arithmetic helpers ────────────────────────────────────────────────

// RN(a/b) from y = RN(1/b) with two residual corrections (Markstein).
// q1 = RN(q0 + r0*y) is within one ulp of a/b; the second correction then
// returns the correctly rounded quotient (Markstein's theorem, y within
// half an ulp of 1/b, q1 faithful).  Residuals r = a - b*q are exact in FMA
// for faithful q as long as nothing underflows; mark_unsafe() routes inputs
// that could underflow/overflow to IEEE division instead.
__device__ __forceinline__ double qdiv(double a, double b, double y) {
    double q = __dmul_rn(a, y);
    double r = __fma_rn(-b, q, a);
    q = __fma_rn(r, y, q);
    r = __fma_rn(-b, q, a);
    return __fma_rn(r, y, q);
}

// numpy float64 floor_divide (npy_divmod) — used for bin assignment at
// index.py:110.  fmod is exact in CUDA; the rest mirrors numpy's steps.
__device__ __forceinline__ double np_floor_divide(double a, double b) {
    if (b == 0.0) return __ddiv_rn(a, b);
    double mod = fmod(a, b);
    double div = __ddiv_rn(__dsub_rn(a, mod), b);
    if (mod != 0.0) {
        if ((b < 0.0) != (mod < 0.0)) {
            mod = __dadd_rn(mod, b);
            div = __dsub_rn(div, 1.0);
        }
    }
    double fl;
    if (div != 0.0) {
        fl = floor(div);
        if (__dsub_rn(div, fl) > 0.5) fl = __dadd_rn(fl, 1.0);
    } else {
        fl = copysign(0.0, __ddiv_rn(a, b));
    }
    return fl;
}

// bin of a start time: min(floor_divide(ts - t0, width), m - 1) (index.py:108-112)
__device__ __forceinline__ int64_t bin_of(double t, double t0, double width, int64_t m) {
    if (!(width > 0.0)) return 0;
    double f = np_floor_divide(__dsub_rn(t, t0), width);
    double mm = (double)(m - 1);
    f = f < mm ? f : mm;  // np.minimum(float, m - 1)
    return (int64_t)f;
}

// ── host-side launchers (defined in the .cu files) ─────────────────────────

void soa_alloc(Soa &s, int64_t n, bool with_ids, cudaStream_t st);
void soa_upload(Soa &s, const tsk_columns *c, cudaStream_t st);
void soa_hoist(Soa &s, cudaStream_t st);  // dx/dy/dz, rcp, unsafe, sorted

struct SearchPlanDev {
    int64_t nb;
    const int64_t *lo, *hi;        // device
    int64_t *first, *last;         // device (filled by K3 or given)
    int64_t *item_off;             // nb + 1
    int64_t *meta;                 // [0]=total items, [1]=sub tiles, [2..] scratch
    unsigned long long *ovl, *hits;  // per batch
};

// Work units of a plan (k_plan_items / K1), in the plan's sharing mode
// (meta[3]).
//  * Pairs (and no sharing): batches are taken in pairs (2k, 2k+1); unit
//    5k+0 is the candidate range the pair shares, evaluated against both
//    batches' queries in one tile (when they fit), units 5k+1/5k+2 are batch
//    2k's candidates left/right of it and 5k+3/5k+4 batch 2k+1's.  A pair
//    that cannot share (a batch without candidates, disjoint ranges, queries
//    beyond one tile, batches not adjacent in the query order, or sharing
//    off) leaves unit 5k+0 empty and puts each batch's whole range in its
//    left unit.
//  * Groups (quads, or octets in the 1,024-query kernel): batches are taken
//    in groups of G = 4 or 8, whose candidate ranges [f_g, l_g] usually
//    advance together (time-sorted queries): with f and l both
//    non-decreasing, the batches holding a candidate c are the contiguous
//    run [ga, gb] (gb: last g with f_g <= c, ga: first g with l_g >= c), so
//    the group's range splits at the sorted boundaries {f_g, l_g + 1} into
//    at most 2G - 1 segments, each evaluated once against its run's queries
//    (one tile of up to G batches): a "staircase" that visits each
//    candidate once per group.  A group that is not monotone, not adjacent
//    in the query order or too large for a tile takes one unit per batch
//    (its whole range).
// Every (candidate, query) pair of the plan is in exactly one unit.  The
// sharing mode is the group size: 0 none, 1 pairs, 4 quads, 8 octets.
constexpr int K1_SHARE_NONE = 0, K1_SHARE_PAIRS = 1, K1_SHARE_QUADS = 4, K1_SHARE_OCTETS = 8;
// most batches in one tile of this build's FP32 kernel (4; the wide build 8)
#ifndef K1_GMAX_DEF
#define K1_GMAX_DEF 4
#endif
constexpr int K1_GMAX = K1_GMAX_DEF;
constexpr int K1_UNIT_GMAX = 8;  // the item planner handles every group size

template <int GM>
struct UnitT {
    int64_t b, b1;    // first batch, second batch of a multi-batch unit (else -1)
    int64_t lo_q, s;  // first query ordinal and query count (all the unit's batches)
    int64_t js;       // tile offset of the second batch's queries (s when single)
    int64_t jx[GM - 2];  // ... of the third to the last (s when absent)
    int64_t f, l;     // candidate segment (empty when f > l)
};

template <int GM>
__host__ __device__ __forceinline__ void unit_offsets(UnitT<GM> &U, int64_t v) {
    U.js = v;
#pragma unroll
    for (int i = 0; i < GM - 2; ++i) U.jx[i] = v;
}

__host__ __device__ __forceinline__ int64_t plan_units_mode(int64_t nb, int mode) {
    return mode >= K1_SHARE_QUADS ? (2 * mode - 1) * ((nb + mode - 1) / mode) : 5 * ((nb + 1) / 2);
}
// the most any mode needs (buffer sizing)
__host__ __device__ __forceinline__ int64_t plan_units(int64_t nb) {
    const int64_t a = plan_units_mode(nb, K1_SHARE_PAIRS), b = plan_units_mode(nb, K1_SHARE_QUADS),
                  c = plan_units_mode(nb, K1_SHARE_OCTETS);
    return a > b ? (a > c ? a : c) : (b > c ? b : c);
}

// (GM: the array bound, >= the group size G)
template <int GM>
__host__ __device__ __forceinline__ UnitT<GM> plan_unit_group(const SearchPlanDev &p, int64_t u, int64_t tqs, int G) {
    const int64_t k = u / (2 * G - 1), kind = u % (2 * G - 1);
    const int64_t b0 = G * k;
    const int gc = (int)(p.nb - b0 < G ? p.nb - b0 : G);
    int64_t f[GM], l[GM], sg[GM];
    bool mono = true;
    int64_t stot = 0;
    for (int g = 0; g < gc; ++g) {
        const int64_t b = b0 + g;
        f[g] = p.first[b];
        l[g] = p.last[b];
        sg[g] = p.hi[b] - p.lo[b] + 1;
        stot += sg[g];
        mono = mono && f[g] >= 0 &&
               (g == 0 || (f[g] >= f[g - 1] && l[g] >= l[g - 1] && p.lo[b] == p.hi[b - 1] + 1));
    }
    mono = mono && stot <= tqs;
    UnitT<GM> U;
    U.b1 = -1;
    U.f = 1;
    U.l = 0;  // empty
    if (!mono) {  // one unit per batch
        const int g = kind < gc ? (int)kind : 0;
        U.b = b0 + g;
        U.lo_q = p.lo[U.b];
        U.s = sg[g];
        unit_offsets(U, sg[g]);
        if (kind < gc && f[g] >= 0) {
            U.f = f[g];
            U.l = l[g];
        }
        return U;
    }
    // sorted segment boundaries {f_g, l_g + 1}
    int64_t bd[2 * GM];
    int nbd = 0;
    for (int g = 0; g < gc; ++g) {
        bd[nbd++] = f[g];
        bd[nbd++] = l[g] + 1;
    }
    for (int i = 1; i < nbd; ++i)
        for (int j = i; j > 0 && bd[j - 1] > bd[j]; --j) {
            const int64_t t = bd[j];
            bd[j] = bd[j - 1];
            bd[j - 1] = t;
        }
    U.b = b0;
    U.lo_q = p.lo[b0];
    U.s = sg[0];
    unit_offsets(U, sg[0]);
    if (kind + 1 >= nbd) return U;
    const int64_t c0 = bd[kind], c1 = bd[kind + 1] - 1;
    if (c0 > c1) return U;
    int ga = gc, gb = -1;  // the run of batches holding the segment
    for (int g = 0; g < gc; ++g) {
        if (f[g] <= c0) gb = g;
        if (ga == gc && l[g] >= c0) ga = g;
    }
    if (ga > gb) return U;  // a gap no batch covers
    U.b = b0 + ga;
    U.lo_q = p.lo[U.b];
    U.s = 0;
    for (int g = ga; g <= gb; ++g) U.s += sg[g];
    unit_offsets(U, U.s);
    if (gb > ga) {
        U.b1 = U.b + 1;
        int64_t acc = sg[ga];
        U.js = acc;
#pragma unroll
        for (int i = 0; i < GM - 2; ++i)  // (constant indices keep U in registers)
            if (ga + 2 + i <= gb) {
                acc += sg[ga + 1 + i];
                U.jx[i] = acc;
            }
    }
    U.f = c0;
    U.l = c1;
    return U;
}

// (FIXED: the group size is GM — a kernel build decodes only its own
// groups; the item planner passes the mode's)
template <int GM, bool FIXED = true>
__host__ __device__ __forceinline__ UnitT<GM> plan_unit(const SearchPlanDev &p, int64_t u, int64_t tqs, int mode) {
    if (mode >= K1_SHARE_QUADS) return plan_unit_group<GM>(p, u, tqs, FIXED ? GM : (mode < GM ? mode : GM));
    const int pair = mode != K1_SHARE_NONE;
    const int64_t k = u / 5, kind = u % 5;
    const int64_t b0 = 2 * k, b1 = 2 * k + 1;
    const bool has1 = b1 < p.nb;
    const int64_t f0 = p.first[b0], l0 = p.last[b0];
    const int64_t f1 = has1 ? p.first[b1] : -1, l1 = has1 ? p.last[b1] : -1;
    const int64_t s0 = p.hi[b0] - p.lo[b0] + 1, s1 = has1 ? p.hi[b1] - p.lo[b1] + 1 : 0;
    const int64_t ilo = f0 > f1 ? f0 : f1, ihi = l0 < l1 ? l0 : l1;
    // (batches must be adjacent in the query order: spans-given plans may
    // hold arbitrary, even overlapping, query ranges)
    const bool shared = pair && has1 && f0 >= 0 && f1 >= 0 && s0 + s1 <= tqs && ilo <= ihi &&
                        p.lo[b1] == p.hi[b0] + 1;
    UnitT<GM> U;
    U.b1 = -1;
    U.f = 1;
    U.l = 0;  // empty
    if (kind == 0) {
        U.b = b0;
        U.lo_q = p.lo[b0];
        U.s = s0 + s1;
        unit_offsets(U, U.s);
        U.js = s0;
        if (shared) {
            U.b1 = b1;
            U.f = ilo;
            U.l = ihi;
        }
        return U;
    }
    const bool second = kind >= 3;
    if (second && !has1) {
        U.b = b0;
        U.lo_q = p.lo[b0];
        U.s = s0;
        unit_offsets(U, s0);
        return U;
    }
    const int64_t b = second ? b1 : b0;
    const int64_t f = second ? f1 : f0, l = second ? l1 : l0;
    U.b = b;
    U.lo_q = p.lo[b];
    U.s = second ? s1 : s0;
    unit_offsets(U, U.s);
    if (f < 0) return U;  // no candidates
    const bool left = kind == 1 || kind == 3;
    if (!shared) {
        if (left) {
            U.f = f;
            U.l = l;
        }
    } else if (left) {
        U.f = f;
        U.l = ilo - 1;
    } else {
        U.f = ihi + 1;
        U.l = l;
    }
    return U;
}

struct K1Launch {
    Soa e;  // by value: device pointers
    const QRec *q;
    SearchPlanDev plan;
    unsigned long long *item_counter;
    unsigned long long *hit_count;
    unsigned long long *eval_count;  // (candidate, query) pairs the FP32 pre-filter evaluated
    uint64_t *keys;
    double *tbeg, *tend;
    uint64_t cap;
    double d2;
    double db_cmax;                          // max |coordinate| of the entries
    double filter_km;                        // 2^-35 - 1 (filter.cuh), a launch value so it stays in a uniform register
    const unsigned long long *q_cmax_bits;   // max |coordinate| of the queries (device, as bits)
    int major_bits, minor_bits;  // key = b << (major+minor) | major << minor | minor
    int query_major;             // 0: (b, entry, query); 1: (b, query, entry)
    int noop;
    int overlaps_only;  // count temporal overlaps only (no geometry, no hits)
    const int *q_unsorted;  // device flag: query start times not sorted -> no windows
    // K1 layout (K1Layout): e is then k.s; orig maps positions to start-sorted
    // ordinals (nullptr: identity); gbox/cull enable the box cull
    const int64_t *orig;
    const float4 *gbox;
    const double2 *gtime;
    const float4 *frec = nullptr;  // K1 layout FP32 records (2 per entry) and group origins
    const double4 *gorig = nullptr;
    int cull;
    // overlap counts come from count_overlaps_ext (store te sorted; used
    // when the query flags say ts and te are both sorted): K1's box-cull
    // fast path then skips whole warps and counts no overlaps itself
    int ext_count;
    int wide = 0;  // launch the wide FP32 kernel (k1_f32_wide.cu: 1,024-query tiles, octets)
};

void launch_ranges(tsk_db *db, const Soa &q, SearchPlanDev &p, bool spans_given, cudaStream_t st);
void launch_plan_items(SearchPlanDev &p, int slots, int stride, int pair, int align, int tq_max, const int *q_flags,
                       cudaStream_t st);
void launch_qprep(const Soa &q, QRec *out, int *flags, unsigned long long *cmax_bits, cudaStream_t st);
bool mapped_columns(const tsk_columns *c, tsk_columns *dev);
void launch_qprep_mapped(const tsk_columns &dev_cols, Soa &q, QRec *out, int *flags, unsigned long long *cmax_bits,
                         cudaStream_t st);
double soa_cmax(const Soa &s, cudaStream_t st);
int soa_ids32(const Soa &s, cudaStream_t st);
void soa_group_bounds(Soa &s, cudaStream_t st);  // GBound per GB_SIZE segments
void launch_k1(const K1Launch &L, int grid, cudaStream_t st);
void build_k1_layout(tsk_db *db, cudaStream_t st);  // layout.cu
void launch_count_overlaps_ext(const SearchPlanDev &p, const Soa &q, const Soa &s, const int *q_flags,
                               const unsigned long long *q_cmax_bits, double db_cmax, double d2, cudaStream_t st);
void free_k1_layout(tsk_db *db);
void canonical_perm(int64_t n, const int64_t *qt, const int64_t *qs, const int64_t *et,
                    const int64_t *es, const double *tb, const double *te, uint32_t *perm,
                    DBuf &scratch, cudaStream_t st);
void permute6(int64_t n, const uint32_t *perm, const int64_t *const in_i[4], const double *const in_f[2],
              int64_t *const out_i[4], double *const out_f[2], cudaStream_t st);
int k1_blocks_per_sm(bool f32);
int k1f_blocks_per_sm();
int k1f_candidates_per_thread();
void launch_k1f(const K1Launch &L, int grid, cudaStream_t st);
// the wide build of the FP32 kernel (k1_f32_wide.cu)
inline namespace wide {
int k1f_stats_wide(unsigned long long *v, int reset);
int k1f_blocks_per_sm_wide();
void launch_k1f_wide(const K1Launch &L, int grid, cudaStream_t st);
}
#ifndef K1W_THREADS_DEF
#define K1W_THREADS_DEF 512
#endif
constexpr int K1W_THREADS = K1W_THREADS_DEF, K1W_TQ = 1024;
bool k1_use_f32(double d2, double db_cmax);
int k1_candidates_per_thread(bool f32);

// 8 warps per CTA, 2 CTAs per SM at up to 128 registers, with 512-query
// tiles (quads of Periodic batches share candidate tiles): the shared
// memory of a 512-query tile fits twice per SM at this width
#ifndef K1_THREADS_DEF
#define K1_THREADS_DEF 256
#endif
constexpr int K1_THREADS = K1_THREADS_DEF;
#ifndef K1_TQ_DEF
#define K1_TQ_DEF 512
#endif
constexpr int K1_TQ = K1_TQ_DEF;   // queries per tile of the FP32 kernel, staged in shared memory
constexpr int K1P_TQ = 256;        // queries per tile of the FP64-filter kernel (k1_pairs.cu)
#ifndef K1_MAX_SUB_DEF
#define K1_MAX_SUB_DEF 32
#endif
constexpr int K1_MAX_SUB = K1_MAX_SUB_DEF;  // candidate sub-tiles (of K1_THREADS) per item

}  // namespace tsk
