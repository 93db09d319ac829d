// k1_f32.cu — K1, the moving-distance pair kernel (GPUTrajDistSearch), with
// the FP32 pre-filter: the common path of every launch whose coordinates
// and threshold are below 2^60 (k1_pairs.cu serves the rest).
//
// Replaces core.pair_intervals (/root/reference/pkg/src/trajseek/core.py:464-565)
// driven by engine.execute_batch/_run_chunks (engine.py:78-148) for every
// batch of a plan at once.
//
// Work decomposition.  A work item is (work unit: one batch, an adjacent
// pair sharing candidates, or a staircase segment of a group of 4 or 8
// batches (tsk_internal.cuh), candidate tile, query tile),
// claimed from a global counter by a persistent grid.  The query tile is
// staged in shared memory as 48-byte FP32 pre-filter records (filter.cuh)
// with the exact start/end times; each lane holds K1F_CPT = 4 candidates
// (lanes l, l+32, l+64, l+96 of the warp's 128 consecutive entries) in FP32
// pre-filter form, and each warp loops over the window of staged queries
// that can overlap any of its candidates (entries and queries are both
// start-time sorted: on tiles whose end times ascend too, the window is the
// min / max of the candidates' own overlap bounds, all found together by
// binary lifting; else four binary searches, one per lane).
//
// Per (candidate, query): 9 FP32 ops decide "cannot hit" for nearly every
// pair (f32_flag, with a proven error margin; issued as FFMA2 / FADD2 /
// FMUL2 on a lane's candidates in pairs, 4.5 instructions per pair, with the
// query's values as the broadcast operand), one NaN-propagating min over
// the lane's four norms and one compare per (query, lane), two queries per
// loop iteration with one vote (f32_scan2; f32_scan where overlaps are
// counted per pair); flagged pairs are queued per warp and re-evaluated 32 at a time with the
// reference's exact binary64 arithmetic (k1_exact.cuh), which is what makes
// the result set bit-exact.  Overlaps are counted exactly: by bisection for
// whole ranges, else with binary64 compares of the exact times.
#include <atomic>

#include "k1_exact.cuh"

// The library builds this file twice: as is (512-query tiles, 8-warp CTAs,
// two per SM) and from k1_f32_wide.cu (K1_WIDE: 1,024-query tiles, 16-warp
// CTAs, one per SM, octets of batches); the wide build's host-visible names
// carry a suffix and its device code lives in tsk::wide.
#ifdef K1_WIDE
#define K1F_NAME(x) x##_wide
#define K1F_NS_OPEN inline namespace wide {
#define K1F_NS_CLOSE }
#else
#define K1F_NAME(x) x
#define K1F_NS_OPEN
#define K1F_NS_CLOSE
#endif

#ifndef K1F_CPT
#define K1F_CPT 4
#endif
#ifndef K1F_MIN_BLOCKS
#define K1F_MIN_BLOCKS 2
#endif

namespace tsk {
K1F_NS_OPEN

// Development counters (built with -DTSK_K1_STATS only; read by
// tsk_k1_stats): 0 box-cull sub-tiles, 1 box tests, 2 box survivors,
// 3 sub-tiles with survivors, 4 pre-filter flags, 5 separating-axis
// survivors, 6 exact-path flushes, 7 items.
__device__ unsigned long long K1F_NAME(k1_stats)[8];
#ifdef TSK_K1_STATS
#define K1_STAT(i, v) \
    do { if ((threadIdx.x & 31) == 0) atomicAdd(&K1F_NAME(k1_stats)[i], (unsigned long long)(v)); } while (0)
#else
#define K1_STAT(i, v) do { } while (0)
#endif

constexpr int CPT = K1F_CPT;
constexpr int WCAND = 32 * CPT;         // candidates per warp
constexpr int QCAP = 32 * (CPT + 1);    // queue entries per warp
static_assert(WCAND <= 65536, "candidate index must fit the 16-bit queue field");

// Dynamic shared memory: FP32 query records | per-warp queues | per-warp
// FP32 candidates (structure of arrays, 7 x WCAND floats per warp).
extern __shared__ __align__(16) unsigned char k1_dyn[];
__device__ __forceinline__ QF32 *f_sqf() { return reinterpret_cast<QF32 *>(k1_dyn); }
__device__ __forceinline__ uint32_t *f_queue(int warp) {
    return reinterpret_cast<uint32_t *>(k1_dyn + sizeof(QF32) * K1_TQ) + warp * QCAP;
}
__device__ __forceinline__ float *f_cands(int warp) {
    return reinterpret_cast<float *>(k1_dyn + sizeof(QF32) * K1_TQ + sizeof(uint32_t) * QCAP * K1_WARPS) +
           warp * 7 * WCAND;
}
// query boxes (2 float4 per staged query: lo, hi of its segment, FP32 outward)
constexpr size_t QBOX_OFF = sizeof(QF32) * K1_TQ + sizeof(uint32_t) * QCAP * K1_WARPS + sizeof(float) * 7 * WCAND * K1_WARPS;
__device__ __forceinline__ float4 *f_qbox() { return reinterpret_cast<float4 *>(k1_dyn + QBOX_OFF); }
// per-warp list of the window's queries that survive the box cull
__device__ __forceinline__ uint16_t *f_wlist(int warp) {
    return reinterpret_cast<uint16_t *>(k1_dyn + QBOX_OFF + 2 * sizeof(float4) * K1_TQ) + warp * K1_TQ;
}
// per-warp queue of the pairs that pass the separating-axis stage (< 64)
constexpr int Q2CAP = 64;
constexpr size_t Q2_OFF = QBOX_OFF + 2 * sizeof(float4) * K1_TQ + sizeof(uint16_t) * K1_TQ * K1_WARPS;
__device__ __forceinline__ uint32_t *f_queue2(int warp) {
    return reinterpret_cast<uint32_t *>(k1_dyn + Q2_OFF) + warp * Q2CAP;
}
__shared__ float k1_sep_rb;  // the item's separating-axis radius term (f32_sep_rbase)

__device__ __forceinline__ void lds4f(uint32_t a, float &x, float &y, float &z, float &w) {
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a));
}
__device__ __forceinline__ void lds2d(uint32_t a, double &x, double &y) {
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}

// The inner loop, a leaf function (no calls inside, so it gets the register
// file to itself): loads the warp's FP32 candidates, scans queries from qa
// until 32 or more flags are queued or the range ends, and returns
// (qa, queued, overlaps).  The caller flushes and resumes.  CNT: count
// overlaps per pair with the exact times (read from L2 once per call).
// The warp's staged FP32 candidates of this lane, packed in pairs (2h, 2h+1).
__device__ __forceinline__ void load_cands_x2(const float *cs, int lane, CandF32x2 (&c)[CPT / 2]) {
#pragma unroll
    for (int h = 0; h < CPT / 2; ++h) {
        const int i0 = (2 * h) * 32 + lane, i1 = i0 + 32;
        c[h].px = make_float2(cs[0 * WCAND + i0], cs[0 * WCAND + i1]);
        c[h].py = make_float2(cs[1 * WCAND + i0], cs[1 * WCAND + i1]);
        c[h].pz = make_float2(cs[2 * WCAND + i0], cs[2 * WCAND + i1]);
        c[h].vx = make_float2(cs[3 * WCAND + i0], cs[3 * WCAND + i1]);
        c[h].vy = make_float2(cs[4 * WCAND + i0], cs[4 * WCAND + i1]);
        c[h].vz = make_float2(cs[5 * WCAND + i0], cs[5 * WCAND + i1]);
    }
}

// The lane's four norms |u|^2 against one query, two FFMA2 chains.
__device__ __forceinline__ void norms_x2(const CandF32x2 (&c)[CPT / 2], float ts, float x, float y, float z,
                                         float (&n)[CPT]) {
#pragma unroll
    for (int h = 0; h < CPT / 2; ++h) {
        const float2 a = f32_n2x2(c[h], ts, x, y, z);
        n[2 * h] = a.x;
        n[2 * h + 1] = a.y;
    }
}

template <int TA, bool CNT>
__device__ __noinline__ uint4 f32_scan(uint32_t qa, uint32_t qa_end, uint32_t base, int qn, int warp, int lane) {
    static_assert(CPT % 2 == 0, "candidates are packed in pairs");
    uint32_t *const wq = f_queue(warp);
    const float *cs = f_cands(warp);
    CandF32x2 c[CPT / 2];
    load_cands_x2(cs, lane, c);
    // one threshold per query and lane: the largest speed bound of the lane's
    // candidates (staged per candidate, reduced here)
    float srl = 0.f;
#pragma unroll
    for (int k = 0; k < CPT; ++k) srl = fmaxf(srl, cs[6 * WCAND + k * 32 + lane]);
    double rts[CPT], rte[CPT];
    if (CNT) {
        const int64_t wb = k1_wctx[warp].wbase;
        const int nv = k1_wctx[warp].nvalid, nlo = k1_wctx[warp].nlo;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int i = k * 32 + lane;
            const bool valid = i >= nlo && i < nv;  // (a K1-layout tile's head below c_lo is another unit's)
            rts[k] = valid ? k1_fcfg.ts[wb + i] : INFINITY;   // invalid lanes never overlap
            rte[k] = valid ? k1_fcfg.te[wb + i] : -INFINITY;
        }
    }
    unsigned long long n_ov = 0;
    const uint32_t qa_js = base + (uint32_t)k1_wctx[warp].js * (uint32_t)sizeof(QF32);  // b1's first query
    for (; qa < qa_end; qa += (uint32_t)sizeof(QF32)) {
        float qts, qx, qy, qz, qa4, qb4, p0, p1;
        lds4f(qa, qts, qx, qy, qz);
        lds4f(qa + 16, qa4, qb4, p0, p1);
        double cts = 0.0, cte = 0.0;
        if (CNT) lds2d(qa + (uint32_t)offsetof(QF32, ts64), cts, cte);
        bool cand[CPT];
        const float R2 = f32_r2(qa4, srl, qb4);
        float n2[CPT];
        norms_x2(c, qts, qx, qy, qz, n2);
        if constexpr (CNT) {
            bool any = false;
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                // TA_C: the query started first, so it overlaps iff it ends at
                // or after r.ts; TA_R: iff it starts at or before r.te
                bool ov;
                if (TA == TA_C) ov = rts[k] <= cte;
                else if (TA == TA_R) ov = cts <= rte[k];
                else ov = rts[k] <= cte && cts <= rte[k];
                n_ov += ov ? (qa >= qa_js ? CNT_B1 : 1ull) : 0ull;
                cand[k] = !f32_far(n2[k], R2) && ov;
                any |= cand[k];
            }
            if (!__any_sync(0xffffffffu, any)) continue;
        } else {
            // one compare per (query, lane) on the smallest norm; the
            // per-candidate flags only on the rare queries that pass
            float mn = n2[0];
#pragma unroll
            for (int k = 1; k < CPT; ++k) mn = f32_min_nan(mn, n2[k]);
            if (!__any_sync(0xffffffffu, !f32_far(mn, R2))) continue;
#pragma unroll
            for (int k = 0; k < CPT; ++k) cand[k] = !f32_far(n2[k], R2);
        }
        // rare: queue the flagged pairs of this query (qn < 32 on entry)
        const uint32_t j = (qa - base) / (uint32_t)sizeof(QF32);
        unsigned lt;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const unsigned m = __ballot_sync(0xffffffffu, cand[k]);
            if (cand[k]) wq[qn + __popc(m & lt)] = ((uint32_t)(k * 32 + lane) << 16) | j;
            qn += __popc(m);
        }
        if (qn >= 32) {
            qa += (uint32_t)sizeof(QF32);
            break;
        }
    }
    return make_uint4(qa, (unsigned)qn, (unsigned)(n_ov & 0xffffffffull), (unsigned)(n_ov >> 32));
}

// Flags of one query's pairs (the lane threshold R2), queued with ballots.
__device__ __forceinline__ void queue_query(uint32_t *wq, const float (&n2)[CPT], float R2, uint32_t j, int lane,
                                            int &qn) {
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const bool cand = !f32_far(n2[k], R2);
        const unsigned m = __ballot_sync(0xffffffffu, cand);
        if (cand) wq[qn + __popc(m & lt)] = ((uint32_t)(k * 32 + lane) << 16) | j;
        qn += __popc(m);
    }
}

// f32_scan without per-pair overlap counting, two queries per iteration:
// one vote for both (the second may lie one record past the range end: it
// is read but never queued).
template <int TA>
__device__ __noinline__ uint4 f32_scan2(uint32_t qa, uint32_t qa_end, uint32_t base, int qn, int warp, int lane) {
    static_assert(CPT % 2 == 0, "candidates are packed in pairs");
    uint32_t *const wq = f_queue(warp);
    const float *cs = f_cands(warp);
    // candidates (2h, 2h+1) of the lane packed in one CandF32x2
    CandF32x2 c[CPT / 2];
    load_cands_x2(cs, lane, c);
    float srl = 0.f;
#pragma unroll
    for (int k = 0; k < CPT; ++k) srl = fmaxf(srl, cs[6 * WCAND + k * 32 + lane]);
    constexpr uint32_t QB = (uint32_t)sizeof(QF32);
    for (; qa < qa_end; qa += 2 * QB) {
        float ts0, x0, y0, z0, a0, b0, ts1, x1, y1, z1, a1, b1, p0, p1;
        lds4f(qa, ts0, x0, y0, z0);
        lds4f(qa + 16, a0, b0, p0, p1);
        lds4f(qa + QB, ts1, x1, y1, z1);
        lds4f(qa + QB + 16, a1, b1, p0, p1);
        const float R0 = f32_r2(a0, srl, b0), R1 = f32_r2(a1, srl, b1);
        float n0[CPT], n1[CPT];
        norms_x2(c, ts0, x0, y0, z0, n0);
        norms_x2(c, ts1, x1, y1, z1, n1);
        float m0 = n0[0], m1 = n1[0];
#pragma unroll
        for (int k = 1; k < CPT; ++k) {
            m0 = f32_min_nan(m0, n0[k]);
            m1 = f32_min_nan(m1, n1[k]);
        }
        const bool f0 = !f32_far(m0, R0), f1 = !f32_far(m1, R1);
        if (!__any_sync(0xffffffffu, f0 || f1)) continue;
        // rare: queue each query's flags (qn < 32 on entry)
        const uint32_t j = (qa - base) / QB;
        if (__any_sync(0xffffffffu, f0)) queue_query(wq, n0, R0, j, lane, qn);
        if (qn >= 32) {  // the second query is scanned again by the next call
            qa += QB;
            break;
        }
        if (qa + QB < qa_end && __any_sync(0xffffffffu, f1)) queue_query(wq, n1, R1, j + 1, lane, qn);
        if (qn >= 32) {
            qa += 2 * QB;
            break;
        }
    }
    if (qa > qa_end) qa = qa_end;
    return make_uint4(qa, (unsigned)qn, 0u, 0u);
}

// Separating-axis stage (filter.cuh f32_sep_far) over up to 32 queued
// pairs, one per lane, converged: the pairs it cannot reject move to the
// warp's stage-2 queue, which feeds the exact path 32 at a time.  Returns
// the new stage-2 count (< 64).
__device__ __noinline__ int sep_stage(const QF32 *__restrict__ sqf, const uint32_t *wq, uint32_t *wq2, int nf,
                                      int qn2, int warp, int lane) {
    const float *cs = f_cands(warp);
    bool keep = false;
    uint32_t ent = 0u;
    if (lane < nf) {
        ent = wq[lane];
        const int ci = (int)(ent >> 16), j = (int)(ent & 0xffffu);
        const uint32_t qa = (uint32_t)__cvta_generic_to_shared(sqf + j);
        float qts, qx, qy, qz, qa4, qb4, qte, qex, qey, qez, p0, p1;
        lds4f(qa, qts, qx, qy, qz);
        lds4f(qa + 16, qa4, qb4, qte, qex);
        lds4f(qa + 32, qey, qez, p0, p1);
        keep = !f32_sep_far(cs[0 * WCAND + ci], cs[1 * WCAND + ci], cs[2 * WCAND + ci], cs[3 * WCAND + ci],
                            cs[4 * WCAND + ci], cs[5 * WCAND + ci], qts, qx, qy, qz, qte, qex, qey, qez, k1_sep_rb);
    }
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) wq2[qn2 + __popc(m & lt)] = ent;
    return qn2 + __popc(m);
}

// flush_queue with the separating-axis stage in front of the exact path:
// stage 1 (the pre-filter's flags, qn) is drained 32 at a time through
// sep_stage; the exact path runs on full batches of 32 survivors (qn2), and
// on the rest when the range is done.  All counts are warp-uniform.
template <int TA, int TB>
__device__ __forceinline__ void flush_tight(const QRec *__restrict__ qt, const QF32 *__restrict__ sqf, uint32_t *wq,
                                            int warp, int lane, int &qn, int &qn2, bool done,
                                            unsigned long long &n_hit) {
    uint32_t *const wq2 = f_queue2(warp);
    while (qn >= 32 || (done && qn > 0)) {
        const int nf = qn < 32 ? qn : 32;
        __syncwarp();
        K1_STAT(4, nf);
        const int q2_in = qn2;
        qn2 = sep_stage(sqf, wq, wq2, nf, qn2, warp, lane);
        K1_STAT(5, qn2 - q2_in);
        __syncwarp();
        uint32_t mv[CPT];
#pragma unroll
        for (int k = 0; k < CPT; ++k) mv[k] = lane + 32 * (k + 1) < qn ? wq[lane + 32 * (k + 1)] : 0u;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < CPT; ++k)
            if (lane + 32 * (k + 1) < qn) wq[lane + 32 * k] = mv[k];
        qn -= nf;
        if (qn2 >= 32) {
            __syncwarp();
            K1_STAT(6, 1);
            rare_flush<TA, TB, false>(qt, wq2, warp, 32, lane, n_hit);
            __syncwarp();
            const uint32_t m2 = lane + 32 < qn2 ? wq2[lane + 32] : 0u;
            __syncwarp();
            if (lane + 32 < qn2) wq2[lane] = m2;
            qn2 -= 32;
        }
    }
    if (done && qn2 > 0) {
        __syncwarp();
        K1_STAT(6, 1);
        rare_flush<TA, TB, false>(qt, wq2, warp, qn2, lane, n_hit);
        __syncwarp();
        qn2 = 0;
    }
}

// f32_scan2 over the warp's list of surviving queries (box cull): the same
// two-query iteration, the tile indices read from the list.  Returns
// (next list position, queued).
__device__ __noinline__ uint2 f32_scanl(int k, int ns, uint32_t base, int qn, int warp, int lane) {
    uint32_t *const wq = f_queue(warp);
    const uint16_t *const wl = f_wlist(warp);
    const float *cs = f_cands(warp);
    CandF32x2 c[CPT / 2];
    load_cands_x2(cs, lane, c);
    float srl = 0.f;
#pragma unroll
    for (int kk = 0; kk < CPT; ++kk) srl = fmaxf(srl, cs[6 * WCAND + kk * 32 + lane]);
    constexpr uint32_t QB = (uint32_t)sizeof(QF32);
    for (; k < ns; k += 2) {
        const uint32_t j0 = wl[k], j1 = k + 1 < ns ? wl[k + 1] : j0;
        const uint32_t qa0 = base + j0 * QB, qa1 = base + j1 * QB;
        float ts0, x0, y0, z0, a0, b0, ts1, x1, y1, z1, a1, b1, p0, p1;
        lds4f(qa0, ts0, x0, y0, z0);
        lds4f(qa0 + 16, a0, b0, p0, p1);
        lds4f(qa1, ts1, x1, y1, z1);
        lds4f(qa1 + 16, a1, b1, p0, p1);
        const float R0 = f32_r2(a0, srl, b0), R1 = f32_r2(a1, srl, b1);
        float n0[CPT], n1[CPT];
        norms_x2(c, ts0, x0, y0, z0, n0);
        norms_x2(c, ts1, x1, y1, z1, n1);
        float m0 = n0[0], m1 = n1[0];
#pragma unroll
        for (int kk = 1; kk < CPT; ++kk) {
            m0 = f32_min_nan(m0, n0[kk]);
            m1 = f32_min_nan(m1, n1[kk]);
        }
        const bool f0 = !f32_far(m0, R0), f1 = !f32_far(m1, R1);
        if (!__any_sync(0xffffffffu, f0 || f1)) continue;
        if (__any_sync(0xffffffffu, f0)) queue_query(wq, n0, R0, j0, lane, qn);
        if (qn >= 32) {  // the second query is scanned again by the next call
            k += 1;
            break;
        }
        if (k + 1 < ns && __any_sync(0xffffffffu, f1)) queue_query(wq, n1, R1, j1, lane, qn);
        if (qn >= 32) {
            k += 2;
            break;
        }
    }
    if (k > ns) k = ns;
    return make_uint2((unsigned)k, (unsigned)qn);
}

// Box cull of a warp's window (K1 layout): lane j tests query jlo + j + 32i
// against the bounding box of the warp's 128 candidates (the union of the
// precomputed boxes of the two BOX_GROUPs they span); survivors are listed
// in f_wlist in window order.  A pair can hit only if its two segments'
// boxes are within R = (1 + 2^-8) d + 2^-10 (D_warp + D_query) + 2^-29 C
// (filter.cuh, box_cull_*; D: box diagonals, the query's share staged in
// its box's .w): the gap is formed from boxes rounded outward and rounded
// down itself, so it never exceeds the true gap.  Returns the number of
// survivors (warp-uniform).
__device__ __forceinline__ int box_cull(float4 lo, float4 hi, int jlo, int jhi, float rbase, int warp, int lane) {
    const float rw = __fadd_ru(rbase, box_cull_dterm(lo.x, lo.y, lo.z, hi.x, hi.y, hi.z));
    const float4 *qb = f_qbox();
    uint16_t *const wl = f_wlist(warp);
    unsigned lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    int ns = 0;
    // two queries per lane per iteration (j and j + 32), packed; survivors
    // keep window order (the first 32's ballot, then the second's)
    for (int jb = jlo; jb < jhi; jb += 64) {
        const int j0 = jb + lane, j1 = j0 + 32;
        const int c0 = j0 < jhi ? j0 : jhi - 1, c1 = j1 < jhi ? j1 : jhi - 1;  // clamped reads
        const float4 l0 = qb[2 * c0], h0 = qb[2 * c0 + 1], l1 = qb[2 * c1], h1 = qb[2 * c1 + 1];
        const float2 g2 = box_gap2_x2(lo.x, lo.y, lo.z, hi.x, hi.y, hi.z, make_float2(l0.x, l1.x),
                                      make_float2(l0.y, l1.y), make_float2(l0.z, l1.z), make_float2(h0.x, h1.x),
                                      make_float2(h0.y, h1.y), make_float2(h0.z, h1.z));
        const float2 R = __fadd2_ru(make_float2(rw, rw), make_float2(l0.w, l1.w));
        const float2 R2 = __fmul2_ru(R, R);
        const bool p0 = j0 < jhi && !(g2.x > R2.x), p1 = j1 < jhi && !(g2.y > R2.y);
        const unsigned m0 = __ballot_sync(0xffffffffu, p0);
        if (p0) wl[ns + __popc(m0 & lt)] = (uint16_t)j0;
        ns += __popc(m0);
        const unsigned m1 = __ballot_sync(0xffffffffu, p1);
        if (p1) wl[ns + __popc(m1 & lt)] = (uint16_t)j1;
        ns += __popc(m1);
    }
    __syncwarp();
    return ns;
}

// The scan over the survivors: scan, flush 32 at a time, resume (the
// single-scan window's cases, TA_BOTH / TB_DYN).
__device__ __forceinline__ void f32_list_range(const QRec *__restrict__ qt, const QF32 *__restrict__ sqf, int ns,
                                               int warp, int lane, unsigned long long &n_hit) {
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sqf);
    uint32_t *const wq = f_queue(warp);
    int k = 0, qn = 0, qn2 = 0;
    for (;;) {
        const uint2 o = f32_scanl(k, ns, base, qn, warp, lane);
        k = (int)o.x;
        qn = (int)o.y;
        const bool done = k >= ns;
        flush_tight<TA_BOTH, TB_DYN>(qt, sqf, wq, warp, lane, qn, qn2, done, n_hit);
        if (done) break;
    }
}

// One (TA, TB) range of the window: scan, flush 32 at a time, resume.
template <int TA, int TB, bool CNT>
__device__ __forceinline__ void f32_range(const QRec *__restrict__ qt, const QF32 *__restrict__ sqf, int j0,
                                          int j1, int warp, int lane, unsigned long long &n_ov,
                                          unsigned long long &n_hit) {
    if (j0 >= j1) return;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sqf);
    uint32_t qa = base + (uint32_t)j0 * (uint32_t)sizeof(QF32);
    const uint32_t qa_end = base + (uint32_t)j1 * (uint32_t)sizeof(QF32);
    uint32_t *const wq = f_queue(warp);
    int qn = 0, qn2 = 0;
    for (;;) {
        const uint4 o = CNT ? f32_scan<TA, CNT>(qa, qa_end, base, qn, warp, lane)
                            : f32_scan2<TA>(qa, qa_end, base, qn, warp, lane);
        qa = o.x;
        qn = (int)o.y;
        n_ov += (unsigned long long)o.z + (unsigned long long)o.w * CNT_B1;
        const bool done = qa >= qa_end;
        flush_tight<TA, TB>(qt, sqf, wq, warp, lane, qn, qn2, done, n_hit);
        if (done) break;
    }
}

// Exact path for a whole window (extreme-exponent tiles, items outside the
// pre-filter's validity): every overlapping pair is queued.
template <int TA>
__device__ __forceinline__ void all_range(const QRec *__restrict__ qt, const QF32 *__restrict__ sqf, int j0, int j1,
                                          const double (&rts)[CPT], const double (&rte)[CPT], int warp, int lane,
                                          unsigned long long &n_ov, unsigned long long &n_hit) {
    uint32_t *const wq = f_queue(warp);
    int qn = 0;
    const int js = k1_wctx[warp].js;
    for (int j = j0; j < j1; ++j) {
        const double cts = sqf[j].ts64, cte = sqf[j].te64;
        const unsigned long long inc = j >= js ? CNT_B1 : 1ull;
        bool cand[CPT];
        bool any = false;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            cand[k] = rts[k] <= cte && cts <= rte[k];
            n_ov += cand[k] ? inc : 0ull;
            any |= cand[k];
        }
        if (__any_sync(0xffffffffu, any)) {
            unsigned lt;
            asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                const unsigned m = __ballot_sync(0xffffffffu, cand[k]);
                if (cand[k]) wq[qn + __popc(m & lt)] = ((uint32_t)(k * 32 + lane) << 16) | (uint32_t)j;
                qn += __popc(m);
            }
        }
        flush_queue<TA, TB_DYN, true, CPT>(qt, wq, warp, lane, qn, j + 1 == j1, n_hit);
    }
}

// The warp's candidates in FP32 pre-filter form, staged in shared memory
// (structure of arrays, lane-interleaved); invalid lanes are far away (and
// rejected exactly if ever flagged).
__device__ __forceinline__ void stage_cands(const K1Launch &L, int64_t wbase, int64_t c_lo, int64_t c_hi,
                                            const double (&rts)[CPT],
                                            const F32Item &fi, float *wcs, int lane) {
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int i = k * 32 + lane;
        const int64_t e = wbase + i;
        CandF32 c;
        c.px = c.py = c.pz = 0x1p60f;
        c.vx = c.vy = c.vz = c.sr = 0.f;
        if (e >= c_lo && e <= c_hi)
            c = f32_cand_sr(rts[k], L.e.sx[e], L.e.sy[e], L.e.sz[e], L.e.vx[e], L.e.vy[e], L.e.vz[e], L.e.sr32[e], fi);
        wcs[0 * WCAND + i] = c.px; wcs[1 * WCAND + i] = c.py; wcs[2 * WCAND + i] = c.pz;
        wcs[3 * WCAND + i] = c.vx; wcs[4 * WCAND + i] = c.vy; wcs[5 * WCAND + i] = c.vz;
        wcs[6 * WCAND + i] = c.sr;
    }
}

// The bounding box of a warp's 128 candidates (K1 layout: the union of the
// boxes of the BOX_GROUPs it spans) and whether a segment in it is unsafe
// (.w of the low corners).
__device__ __forceinline__ void warp_box(const K1Launch &L, int64_t wbase, int64_t c_hi, float4 &lo, float4 &hi,
                                         bool &unsafe) {
    const int64_t g0 = wbase / BOX_GROUP;
    const int64_t g1 = (wbase + WCAND - 1 < c_hi ? wbase + WCAND - 1 : c_hi) / BOX_GROUP;
    lo = L.gbox[2 * g0];
    hi = L.gbox[2 * g0 + 1];
    unsafe = lo.w != 0.f;
    if (g1 != g0) {
        const float4 l1 = L.gbox[2 * g1], h1 = L.gbox[2 * g1 + 1];
        unsafe |= l1.w != 0.f;
        lo = make_float4(fminf(lo.x, l1.x), fminf(lo.y, l1.y), fminf(lo.z, l1.z), 0.f);
        hi = make_float4(fmaxf(hi.x, h1.x), fmaxf(hi.y, h1.y), fmaxf(hi.z, h1.z), 0.f);
    }
}

// Two of a lane's candidates (k0, k0 + 1): their raw columns in registers
// (every global load issued before any use), then their FP32 pre-filter
// form staged in shared memory; lanes past the item's range stage a
// far-away point.
struct RawPair {
    double ts[2], sx[2], sy[2], sz[2], vx[2], vy[2], vz[2];
    float sr[2];
    bool ok[2];
};

__device__ __forceinline__ void load_pair(const K1Launch &L, int64_t wbase, int64_t c_lo, int64_t c_hi, int k0,
                                          int lane, RawPair &r) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int64_t e = wbase + (k0 + h) * 32 + lane;
        r.ok[h] = e >= c_lo && e <= c_hi;
        const int64_t ec = r.ok[h] ? e : c_lo;  // loads stay unconditional
        r.ts[h] = L.e.ts[ec];
        r.sx[h] = L.e.sx[ec]; r.sy[h] = L.e.sy[ec]; r.sz[h] = L.e.sz[ec];
        r.vx[h] = L.e.vx[ec]; r.vy[h] = L.e.vy[ec]; r.vz[h] = L.e.vz[ec];
        r.sr[h] = L.e.sr32[ec];
    }
}

__device__ __forceinline__ void store_pair(const RawPair &r, int k0, const F32Item &fi, float *wcs, int lane) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int i = (k0 + h) * 32 + lane;
        CandF32 c;
        c.px = c.py = c.pz = 0x1p60f;
        c.vx = c.vy = c.vz = c.sr = 0.f;
        if (r.ok[h]) c = f32_cand_sr(r.ts[h], r.sx[h], r.sy[h], r.sz[h], r.vx[h], r.vy[h], r.vz[h], r.sr[h], fi);
        wcs[0 * WCAND + i] = c.px; wcs[1 * WCAND + i] = c.py; wcs[2 * WCAND + i] = c.pz;
        wcs[3 * WCAND + i] = c.vx; wcs[4 * WCAND + i] = c.vy; wcs[5 * WCAND + i] = c.vz;
        wcs[6 * WCAND + i] = c.sr;
    }
}

// The warp's candidates from the K1 layout's FP32 records (one group: the
// fast path's sub-tiles are BOX_GROUP-aligned), re-based to the item's
// origin (filter.cuh f32_cand_rebase): two 16-byte loads per candidate.
__device__ __forceinline__ void stage_rebased(const K1Launch &L, int64_t wbase, int64_t c_lo, int64_t c_hi,
                                              const F32Item &fi, float *wcs, int lane) {
    const double4 go = L.gorig[wbase / BOX_GROUP];
    float4 a[CPT], b[CPT];
    bool ok[CPT];
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int64_t e = wbase + k * 32 + lane;
        ok[k] = e >= c_lo && e <= c_hi;
        const int64_t ec = ok[k] ? e : c_lo;
        a[k] = L.frec[2 * ec];
        b[k] = L.frec[2 * ec + 1];
    }
    const float dox = TSK_F2F_RN(go.x - fi.ox), doy = TSK_F2F_RN(go.y - fi.oy), doz = TSK_F2F_RN(go.z - fi.oz);
    const float dt = TSK_F2F_RN(go.w - fi.t0);
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
        const int i = k * 32 + lane;
        CandF32 c;
        c.px = c.py = c.pz = 0x1p60f;
        c.vx = c.vy = c.vz = c.sr = 0.f;
        if (ok[k]) c = f32_cand_rebase(a[k].x, a[k].y, a[k].z, b[k].x, b[k].y, b[k].z, a[k].w, dox, doy, doz, dt);
        wcs[0 * WCAND + i] = c.px; wcs[1 * WCAND + i] = c.py; wcs[2 * WCAND + i] = c.pz;
        wcs[3 * WCAND + i] = c.vx; wcs[4 * WCAND + i] = c.vy; wcs[5 * WCAND + i] = c.vz;
        wcs[6 * WCAND + i] = c.sr;
    }
}

__device__ __forceinline__ void stage_pair(const K1Launch &L, int64_t wbase, int64_t c_lo, int64_t c_hi, int k0,
                                           const F32Item &fi, float *wcs, int lane) {
    RawPair r;
    load_pair(L, wbase, c_lo, c_hi, k0, lane, r);
    store_pair(r, k0, fi, wcs, lane);
}

// jlo = #{j < nt : pm[j] < x} (pm ascending) and jhi = #{j < nt : sm[j] <= y}
// (sm ascending), both arrays +inf padded to K1_PMN (k1_exact.cuh): 16-ary rounds, lanes
// 0-15 on pm and 16-31 on sm (a shared load, a ballot and a popcount each:
// two rounds for 256 queries, three for 512 or 1,024) instead of two serial
// bisections.
static_assert(K1_TQ == 256 || K1_TQ == 512 || K1_TQ == 1024, "window_bounds covers 256, 512 or 1024 queries");
__device__ __forceinline__ void window_bounds(const double *pm, const double *sm, int nt, double x, double y, int lane,
                                              int &jlo, int &jhi) {
    const int l = lane & 15;
    const bool lo_half = lane < 16;
    const double *a = lo_half ? pm : sm;
    int r_lo = 0, r_hi = 0;
#pragma unroll
    for (int step = K1_TQ / 16; step >= 1; step = step >= 16 ? step / 16 : (step > 1 ? 1 : 0)) {
        // block l of `step` entries past the current bound ends at r + step (l + 1) - 1
        const int r = lo_half ? r_lo : r_hi;
        const int idx = r + step * (l + 1) - 1;
        const double v = idx < K1_PMN ? a[idx] : INFINITY;
        const unsigned m = __ballot_sync(0xffffffffu, lo_half ? v < x : v <= y);
        r_lo += step * __popc(m & 0xffffu);
        r_hi += step * __popc(m >> 16);
        if (step == 1) break;
    }
    jlo = r_lo < nt ? r_lo : nt;
    jhi = r_hi < nt ? r_hi : nt;
}

// Block-shared state of the FP32 kernel at file scope, so the sub-tile
// functions reach it without carrying pointers in registers across their
// calls (every value a caller keeps live across a call costs a spill).
__shared__ __align__(16) unsigned char k1f_lraw[sizeof(K1Launch)];  // the launch parameters
__device__ __forceinline__ const K1Launch &k1f_L() { return *reinterpret_cast<const K1Launch *>(k1f_lraw); }
__shared__ double k1f_pm[K1_PMN];  // running max / suffix min of te (or te / ts), +inf padded
__shared__ double k1f_sm[K1_PMN];
__shared__ F32Item k1f_fi;            // the item's FP32 origin and error bound
__shared__ ItemCtx k1f_it;            // the item
__shared__ float k1f_cull_rb;         // the launch's box-cull radius base
__shared__ int k1f_item_f32;          // the item takes the FP32 path

// Item-level key bases of the K1 layout (hits add their own orig - f).
__shared__ uint64_t k1_kb[K1_GMAX];  // per batch of the tile (pairs: 2, quads: 4, octets: 8)
__shared__ int64_t k1_kf[K1_GMAX];
__shared__ int k1_nbat;               // batches in the item's tile

// One warp sub-tile on the box-cull fast path (K1 layout, overlaps counted
// outside K1).  The window is every query whose extent meets the time range
// of the candidates' groups (two bisections on the tile's sorted ts / te);
// pairs in it that do not overlap in time are rejected by the exact path if
// they are ever flagged (its tb case is chosen per pair: the warp's end-time
// bounds are left open).  Only warps with a query near their box load their
// candidates, all columns in one round trip.
__device__ __noinline__ void fast_subtile(int64_t wbase, int warp, int lane, unsigned long long &n_ev, unsigned long long &n_hit) {
    const K1Launch &L = k1f_L();
    const ItemCtx &it = k1f_it;
    const F32Item &fi = k1f_fi;
    const QRec *const qt = L.q + it.lo_q;
    const QF32 *const sqf = f_sqf();
    const double *const pm = k1f_pm, *const sm = k1f_sm;
    float *const wcs = f_cands(warp);
    const float cull_rb = k1f_cull_rb;
    const bool item_f32 = k1f_item_f32 != 0;
    const int64_t g0 = wbase / BOX_GROUP;
    const int64_t g1 = (wbase + WCAND - 1 < it.c_hi ? wbase + WCAND - 1 : it.c_hi) / BOX_GROUP;
    // the groups' time range and box, loaded together
    double2 tr = L.gtime[g0];
    float4 blo, bhi;
    bool unsafe_g;
    warp_box(L, wbase, it.c_hi, blo, bhi, unsafe_g);
    if (g1 != g0) {
        const double2 t1 = L.gtime[g1];
        tr.x = tr.x < t1.x ? tr.x : t1.x;
        tr.y = tr.y > t1.y ? tr.y : t1.y;
    }
    // window [jlo, jhi): te_j >= min ts (pm: te ascending) and ts_j <= max te
    // (sm: ts ascending); both arrays are +inf padded to K1_PMN
    int jlo, jhi;
    window_bounds(pm, sm, it.nt, tr.x, tr.y, lane, jlo, jhi);
    if (jhi < jlo) jhi = jlo;
    const int ns = box_cull(blo, bhi, jlo, jhi, cull_rb, warp, lane);
    K1_STAT(0, 1);
    K1_STAT(1, jhi - jlo);
    K1_STAT(2, ns);
    K1_STAT(3, ns > 0);
    if (ns == 0) return;
    if (lane == 0) {
        const int nbat = k1_nbat;
#pragma unroll
        for (int g = 0; g < K1_GMAX; ++g)
            if (g < nbat) {
                k1_wctx[warp].key_base[g] = k1_kb[g];
                k1_wctx[warp].f[g] = k1_kf[g];
            }
        k1_wctx[warp].js = it.js;
#pragma unroll
        for (int i = 0; i < K1_GMAX - 2; ++i) k1_wctx[warp].jx[i] = it.jx[i];
        k1_wctx[warp].wbase = wbase;
        const int64_t nv = it.c_hi - wbase + 1;
        k1_wctx[warp].nvalid = nv < 0 ? 0 : (nv > WCAND ? WCAND : (int)nv);
        k1_wctx[warp].nlo = it.c_lo > wbase ? (int)(it.c_lo - wbase < WCAND ? it.c_lo - wbase : WCAND) : 0;
        // the exact path picks each pair's tb case itself (TB_DYN, open bounds)
        k1_wctx[warp].wmin_te = -INFINITY;
        k1_wctx[warp].wmax = INFINITY;
    }
    __syncwarp();
    if (!item_f32 || unsafe_g) {
        // extreme-exponent candidates or an item outside the FP32 path's
        // bounds: the exact path over the whole window
        // (its per-pair overlap counts are not needed here)
        double rts[CPT], rte[CPT];
        double wmin = INFINITY, wmax = -INFINITY, wmin_te = INFINITY, wmax_ts = -INFINITY;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int64_t e = wbase + k * 32 + lane;
            rts[k] = INFINITY;
            rte[k] = -INFINITY;
            if (e >= it.c_lo && e <= it.c_hi) {
                rts[k] = L.e.ts[e];
                rte[k] = L.e.te[e];
                wmin = rts[k] < wmin ? rts[k] : wmin;
                wmax = rte[k] > wmax ? rte[k] : wmax;
                wmin_te = rte[k] < wmin_te ? rte[k] : wmin_te;
                wmax_ts = rts[k] > wmax_ts ? rts[k] : wmax_ts;
            }
        }
        wmax = warp_max(wmax);
        wmin_te = warp_min(wmin_te);
        wmin = warp_min(wmin);
        wmax_ts = warp_max(wmax_ts);
        if (lane == 0) {
            k1_wctx[warp].wmin_te = wmin_te;
            k1_wctx[warp].wmax = wmax;
        }
        __syncwarp();
        unsigned long long ov_unused = 0;
        const int4 w = warp_window(sqf, pm, it.nt, false, wmin, wmax, wmax_ts, lane);
        all_range<TA_C>(qt, sqf, w.x, w.y, rts, rte, warp, lane, ov_unused, n_hit);
        all_range<TA_BOTH>(qt, sqf, w.y, w.z, rts, rte, warp, lane, ov_unused, n_hit);
        all_range<TA_R>(qt, sqf, w.z, w.w, rts, rte, warp, lane, ov_unused, n_hit);
        return;
    }
    n_ev += (unsigned long long)ns * (unsigned long long)k1_wctx[warp].nvalid;
    if (L.frec && wbase % BOX_GROUP == 0) {
        stage_rebased(L, wbase, it.c_lo, it.c_hi, fi, wcs, lane);
    } else {
        RawPair r0, r1;
        load_pair(L, wbase, it.c_lo, it.c_hi, 0, lane, r0);
        load_pair(L, wbase, it.c_lo, it.c_hi, 2, lane, r1);
        store_pair(r0, 0, fi, wcs, lane);
        store_pair(r1, 2, fi, wcs, lane);
    }
    __syncwarp();
    f32_list_range(qt, sqf, ns, warp, lane, n_hit);
}

// One warp sub-tile outside the box-cull fast path (start-sorted store,
// spans given by the caller, unsorted queries, counting modes, extreme
// exponents): per-pair overlap counts, the three start-time ranges, the
// exact path where the FP32 pre-filter does not apply.  Kept out of the
// kernel body so the fast path's register allocation is its own.
__device__ __noinline__ void slow_subtile(const K1Launch &L, const ItemCtx &it, const QRec *__restrict__ qt,
                                          const QF32 *__restrict__ sqf, const double *pm, const double *sm,
                                          int64_t wbase, float cull_rb, const F32Item &fi, bool item_f32,
                                          bool single_scan, bool te_sorted, bool q_unsorted, bool cull, float *wcs,
                                          int warp, int lane, unsigned long long &n_ov, unsigned long long &n_hit,
                                          unsigned long long &n_ev) {
        double rts[CPT], rte[CPT];
        bool valid_any = false, unsafe_r = false;
        double wmin = INFINITY, wmax = -INFINITY, wmin_te = INFINITY, wmax_ts = -INFINITY;
#pragma unroll
        for (int k = 0; k < CPT; ++k) {
            const int64_t e = wbase + k * 32 + lane;
            const bool valid = e >= it.c_lo && e <= it.c_hi;
            rts[k] = INFINITY;
            rte[k] = -INFINITY;
            if (valid) {
                rts[k] = L.e.ts[e];
                rte[k] = L.e.te[e];
                unsafe_r |= L.e.unsafe[e] != 0;
                // times are finite (validated): plain selects, no NaN handling
                wmin = rts[k] < wmin ? rts[k] : wmin;
                wmax = rte[k] > wmax ? rte[k] : wmax;
                wmin_te = rte[k] < wmin_te ? rte[k] : wmin_te;
                wmax_ts = rts[k] > wmax_ts ? rts[k] : wmax_ts;
            }
            valid_any |= valid;
        }
        if (L.noop) return;
        if (!__any_sync(0xffffffffu, valid_any)) return;
        wmax = warp_max(wmax);
        wmin_te = warp_min(wmin_te);
        if (lane == 0) {
            set_key_bases(L, it, wbase, warp);
            k1_wctx[warp].js = it.js;
            k1_wctx[warp].wbase = wbase;
            const int64_t nv = it.c_hi - wbase + 1;
            k1_wctx[warp].nvalid = nv < 0 ? 0 : (nv > WCAND ? WCAND : (int)nv);
            k1_wctx[warp].nlo = it.c_lo > wbase ? (int)(it.c_lo - wbase < WCAND ? it.c_lo - wbase : WCAND) : 0;
            k1_wctx[warp].wmin_te = wmin_te;
            k1_wctx[warp].wmax = wmax;
        }
        __syncwarp();
        const bool exact_only = !item_f32 || __any_sync(0xffffffffu, unsafe_r);
        if (single_scan && !exact_only) {
            // start and end times both ascending over the tile: a
            // candidate overlaps exactly the queries j with
            // ts_j <= r.te (a prefix) and te_j >= r.ts (a suffix), so its
            // count is two bisections, the window [jlo, jhi) of the warp
            // is their min / max (the warp_window bounds of wmin, wmax),
            // and the whole window is one scan (the exact path decides the
            // clip cases per pair)
            int lo[CPT], hi[CPT];
            tile_bounds<CPT>(sm, pm, it.nt, rts, rte, lo, hi);
            int jlo = it.nt, jhi = 0;
#pragma unroll
            for (int k = 0; k < CPT; ++k) {
                n_ov += split_count(lo[k], hi[k], it.js);
                jlo = lo[k] < jlo ? lo[k] : jlo;
                jhi = hi[k] > jhi ? hi[k] : jhi;
            }
            jlo = __reduce_min_sync(0xffffffffu, jlo);
            jhi = __reduce_max_sync(0xffffffffu, jhi);
            if (jhi < jlo) jhi = jlo;
            if (cull) {
                // K1 layout: one box test per (query, warp) first; the
                // candidates are converted only when a query survives
                float4 blo, bhi;
                bool bunsafe;
                warp_box(L, wbase, it.c_hi, blo, bhi, bunsafe);
                const int ns = box_cull(blo, bhi, jlo, jhi, cull_rb, warp, lane);
                n_ev += (unsigned long long)ns * (unsigned long long)k1_wctx[warp].nvalid;
                if (ns == 0) return;
                stage_cands(L, wbase, it.c_lo, it.c_hi, rts, fi, wcs, lane);
                __syncwarp();
                f32_list_range(qt, sqf, ns, warp, lane, n_hit);
                return;
            }
            stage_cands(L, wbase, it.c_lo, it.c_hi, rts, fi, wcs, lane);
            __syncwarp();
            n_ev += (unsigned long long)(jhi - jlo) * (unsigned long long)k1_wctx[warp].nvalid;
            f32_range<TA_BOTH, TB_DYN, false>(qt, sqf, jlo, jhi, warp, lane, n_ov, n_hit);
            return;
        }
        if (item_f32) stage_cands(L, wbase, it.c_lo, it.c_hi, rts, fi, wcs, lane);
        __syncwarp();
        wmin = warp_min(wmin);
        wmax_ts = warp_max(wmax_ts);
        const int4 w = warp_window(sqf, pm, it.nt, q_unsorted, wmin, wmax, wmax_ts, lane);
        const int jlo = w.x, ja = w.y, jb = w.z, jhi = w.w;
        if (L.overlaps_only) {
            n_ov += count_overlaps<CPT>(sqf, jlo, jhi, it.js, rts, rte);
            return;
        }
        if (exact_only) {
            all_range<TA_C>(qt, sqf, jlo, ja, rts, rte, warp, lane, n_ov, n_hit);
            all_range<TA_BOTH>(qt, sqf, ja, jb, rts, rte, warp, lane, n_ov, n_hit);
            all_range<TA_R>(qt, sqf, jb, jhi, rts, rte, warp, lane, n_ov, n_hit);
            return;
        }
        n_ev += (unsigned long long)(jhi - jlo) * (unsigned long long)k1_wctx[warp].nvalid;
        // TA_C range: every query ends before all candidates (running max
        // < min te) and te is sorted → overlaps counted by bisection
        if (jlo < ja && pm[ja - 1] < wmin_te && te_sorted) {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                n_ov += split_count(clampi(lower_bound_te(sqf, it.nt, rts[k]), jlo, ja), ja, it.js);
            f32_range<TA_C, TB_R, false>(qt, sqf, jlo, ja, warp, lane, n_ov, n_hit);
        } else {
            f32_range<TA_C, TB_DYN, true>(qt, sqf, jlo, ja, warp, lane, n_ov, n_hit);
        }
        f32_range<TA_BOTH, TB_DYN, true>(qt, sqf, ja, jb, warp, lane, n_ov, n_hit);
        // TA_R range: every query ends after all candidates (suffix min >
        // max te) → overlap <=> cts <= r.te, counted by bisection
        if (jb < jhi && sm[jb] > wmax) {
#pragma unroll
            for (int k = 0; k < CPT; ++k)
                n_ov += split_count(jb, clampi(upper_bound_ts(sqf, it.nt, rte[k]), jb, jhi), it.js);
            f32_range<TA_R, TB_C, false>(qt, sqf, jb, jhi, warp, lane, n_ov, n_hit);
        } else {
            f32_range<TA_R, TB_DYN, true>(qt, sqf, jb, jhi, warp, lane, n_ov, n_hit);
        }
}

__global__ void __launch_bounds__(K1_THREADS, K1F_MIN_BLOCKS) K1F_NAME(k1_pairs_f32)(K1Launch Lp) {
    // the launch parameters in shared memory: the device functions take them
    // by reference, and a reference to the parameter space would make every
    // thread keep a copy on its stack (local memory)
    if (threadIdx.x == 0) *reinterpret_cast<K1Launch *>(k1f_lraw) = Lp;
    __syncthreads();
    const K1Launch &L = k1f_L();
    // running max / suffix min of te over the tile; on single-scan items
    // (times ascending) te / ts themselves, +inf padded for tile_bounds
    double *const pm = k1f_pm;
    double *const sm = k1f_sm;
    __shared__ double f32b[8];    // per-item magnitude bounds
    __shared__ double f32p[K1_WARPS][4];  // per-warp partial maxima of the bounds pass
    F32Item &fi_sh = k1f_fi;      // the item's FP32 origin and error bound
    ItemCtx &it_sh = k1f_it;
    __shared__ int64_t item_sh;
    __shared__ int flags_sh;      // bit 0: unsafe query, bit 1: te not sorted
    __shared__ unsigned long long red[4], red_ev;  // per-batch overlap / hit sums, evaluated pairs
    __shared__ int wsub_next;     // fast path: the item's next unclaimed warp sub-tile

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        fill_flush_cfg(L);
        for (int i = 0; i < K1_GMAX - 2; ++i) k1_hitsx[i] = 0;
    }
    QF32 *const sqf = f_sqf();
    float *const wcs = f_cands(warp);
    const int64_t total = L.plan.meta[0];
    const int sub = (int)L.plan.meta[1];
    const int64_t tqs = L.plan.meta[2];  // query tile size chosen by k_plan_items (<= K1_TQ)
    constexpr int64_t STRIDE = (int64_t)K1_THREADS * CPT;  // candidates per sub-tile
    const int64_t ct = STRIDE * sub;
    const double cq = __longlong_as_double((long long)*L.q_cmax_bits);
    const double cmax = L.db_cmax > cq ? L.db_cmax : cq;
    // launch-level validity: the FP32 pre-filter needs |coordinates| and d
    // below 2^60 (and the FP64 filter's window for the exact division)
    const bool launch_ok = k1f_launch_ok(cmax, L.d2);
    const double dthr = sqrt(L.d2);  // d (sqrt(RN(d^2)) >= d (1 - 2^-52); the margin covers it)
    const float cull_rb = box_cull_rbase(dthr, cmax);  // filter.cuh
    if (threadIdx.x == 0) k1f_cull_rb = cull_rb;
    const bool cull = L.cull && launch_ok;

    for (;;) {
        if (tid == 0) {
            const int64_t item = (int64_t)atomicAdd(L.item_counter, 1ull);
            item_sh = item;
            if (item < total) it_sh = decode_item(L, item, ct, tqs);
            red[0] = red[1] = red[2] = red[3] = 0;
            red_ev = 0;
            wsub_next = 0;
            flags_sh = 0;
        }
        __syncthreads();
        if (item_sh >= total) break;
        if (tid == 0) K1_STAT(7, 1);
        const ItemCtx &it = it_sh;  // read from shared memory (a register copy spills to the stack)
        const QRec *const qt = L.q + it.lo_q;  // the tile's exact records (global; rare path)

        // pass 1 over the tile: flags, and the item's magnitude bounds
        // relative to (O, T0) = the first query's start (warps 2, 3)
        {
            int fl = 0;
            for (int j = tid; j < it.nt; j += K1_THREADS) {
                if (qt[j].flag != 0.0) fl |= 1;
                if (j + 1 < it.nt && qt[j + 1].te < qt[j].te) fl |= 2;
            }
            if (fl) atomicOr(&flags_sh, fl);
            const double ox = qt[0].sx, oy = qt[0].sy, oz = qt[0].sz, t0 = qt[0].ts;
            // warps 2 .. 2 + KW - 1 bound the candidate groups, the warps above
            // them the queries; thread 0 folds the per-warp maxima (fmax is
            // exact and order-free) after the barrier
            constexpr int KW = (K1_WARPS - 2) / 2;
            if (warp >= 2 && warp < 2 + KW) {
                double ar = 0.0, tvr = 0.0, vr = 0.0, trr = 0.0;
                for (int64_t g = it.first_c / GB_SIZE + (warp - 2) * 32 + lane; g <= it.c_hi / GB_SIZE; g += 32 * KW) {
                    const GBound gb = L.e.gb[g];
                    ar = fmax(ar, fmax(fmax(fabs(gb.hi[0] - ox), fabs(ox - gb.lo[0])),
                                       fmax(fmax(fabs(gb.hi[1] - oy), fabs(oy - gb.lo[1])),
                                            fmax(fabs(gb.hi[2] - oz), fabs(oz - gb.lo[2])))));
                    const double tg = fmax(fabs(gb.ts_hi - t0), fabs(t0 - gb.ts_lo));
                    tvr = fmax(tvr, tg * gb.vmax);
                    trr = fmax(trr, tg);
                    vr = fmax(vr, gb.vmax);
                }
                ar = warp_max(ar);
                tvr = warp_max(tvr);
                vr = warp_max(vr);
                trr = warp_max(trr);
                if (lane == 0) {
                    f32p[warp][0] = ar;
                    f32p[warp][1] = tvr;
                    f32p[warp][2] = vr;
                    f32p[warp][3] = trr;
                }
            } else if (warp >= 2 + KW) {
                constexpr int QW = K1_WARPS - 2 - KW;
                double aq = 0.0, tq = 0.0, eq = 0.0, dq = 0.0;
                for (int j = (warp - 2 - KW) * 32 + lane; j < it.nt; j += 32 * QW) {
                    const QRec &q = qt[j];
                    aq = fmax(aq, fmax(fabs(q.sx - ox), fmax(fabs(q.sy - oy), fabs(q.sz - oz))));
                    tq = fmax(tq, fabs(q.ts - t0));
                    eq = fmax(eq, q.ext);
                    dq = fmax(dq, fmax(fabs(q.dx), fmax(fabs(q.dy), fabs(q.dz))));
                }
                aq = warp_max(aq);
                tq = warp_max(tq);
                eq = warp_max(eq);
                dq = warp_max(dq);
                if (lane == 0) {
                    f32p[warp][0] = aq;
                    f32p[warp][1] = tq;
                    f32p[warp][2] = eq;
                    f32p[warp][3] = dq;
                }
            }
        }
        __syncthreads();
        const bool unsafe_q = flags_sh & 1;
        const bool te_sorted = !(flags_sh & 2);
        const bool q_unsorted = (*L.q_unsorted & 1) != 0;  // bit 0: query ts, bit 1: query te not sorted
        const bool single_scan = te_sorted && !q_unsorted && !L.overlaps_only;
        // box-cull fast path: overlaps are counted outside K1
        // (count_overlaps_ext), so a warp whose window has no query near its
        // box costs two bisections and the box tests, nothing per candidate
        const bool fast = cull && L.ext_count && (*L.q_unsorted & 3) == 0 && single_scan;
        if (tid == 0) {
            {  // fold the bounds pass's per-warp maxima
                constexpr int KW = (K1_WARPS - 2) / 2;
                double m[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                for (int w = 2; w < K1_WARPS; ++w)
                    for (int k = 0; k < 4; ++k) {
                        const int o = w < 2 + KW ? k : 4 + k;
                        m[o] = fmax(m[o], f32p[w][k]);
                    }
                f32b[0] = m[0];  // ar
                f32b[1] = m[1];  // tvr
                f32b[2] = m[2];  // vr
                f32b[7] = m[3];  // trr
                f32b[3] = m[4];  // aq
                f32b[4] = m[5];  // tq
                f32b[5] = m[6];  // eq
                f32b[6] = m[7];  // dq
            }
            fi_sh = f32_item(qt[0].sx, qt[0].sy, qt[0].sz, qt[0].ts, f32b[0], f32b[1], f32b[2], f32b[3], f32b[4],
                             f32b[5], cmax, f32b[7]);
            fi_sh.ok = fi_sh.ok && launch_ok && !unsafe_q;
            // separating-axis stage: M2 = A_r + TV_r + (T_q + E_q) V_r + A_q + D_q
            const double M2 = f32b[0] + f32b[1] + (f32b[4] + f32b[5] + f32b[7]) * f32b[2] + f32b[3] + f32b[6];
            k1_sep_rb = f32_sep_rbase(dthr, cmax, M2);
            if (L.orig) {  // K1 layout: key bases are per item and batch
                const int nbat = item_batches(it);
                k1_nbat = nbat;
                for (int g = 0; g < nbat; ++g) {
                    k1_kf[g] = L.plan.first[it.b + g];
                    k1_kb[g] = make_key(L, it.b + g, 0, g == 0 ? it.q0 : 0);
                }
            }
        }
        __syncthreads();
        const bool item_f32 = fi_sh.ok;
        if (tid == 0) k1f_item_f32 = item_f32 ? 1 : 0;  // read after the next barrier
        // pass 2: the FP32 records (exact times always, for windows and counts)
        for (int j = tid; j < it.nt; j += K1_THREADS) {
            const QRec &q = qt[j];
            QF32 f;
            if (item_f32) {
                float v[6];
                f32_query(q.ts, q.sx, q.sy, q.sz, q.ext, q.dx, q.dy, q.dz, fi_sh, dthr, v);
                f.ts = v[0]; f.x = v[1]; f.y = v[2]; f.z = v[3]; f.a = v[4]; f.b = v[5];
                float w[4];
                f32_query_end(q.te, q.ex, q.ey, q.ez, fi_sh, w);
                f.te = w[0]; f.ex = w[1]; f.ey = w[2]; f.ez = w[3];
            } else {
                f.ts = f.x = f.y = f.z = f.a = f.b = 0.f;
                f.te = f.ex = f.ey = f.ez = 0.f;
            }
            f.pad0 = f.pad1 = 0.f;
            f.ts64 = q.ts;
            f.te64 = q.te;
            sqf[j] = f;
            if (cull) {  // the query segment's box, rounded outward
                // .w of the low corner: the box's share of the cull radius
                const float lx = __double2float_rd(fmin(q.sx, q.ex)), ly = __double2float_rd(fmin(q.sy, q.ey)),
                            lz = __double2float_rd(fmin(q.sz, q.ez));
                const float hx = __double2float_ru(fmax(q.sx, q.ex)), hy = __double2float_ru(fmax(q.sy, q.ey)),
                            hz = __double2float_ru(fmax(q.sz, q.ez));
                f_qbox()[2 * j] = make_float4(lx, ly, lz, box_cull_dterm(lx, ly, lz, hx, hy, hz));
                f_qbox()[2 * j + 1] = make_float4(hx, hy, hz, 0.f);
            }
        }
        __syncthreads();
        if (single_scan) {
            for (int j = tid; j < K1_PMN; j += K1_THREADS) {
                pm[j] = j < it.nt ? sqf[j].te64 : INFINITY;
                sm[j] = j < it.nt ? sqf[j].ts64 : INFINITY;
            }
        } else {
            te_scans(sqf, it.nt, pm, sm, warp, lane);
        }
        __syncthreads();

        unsigned long long n_ov = 0, n_hit = 0;  // batch b in the low half, b1 in the high half
        unsigned long long n_ev = 0;  // pairs evaluated by the pre-filter (warp-uniform)
        if (fast && !L.noop) {
            // warps claim the item's warp sub-tiles (128 candidates) one at a
            // time, so the end-of-item barrier waits for one sub-tile at most
            const int nw = (int)((it.c_hi - it.first_c) / WCAND) + 1;
            for (;;) {
                int w = 0;
                if (lane == 0) w = atomicAdd(&wsub_next, 1);
                w = __shfl_sync(0xffffffffu, w, 0);
                if (w >= nw) break;
                fast_subtile(it.first_c + (int64_t)w * WCAND, warp, lane, n_ev, n_hit);
            }
        }
        for (int s = 0; s < sub && !(fast && !L.noop); ++s) {
            const int64_t base = it.first_c + (int64_t)s * STRIDE;
            if (base > it.c_hi) break;  // block-uniform
            const int64_t wbase = base + (int64_t)warp * WCAND;
            if (fast) {
                if (wbase > it.c_hi || L.noop) continue;
                fast_subtile(wbase, warp, lane, n_ev, n_hit);
                continue;
            }
            slow_subtile(L, it, qt, sqf, pm, sm, wbase, cull_rb, fi_sh, item_f32, single_scan, te_sorted, q_unsorted,
                         cull, wcs, warp, lane, n_ov, n_hit, n_ev);
        }
        if (lane == 0 && n_ev) atomicAdd(&red_ev, n_ev);
        item_counters(L, it, n_ov, n_hit, lane, tid, red, &red_ev);
    }
}

static size_t k1f_dyn_smem() { return Q2_OFF + sizeof(uint32_t) * Q2CAP * K1_WARPS; }

static void k1f_set_attrs() {
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(done_mask.load() & bit)) {
        TSK_CUDA(cudaFuncSetAttribute(K1F_NAME(k1_pairs_f32), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k1f_dyn_smem()));
        done_mask.fetch_or(bit);
    }
}

int K1F_NAME(k1f_blocks_per_sm)() {
    k1f_set_attrs();
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, K1F_NAME(k1_pairs_f32), K1_THREADS, k1f_dyn_smem());
    return n > 0 ? n : 1;
}

int K1F_NAME(k1f_candidates_per_thread)() { return CPT; }

K1F_NS_CLOSE
}  // namespace tsk

#ifndef K1_WIDE
// Development counters of K1 (zeros unless built with -DTSK_K1_STATS):
// both builds' counters, summed.
extern "C" int tsk_k1_stats(int device, unsigned long long *out, int n, int reset) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    unsigned long long v[8] = {0}, w[8] = {0};
    if (cudaMemcpyFromSymbol(v, tsk::k1_stats, sizeof(v)) != cudaSuccess) return 1;
    if (tsk::k1f_stats_wide(w, reset) != 0) return 1;
    for (int i = 0; i < n && i < 8; ++i) out[i] = v[i] + w[i];
    if (reset) {
        const unsigned long long z[8] = {0};
        if (cudaMemcpyToSymbol(tsk::k1_stats, z, sizeof(z)) != cudaSuccess) return 1;
    }
    return 0;
}
#else
namespace tsk {
inline namespace wide {
// the wide build's development counters (read, optionally reset)
int k1f_stats_wide(unsigned long long *v, int reset) {
    if (cudaMemcpyFromSymbol(v, k1_stats_wide, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (reset) {
        const unsigned long long z[8] = {0};
        if (cudaMemcpyToSymbol(k1_stats_wide, z, sizeof(z)) != cudaSuccess) return 1;
    }
    return 0;
}
}  // namespace wide
}  // namespace tsk
#endif

namespace tsk {
K1F_NS_OPEN

void K1F_NAME(launch_k1f)(const K1Launch &L, int grid, cudaStream_t st) {
    k1f_set_attrs();
    K1F_NAME(k1_pairs_f32)<<<grid, K1_THREADS, k1f_dyn_smem(), st>>>(L);
    TSK_CUDA(cudaGetLastError());
}

K1F_NS_CLOSE
}  // namespace tsk
