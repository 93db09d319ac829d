// k1_pairs.cu — K1 with the FP64 filter (GPUTrajDistSearch).
//
// The FP32 pre-filter kernel (k1_f32.cu) is the common path; this kernel
// serves launches whose magnitudes are outside the FP32 pre-filter's
// validity (|coordinate| > 2^60 or d > 2^60), with the FP64 filter of
// filter.cuh in its inner loop.
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

#include "k1_exact.cuh"

#ifndef K1_CPT
#define K1_CPT 2
#endif
#ifndef K1_MIN_BLOCKS
#define K1_MIN_BLOCKS 1  // K1_THREADS = 448: one CTA's registers, no spills
#endif

namespace tsk {

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

// Queue entries per warp.  A query iteration starts with fewer than 32
// queued and appends at most 32 * K1_CPT.
constexpr int K1_QCAP = 32 * (K1_CPT + 1);

extern __shared__ __align__(16) unsigned char k1_dyn[];
__device__ __forceinline__ uint32_t *warp_q(int warp) { return reinterpret_cast<uint32_t *>(k1_dyn) + warp * K1_QCAP; }

// One warp, K1_CPT candidates per lane, staged queries j0..j1-1 of one
// (TA, TB) case.  SLOW: every overlapping pair is queued for the exact IEEE
// path (extreme-exponent tiles, launches outside the filter bounds);
// otherwise the FP64 filter decides.  CNT: count overlaps per iteration;
// otherwise the caller counts them for the whole range by binary search and
// lanes that do not overlap a query are rejected on the rare path (window
// edges only).  Flagged pairs are queued and evaluated exactly 32 at a time
// (rare_flush), so hit-dense workloads do not serialise the warp.
template <int TA, int TB, bool SLOW, bool CNT>
__device__ __forceinline__ void pair_run(const QRec *__restrict__ sq, int j0, int j1, const CandF (&r)[K1_CPT],
                                         double wmin_te, double wmax_te, int warp, int lane,
                                         unsigned long long &n_ov, unsigned long long &n_hit, const FilterK &K) {
    uint32_t *const wq = warp_q(warp);
    constexpr uint32_t STRIDE = (uint32_t)sizeof(QRec);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sq);
    int qn = 0;  // queued entries (warp-uniform)
    uint32_t qa = base + (uint32_t)j0 * STRIDE;
    const uint32_t qa_end = base + (uint32_t)j1 * STRIDE;
    for (;;) {
        // inner loop: loads, math, one vote, one branch per query; it exits
        // when 32 or more flags are queued (the flush runs outside it)
        for (; qa < qa_end; qa += STRIDE) {
            bool cand[K1_CPT];
            if (SLOW) {
                double cts, cte;
                lds2(qa, cts, cte);
#pragma unroll
                for (int k = 0; k < K1_CPT; ++k) {
                    const bool ov = r[k].ts <= cte && cts <= r[k].te;  // invalid lanes: ts = +inf
                    if (CNT) n_ov += ov ? 1ull : 0ull;
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
                        n_ov += ov ? 1ull : 0ull;
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
        const bool done = qa >= qa_end;
        flush_queue<TA, TB, SLOW, K1_CPT>(sq, wq, warp, lane, qn, done, n_hit);
        if (done) break;
    }
}

// The three start-time ranges of a warp's window.  C_BISECT: every query of
// the TA_C range ends before all candidates and te is sorted, so overlaps
// are counted by bisection; R_BISECT likewise for the TA_R range (every
// query ends after all candidates).
template <bool SLOW>
__device__ __forceinline__ void run_cases(const QRec *__restrict__ sq, int nt, int4 w, bool c_bisect,
                                          bool r_bisect, const CandF (&r)[K1_CPT], double wmin_te,
                                          double wmax, int warp, int lane, unsigned long long &n_ov, unsigned long long &n_hit,
                                          const FilterK &K) {
    const int jlo = w.x, ja = w.y, jb = w.z, jhi = w.w;
    if (c_bisect && !SLOW) {
        // overlap <=> r.ts <= cte; cte ascending over the tile
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k)
            n_ov += (unsigned long long)(ja - clampi(lower_bound_te(sq, nt, r[k].ts), jlo, ja));
        pair_run<TA_C, TB_R, SLOW, false>(sq, jlo, ja, r, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    } else {
        pair_run<TA_C, TB_DYN, SLOW, true>(sq, jlo, ja, r, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    }
    pair_run<TA_BOTH, TB_DYN, SLOW, true>(sq, ja, jb, r, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    if (r_bisect && !SLOW) {
        // overlap <=> cts <= r.te; cts ascending over the tile
#pragma unroll
        for (int k = 0; k < K1_CPT; ++k)
            n_ov += (unsigned long long)(clampi(upper_bound_ts(sq, nt, r[k].te), jb, jhi) - jb);
        pair_run<TA_R, TB_C, SLOW, false>(sq, jb, jhi, r, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    } else {
        pair_run<TA_R, TB_DYN, SLOW, true>(sq, jb, jhi, r, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
    }
}

__global__ void __launch_bounds__(K1_THREADS, K1_MIN_BLOCKS) k1_pairs(K1Launch L) {
    __shared__ QRec sq[K1P_TQ];
    __shared__ double pm[K1P_TQ];  // running max of te over the tile
    __shared__ double sm[K1P_TQ];  // suffix min of te over the tile
    __shared__ ItemCtx it_sh;
    __shared__ int64_t item_sh;
    __shared__ unsigned long long red[4];  // per-batch overlap / hit sums

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        fill_flush_cfg(L);
        for (int i = 0; i < K1_GMAX - 2; ++i) k1_hitsx[i] = 0;
    }
    const int64_t total = L.plan.meta[0];
    const int sub = (int)L.plan.meta[1];
    const int64_t tqs = L.plan.meta[2];  // query tile size chosen by k_plan_items (<= K1P_TQ)
    constexpr int64_t STRIDE = (int64_t)K1_THREADS * K1_CPT;  // candidates per sub-tile
    const int64_t ct = STRIDE * sub;
    // filter constants (filter.cuh); C = max |coordinate| of entries and queries
    const double cq = __longlong_as_double((long long)*L.q_cmax_bits);
    const double cmax = L.db_cmax > cq ? L.db_cmax : cq;
    FilterK K = filter_consts(cmax, L.d2);
    K.km = L.filter_km;
    const bool launch_exact = !filter_ok(cmax, L.d2);

    for (;;) {
        if (tid == 0) {
            const int64_t item = (int64_t)atomicAdd(L.item_counter, 1ull);
            item_sh = item;
            if (item < total) it_sh = decode_item(L, item, ct, tqs);
            red[0] = red[1] = red[2] = red[3] = 0;
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
        te_scans(sq, it.nt, pm, sm, warp, lane);
        __syncthreads();

        unsigned long long n_ov = 0, n_hit = 0;
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
                const bool valid = e >= it.c_lo && e <= it.c_hi;
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
            if (L.noop) continue;
            if (!__any_sync(0xffffffffu, valid_any)) continue;
            wmin = warp_min(wmin);
            wmax = warp_max(wmax);
            wmin_te = warp_min(wmin_te);
            wmax_ts = warp_max(wmax_ts);
            if (lane == 0) {
                set_key_bases(L, it, wbase, warp);  // (no shared units in this kernel: b1 < 0)
                k1_wctx[warp].js = it.nt;
                k1_wctx[warp].wbase = wbase;
                const int64_t nv = it.c_hi - wbase + 1;
                k1_wctx[warp].nvalid = nv < 0 ? 0 : (nv > 32 * K1_CPT ? 32 * K1_CPT : (int)nv);
                k1_wctx[warp].nlo = it.c_lo > wbase ? (int)(it.c_lo - wbase < 32 * K1_CPT ? it.c_lo - wbase : 32 * K1_CPT) : 0;
                k1_wctx[warp].wmin_te = wmin_te;
                k1_wctx[warp].wmax = wmax;
            }
            __syncwarp();
            const int4 w = warp_window(sq, pm, it.nt, (*L.q_unsorted & 1) != 0, wmin, wmax, wmax_ts, lane);
            if (L.overlaps_only) {
                double ts[K1_CPT], te[K1_CPT];
#pragma unroll
                for (int k = 0; k < K1_CPT; ++k) {
                    ts[k] = r[k].ts;
                    te[k] = r[k].te;
                }
                n_ov += count_overlaps<K1_CPT>(sq, w.x, w.w, it.nt, ts, te);
                continue;
            }
            const bool slow = launch_exact || unsafe_q || __any_sync(0xffffffffu, unsafe_r);
            // tb case of a whole range: every query of the TA_C range ends
            // before all candidates (running max < min te), or every query of
            // the TA_R range ends after all of them (suffix min > max te)
            const bool c_tb_r = w.x < w.y && pm[w.y - 1] < wmin_te;
            const bool r_tb_c = w.z < w.w && sm[w.z] > wmax;
            if (slow)
                run_cases<true>(sq, it.nt, w, false, false, r, wmin_te, wmax, warp, lane, n_ov, n_hit, K);
            else
                run_cases<false>(sq, it.nt, w, c_tb_r && te_sorted, r_tb_c, r, wmin_te, wmax, warp, lane, n_ov,
                                 n_hit, K);
        }
        item_counters(L, it, n_ov, n_hit, lane, tid, red);
    }
}

static size_t k1_dyn_smem() { return sizeof(uint32_t) * K1_QCAP * K1_WARPS; }

// The dynamic shared-memory limit is a per-device function attribute.
static void k1_set_attrs() {
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(done_mask.load() & bit)) {
        TSK_CUDA(cudaFuncSetAttribute(k1_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k1_dyn_smem()));
        done_mask.fetch_or(bit);
    }
}

bool k1_use_f32(double d2, double db_cmax) { return d2 <= 0x1p120 && db_cmax <= 0x1p60; }

int k1_blocks_per_sm(bool f32) {
    if (f32) return k1f_blocks_per_sm();
    k1_set_attrs();
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k1_pairs, K1_THREADS, k1_dyn_smem());
    return n > 0 ? n : 1;
}

int k1_candidates_per_thread(bool f32) { return f32 ? k1f_candidates_per_thread() : K1_CPT; }

void launch_k1(const K1Launch &L, int grid, cudaStream_t st) {
    if (k1_use_f32(L.d2, L.db_cmax)) {
        if (L.wide) launch_k1f_wide(L, grid, st);
        else launch_k1f(L, grid, st);
        return;
    }
    k1_set_attrs();
    k1_pairs<<<grid, K1_THREADS, k1_dyn_smem(), st>>>(L);
    TSK_CUDA(cudaGetLastError());
}

}  // namespace tsk
