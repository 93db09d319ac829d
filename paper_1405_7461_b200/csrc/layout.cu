// layout.cu — K1's spatially ordered copy of an indexed store (K1Layout).
//
// Built by tsk_index_build after the bins exist (index.py:85-146): every
// entry gets the key (bin, Morton code of its segment midpoint), the code
// reversed in odd bins so the groups that straddle a bin boundary stay
// compact too; a stable radix sort of the keys gives the permutation, and
// the hoisted SoA columns are gathered into the new order.  Candidate
// ranges of indexed searches are unions of whole bins (index.py:160-173),
// hence the same ordinal range in both orders, and the reference's result
// order is restored through `orig` (hit keys carry start-sorted ordinals).
//
// Per BOX_GROUP (128) consecutive entries of the new order K1 gets the
// bounding box of their segments, rounded outward to FP32.  While both
// segments of a pair are active each point lies on its own segment, so a
// reference hit needs the two segments' boxes within the threshold (plus
// the margin derived in filter.cuh, see box_cull_r2); K1 tests a warp's
// 128 candidates against each query of its window with one box test.
//
// Bound: HBM (one read of the store's 125 B/segment of K1 columns, one
// write, a 16-byte key/value sort) — setup, outside the response time.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "filter.cuh"
#include "tsk_internal.cuh"

namespace tsk {

// order-preserving u64 image of a double (for atomicMin/Max)
__device__ __forceinline__ unsigned long long ord_bits(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
static double ord_value(unsigned long long o) {
    const unsigned long long b = (o >> 63) ? (o & 0x7fffffffffffffffull) : ~o;
    double v;
    memcpy(&v, &b, 8);
    return v;
}

// bounding box of the segment midpoints: out[0..2] min, out[3..5] max (ord_bits)
__global__ void k_mid_box(int64_t n, const double *__restrict__ sx, const double *__restrict__ sy,
                          const double *__restrict__ sz, const double *__restrict__ ex,
                          const double *__restrict__ ey, const double *__restrict__ ez,
                          unsigned long long *out) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double m[3] = {0.5 * (sx[i] + ex[i]), 0.5 * (sy[i] + ey[i]), 0.5 * (sz[i] + ez[i])};
        for (int c = 0; c < 3; ++c) {
            lo[c] = fmin(lo[c], m[c]);
            hi[c] = fmax(hi[c], m[c]);
        }
    }
    for (int o = 16; o; o >>= 1)
        for (int c = 0; c < 3; ++c) {
            lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int c = 0; c < 3; ++c) {
            atomicMin(&out[c], ord_bits(lo[c]));
            atomicMax(&out[3 + c], ord_bits(hi[c]));
        }
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {  // 10 bits -> every third bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

struct MortonFrame {
    double lo[3], scale[3];  // cell = (m - lo) * scale, clamped to [0, 1023]
};

__global__ void k_layout_keys(int64_t n, const double *__restrict__ ts, const double *__restrict__ sx,
                              const double *__restrict__ sy, const double *__restrict__ sz,
                              const double *__restrict__ ex, const double *__restrict__ ey,
                              const double *__restrict__ ez, double t0, double width, int64_t m,
                              MortonFrame fr, uint64_t *__restrict__ keys, int64_t *__restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double mid[3] = {0.5 * (sx[i] + ex[i]), 0.5 * (sy[i] + ey[i]), 0.5 * (sz[i] + ez[i])};
        uint32_t code = 0;
        for (int c = 0; c < 3; ++c) {
            double q = (mid[c] - fr.lo[c]) * fr.scale[c];
            q = q > 0.0 ? (q < 1023.0 ? q : 1023.0) : 0.0;  // NaN -> 0
            code |= spread10((uint32_t)q) << c;
        }
        const int64_t b = bin_of(ts[i], t0, width, m);
        if (b & 1) code = 0x3fffffffu - code;  // boustrophedon: bins alternate direction
        keys[i] = ((uint64_t)b << 30) | code;
        vals[i] = i;
    }
}

__global__ void k_layout_gather(int64_t n, const int64_t *__restrict__ perm, Soa src, Soa dst,
                                int64_t *__restrict__ orig) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = perm[i];
        orig[i] = j;
        dst.ts[i] = src.ts[j]; dst.te[i] = src.te[j];
        dst.sx[i] = src.sx[j]; dst.sy[i] = src.sy[j]; dst.sz[i] = src.sz[j];
        dst.ex[i] = src.ex[j]; dst.ey[i] = src.ey[j]; dst.ez[i] = src.ez[j];
        dst.dx[i] = src.dx[j]; dst.dy[i] = src.dy[j]; dst.dz[i] = src.dz[j];
        dst.rcp[i] = src.rcp[j];
        dst.vx[i] = src.vx[j]; dst.vy[i] = src.vy[j]; dst.vz[i] = src.vz[j];
        dst.sr32[i] = src.sr32[j];
        dst.unsafe[i] = src.unsafe[j];
    }
}

// one warp per BOX_GROUP entries: the segments' bounding box, rounded outward,
// the group's time range and whether it holds an unsafe segment
__global__ void k_group_boxes(int64_t n, Soa s, float4 *__restrict__ box, double2 *__restrict__ gtime) {
    const int lane = threadIdx.x & 31;
    const int64_t ng = (n + BOX_GROUP - 1) / BOX_GROUP;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < ng;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        double tlo = INFINITY, thi = -INFINITY;
        bool unsafe = false;
        for (int k = lane; k < BOX_GROUP; k += 32) {
            const int64_t i = g * BOX_GROUP + k;
            if (i >= n) break;
            unsafe |= s.unsafe[i] != 0;
            tlo = fmin(tlo, s.ts[i]);
            thi = fmax(thi, s.te[i]);
            const double a[3] = {s.sx[i], s.sy[i], s.sz[i]}, b[3] = {s.ex[i], s.ey[i], s.ez[i]};
            for (int c = 0; c < 3; ++c) {
                lo[c] = fmin(lo[c], fmin(a[c], b[c]));
                hi[c] = fmax(hi[c], fmax(a[c], b[c]));
            }
        }
        for (int o = 16; o; o >>= 1) {
            for (int c = 0; c < 3; ++c) {
                lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
                hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
            }
            tlo = fmin(tlo, __shfl_xor_sync(0xffffffffu, tlo, o));
            thi = fmax(thi, __shfl_xor_sync(0xffffffffu, thi, o));
        }
        unsafe = __any_sync(0xffffffffu, unsafe);
        if (lane == 0) {
            gtime[g] = make_double2(tlo, thi);
            // .w of the low corner: 1 when a segment of the group has extreme
            // exponents (K1 then evaluates its pairs exactly)
            box[2 * g] = make_float4(__double2float_rd(lo[0]), __double2float_rd(lo[1]),
                                     __double2float_rd(lo[2]), unsafe ? 1.f : 0.f);
            box[2 * g + 1] = make_float4(__double2float_ru(hi[0]), __double2float_ru(hi[1]),
                                         __double2float_ru(hi[2]), 0.f);
        }
    }
}

// FP32 pre-filter records relative to each group's origin (the start of its
// first entry): f32_cand_sr with that origin, stored once per store.
__global__ void k_f32_records(int64_t n, Soa s, float4 *__restrict__ frec, double4 *__restrict__ gorig) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g0 = (i / BOX_GROUP) * BOX_GROUP;
        F32Item o;
        o.ox = s.sx[g0]; o.oy = s.sy[g0]; o.oz = s.sz[g0]; o.t0 = s.ts[g0];
        const CandF32 c = f32_cand_sr(s.ts[i], s.sx[i], s.sy[i], s.sz[i], s.vx[i], s.vy[i], s.vz[i], s.sr32[i], o);
        frec[2 * i] = make_float4(c.px, c.py, c.pz, c.sr);
        frec[2 * i + 1] = make_float4(c.vx, c.vy, c.vz, 0.f);
        if (i == g0) gorig[i / BOX_GROUP] = make_double4(o.ox, o.oy, o.oz, o.t0);
    }
}

// Temporal overlaps per batch without K1 (stores and queries whose start and
// end times are both non-decreasing): query q overlaps entry e iff
// e.ts <= q.te and q.ts <= e.te (core.py:490-492), so over a batch's range
// [f, l] of the start-sorted store
//   overlaps(q) = #{e: ts_e <= q.te} - #{e: te_e < q.ts}
// (te_e < q.ts implies ts_e <= q.te), two bisections per query.  One block
// per batch; the sum goes to the batch's overlap counter.  Runs only when
// the device flags of the query set say both time columns are sorted
// (else K1 counts per pair as before).
__global__ void __launch_bounds__(128) k_count_overlaps_ext(SearchPlanDev p, const double *__restrict__ qts,
                                                            const double *__restrict__ qte,
                                                            const double *__restrict__ ets,
                                                            const double *__restrict__ ete, const int *q_flags,
                                                            const unsigned long long *q_cmax_bits, double db_cmax,
                                                            double d2) {
    // exactly when K1 takes its fast path for every item (k1_f32.cu)
    const double cq = __longlong_as_double((long long)*q_cmax_bits);
    if ((*q_flags & 3) != 0 || !k1f_launch_ok(db_cmax > cq ? db_cmax : cq, d2)) return;
    __shared__ unsigned long long red[4];
    for (int64_t b = blockIdx.x; b < p.nb; b += gridDim.x) {
        const int64_t f = p.first[b], l = p.last[b];
        unsigned long long cnt = 0;
        if (f >= 0) {
            for (int64_t q = p.lo[b] + threadIdx.x; q <= p.hi[b]; q += blockDim.x) {
                const double te_q = qte[q], ts_q = qts[q];
                int64_t a = f, z = l + 1;  // first e with ts_e > te_q
                while (a < z) {
                    const int64_t m = (a + z) >> 1;
                    if (ets[m] <= te_q) a = m + 1;
                    else z = m;
                }
                const int64_t c1 = a - f;
                a = f;
                z = l + 1;  // first e with te_e >= ts_q
                while (a < z) {
                    const int64_t m = (a + z) >> 1;
                    if (ete[m] < ts_q) a = m + 1;
                    else z = m;
                }
                cnt += (unsigned long long)(c1 - (a - f));
            }
        }
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned long long t = red[0] + red[1] + red[2] + red[3];
            if (t) atomicAdd(&p.ovl[b], t);
        }
        __syncthreads();
    }
}

void launch_count_overlaps_ext(const SearchPlanDev &p, const Soa &q, const Soa &s, const int *q_flags,
                               const unsigned long long *q_cmax_bits, double db_cmax, double d2, cudaStream_t st) {
    const int grid = (int)std::min<int64_t>(p.nb, 148 * 16);
    k_count_overlaps_ext<<<grid, 128, 0, st>>>(p, q.ts, q.te, s.ts, s.te, q_flags, q_cmax_bits, db_cmax, d2);
    TSK_CUDA(cudaGetLastError());
}

void free_k1_layout(tsk_db *db) {
    K1Layout &k = db->k;
    k.s.storage.release(db->stream);
    k.aux.release(db->stream);
    k.orig = nullptr;
    k.box = nullptr;
    k.gtime = nullptr;
    k.frec = nullptr;
    k.gorig = nullptr;
    k.ngroups = 0;
    k.built = false;
}

static bool spatial_enabled() {
    const char *e = getenv("TSK_SPATIAL");
    return !(e && (!strcmp(e, "off") || !strcmp(e, "0")));
}

void build_k1_layout(tsk_db *db, cudaStream_t st) {
    K1Layout &k = db->k;
    k.built = false;
    const Soa &s = db->s;
    const int64_t n = s.n;
    if (!spatial_enabled() || n < 2 * BOX_GROUP || !db->ix.built) {
        free_k1_layout(db);
        return;
    }
    const Index &ix = db->ix;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
    // Morton frame over the midpoints' bounding box
    unsigned long long hb[6];
    {
        unsigned long long *d;
        TSK_CUDA(cudaMallocAsync(&d, 48, st));
        unsigned long long init[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
        TSK_CUDA(cudaMemcpyAsync(d, init, 48, cudaMemcpyHostToDevice, st));
        k_mid_box<<<grid, 256, 0, st>>>(n, s.sx, s.sy, s.sz, s.ex, s.ey, s.ez, d);
        TSK_CUDA(cudaGetLastError());
        TSK_CUDA(cudaMemcpyAsync(hb, d, 48, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaFreeAsync(d, st));
        TSK_CUDA(cudaStreamSynchronize(st));
    }
    MortonFrame fr;
    for (int c = 0; c < 3; ++c) {
        const double lo = ord_value(hb[c]), hi = ord_value(hb[3 + c]);
        fr.lo[c] = std::isfinite(lo) ? lo : 0.0;
        const double ext = hi - lo;
        fr.scale[c] = (std::isfinite(ext) && ext > 0.0) ? 1024.0 / ext : 0.0;
    }
    // keys (bin, code) and the stable sort
    uint64_t *k0, *k1;
    int64_t *v0, *v1;
    const size_t nb8 = (size_t)n * 8;
    TSK_CUDA(cudaMallocAsync(&k0, nb8, st));
    TSK_CUDA(cudaMallocAsync(&k1, nb8, st));
    TSK_CUDA(cudaMallocAsync(&v0, nb8, st));
    TSK_CUDA(cudaMallocAsync(&v1, nb8, st));
    k_layout_keys<<<grid, 256, 0, st>>>(n, s.ts, s.sx, s.sy, s.sz, s.ex, s.ey, s.ez, ix.t0, ix.width, ix.m, fr, k0,
                                        v0);
    TSK_CUDA(cudaGetLastError());
    int end_bit = 30;
    while (end_bit < 64 && (int64_t(1) << (end_bit - 30)) < ix.m) ++end_bit;
    size_t tb = 0;
    TSK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, n, 0, end_bit, st));
    void *tmp;
    TSK_CUDA(cudaMallocAsync(&tmp, tb, st));
    TSK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, end_bit, st));
    TSK_CUDA(cudaFreeAsync(tmp, st));
    TSK_CUDA(cudaFreeAsync(k0, st));
    TSK_CUDA(cudaFreeAsync(k1, st));
    TSK_CUDA(cudaFreeAsync(v0, st));
    // the reordered columns (no id columns: ids are gathered by start-sorted ordinal)
    soa_alloc(k.s, n, false, st);
    k.ngroups = (n + BOX_GROUP - 1) / BOX_GROUP;
    k.aux.reserve(nb8 + (size_t)k.ngroups * (2 * sizeof(float4) + sizeof(double2) + sizeof(double4)) +
                      (size_t)n * 2 * sizeof(float4) + 128,
                  st);
    k.orig = k.aux.as<int64_t>();
    k.box = reinterpret_cast<float4 *>(k.aux.as<char>() + ((nb8 + 31) & ~size_t(31)));
    k.gtime = reinterpret_cast<double2 *>(k.box + 2 * k.ngroups);
    k.gorig = reinterpret_cast<double4 *>(k.gtime + k.ngroups + (k.ngroups & 1));  // 32-byte aligned
    k.frec = reinterpret_cast<float4 *>(k.gorig + k.ngroups);
    k_layout_gather<<<grid, 256, 0, st>>>(n, v1, s, k.s, k.orig);
    TSK_CUDA(cudaGetLastError());
    TSK_CUDA(cudaFreeAsync(v1, st));
    soa_group_bounds(k.s, st);
    const int gg = (int)std::min<int64_t>((k.ngroups * 32 + 255) / 256, 148 * 16);
    k_group_boxes<<<gg, 256, 0, st>>>(n, k.s, k.box, k.gtime);
    TSK_CUDA(cudaGetLastError());
    k_f32_records<<<grid, 256, 0, st>>>(n, k.s, k.frec, k.gorig);
    TSK_CUDA(cudaGetLastError());
    k.s.any_unsafe = s.any_unsafe;
    k.s.sorted = 0;
    k.s.te_sorted = 0;
    TSK_CUDA(cudaStreamSynchronize(st));
    k.built = true;
}

}  // namespace tsk
