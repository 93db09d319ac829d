// db.cu — device-resident segment store, temporal index (K2) and candidate
// ranges (K3).
//
//   SegmentStore residency ........ /root/reference/pkg/src/trajseek/core.py:121-243
//   stable start-time sort ........ core.py:162-166
//   build_index ................... index.py:85-146          (K2)
//   candidate_range ............... index.py:149-173         (K3)
//   batch extent (range_extent) ... core.py:239-243, engine.py:177-179
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>

#include "filter.cuh"
#include "tsk_internal.cuh"

namespace tsk {

void DBuf::reserve(size_t need, cudaStream_t) {
    if (need <= bytes) return;
    if (p) TSK_CUDA(cudaFree(p));
    p = nullptr;
    bytes = 0;
    size_t want = need + need / 4 + 256;
    TSK_CUDA(cudaMalloc(&p, want));
    bytes = want;
}

void DBuf::release(cudaStream_t) {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

// ── SoA storage ────────────────────────────────────────────────────────────

void soa_alloc(Soa &s, int64_t n, bool with_ids, cudaStream_t st) {
    size_t nn = (size_t)(n > 0 ? n : 1);
    size_t per = 15 * sizeof(double) + (with_ids ? 2 * sizeof(int64_t) : 0) + sizeof(float) + 1;
    const size_t ngb = (nn + GB_SIZE - 1) / GB_SIZE;
    s.storage.reserve(nn * per + ngb * sizeof(GBound) + 64, st);
    char *base = s.storage.as<char>();
    double **cols[15] = {&s.ts, &s.te, &s.sx, &s.sy, &s.sz, &s.ex, &s.ey, &s.ez,
                         &s.dx, &s.dy, &s.dz, &s.rcp, &s.vx, &s.vy, &s.vz};
    for (int k = 0; k < 15; ++k) {
        *cols[k] = reinterpret_cast<double *>(base);
        base += nn * sizeof(double);
    }
    if (with_ids) {
        s.traj = reinterpret_cast<int64_t *>(base);
        base += nn * sizeof(int64_t);
        s.seg = reinterpret_cast<int64_t *>(base);
        base += nn * sizeof(int64_t);
    } else {
        s.traj = s.seg = nullptr;
    }
    s.sr32 = reinterpret_cast<float *>(base);
    base += nn * sizeof(float);
    s.unsafe = reinterpret_cast<uint8_t *>(base);
    base += nn;
    // group bounds after the byte column, 16-byte aligned
    base = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(base) + 15) & ~uintptr_t(15));
    s.gb = reinterpret_cast<GBound *>(base);
    s.n = n;
}

void soa_upload(Soa &s, const tsk_columns *c, cudaStream_t st) {
    size_t b = (size_t)c->n * sizeof(double);
    if (c->n == 0) return;
    const double *src[8] = {c->ts, c->te, c->xs, c->ys, c->zs, c->xe, c->ye, c->ze};
    double *dst[8] = {s.ts, s.te, s.sx, s.sy, s.sz, s.ex, s.ey, s.ez};
    for (int k = 0; k < 8; ++k) TSK_CUDA(cudaMemcpyAsync(dst[k], src[k], b, cudaMemcpyHostToDevice, st));
    if (s.traj) {
        TSK_CUDA(cudaMemcpyAsync(s.traj, c->traj, (size_t)c->n * 8, cudaMemcpyHostToDevice, st));
        TSK_CUDA(cudaMemcpyAsync(s.seg, c->seg, (size_t)c->n * 8, cudaMemcpyHostToDevice, st));
    }
}

// Exponent window inside which qdiv() is proven exact and K1's filter
// bound holds (filter.cuh): times and extents 0 or of magnitude in
// [2^-900, 2^1000], coordinates of magnitude <= 2^1000, velocity components
// 0 or of magnitude in [2^-1000, 2^1000].  NaN fails every test.  Unsafe
// segments send their K1 tiles to the exact IEEE path.
__device__ __forceinline__ bool mag_ok(double v) {
    const double a = fabs(v);
    return a == 0.0 || (a >= 0x1p-900 && a <= 0x1p1000);
}
__device__ __forceinline__ bool coord_ok(double v) { return fabs(v) <= 0x1p1000; }
__device__ __forceinline__ bool vel_ok(double v) {
    const double a = fabs(v);
    return a == 0.0 || (a >= 0x1p-1000 && a <= 0x1p1000);
}

struct SegHoist {
    double ext, rcp, d[3], v[3];
    bool unsafe;
};

__device__ __forceinline__ SegHoist seg_hoist(double t0, double t1, const double s[3], const double e[3]) {
    SegHoist h;
    h.ext = __dsub_rn(t1, t0);
    h.rcp = h.ext > 0.0 ? __drcp_rn(h.ext) : 0.0;
    bool ok = mag_ok(t0) && mag_ok(t1) && mag_ok(h.ext);
    for (int i = 0; i < 3; ++i) {
        h.d[i] = __dsub_rn(e[i], s[i]);
        h.v[i] = __dmul_rn(h.d[i], h.rcp);  // seg_velocity (filter.cuh)
        ok = ok && coord_ok(s[i]) && coord_ok(e[i]) && vel_ok(h.v[i]);
    }
    h.unsafe = !ok;
    return h;
}

__global__ void k_hoist(int64_t n, const double *__restrict__ ts, const double *__restrict__ te,
                        const double *__restrict__ sx, const double *__restrict__ sy,
                        const double *__restrict__ sz, const double *__restrict__ ex,
                        const double *__restrict__ ey, const double *__restrict__ ez,
                        double *__restrict__ dx, double *__restrict__ dy, double *__restrict__ dz,
                        double *__restrict__ rcp, double *__restrict__ vx, double *__restrict__ vy,
                        double *__restrict__ vz, float *__restrict__ sr32, uint8_t *__restrict__ unsafe,
                        int *flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double t0 = ts[i];
        const double s[3] = {sx[i], sy[i], sz[i]}, e[3] = {ex[i], ey[i], ez[i]};
        const SegHoist h = seg_hoist(t0, te[i], s, e);
        dx[i] = h.d[0]; dy[i] = h.d[1]; dz[i] = h.d[2];
        vx[i] = h.v[0]; vy[i] = h.v[1]; vz[i] = h.v[2];
        sr32[i] = f32_speed(h.v[0], h.v[1], h.v[2]);
        rcp[i] = h.rcp;
        unsafe[i] = h.unsafe ? 1 : 0;
        if (h.unsafe) atomicOr(&flags[0], 1);
        if (i + 1 < n && ts[i + 1] < t0) atomicOr(&flags[1], 1);
        if (i + 1 < n && te[i + 1] < te[i]) atomicOr(&flags[1], 2);
    }
}

void soa_hoist(Soa &s, cudaStream_t st) {
    if (s.n == 0) {
        s.any_unsafe = 0;
        s.sorted = 1;
        return;
    }
    int *flags;
    TSK_CUDA(cudaMallocAsync(&flags, 2 * sizeof(int), st));
    TSK_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st));
    int grid = (int)std::min<int64_t>((s.n + 255) / 256, 148 * 16);
    k_hoist<<<grid, 256, 0, st>>>(s.n, s.ts, s.te, s.sx, s.sy, s.sz, s.ex, s.ey, s.ez, s.dx, s.dy,
                                  s.dz, s.rcp, s.vx, s.vy, s.vz, s.sr32, s.unsafe, flags);
    TSK_CUDA(cudaGetLastError());
    int h[2];
    TSK_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, st));
    TSK_CUDA(cudaFreeAsync(flags, st));
    TSK_CUDA(cudaStreamSynchronize(st));
    s.any_unsafe = h[0];
    s.sorted = (h[1] & 1) ? 0 : 1;
    s.te_sorted = (h[1] & 2) ? 0 : 1;
}

// Group bounds (GBound): one warp per group of GB_SIZE segments.
__global__ void k_group_bounds(int64_t n, const double *__restrict__ ts, const double *__restrict__ sx,
                               const double *__restrict__ sy, const double *__restrict__ sz,
                               const double *__restrict__ vx, const double *__restrict__ vy,
                               const double *__restrict__ vz, GBound *__restrict__ gb) {
    const int lane = threadIdx.x & 31;
    const int64_t ngb = (n + GB_SIZE - 1) / GB_SIZE;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < ngb;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        double tlo = INFINITY, thi = -INFINITY, vm = 0.0;
        for (int k = lane; k < GB_SIZE; k += 32) {
            const int64_t i = g * GB_SIZE + k;
            if (i >= n) break;
            const double s3[3] = {sx[i], sy[i], sz[i]};
            for (int c = 0; c < 3; ++c) {
                lo[c] = fmin(lo[c], s3[c]);
                hi[c] = fmax(hi[c], s3[c]);
            }
            tlo = fmin(tlo, ts[i]);
            thi = fmax(thi, ts[i]);
            vm = fmax(vm, fmax(fabs(vx[i]), fmax(fabs(vy[i]), fabs(vz[i]))));
        }
        for (int o = 16; o; o >>= 1) {
            for (int c = 0; c < 3; ++c) {
                lo[c] = fmin(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
                hi[c] = fmax(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
            }
            tlo = fmin(tlo, __shfl_xor_sync(0xffffffffu, tlo, o));
            thi = fmax(thi, __shfl_xor_sync(0xffffffffu, thi, o));
            vm = fmax(vm, __shfl_xor_sync(0xffffffffu, vm, o));
        }
        if (lane == 0) {
            GBound b;
            for (int c = 0; c < 3; ++c) {
                b.lo[c] = lo[c];
                b.hi[c] = hi[c];
            }
            b.ts_lo = tlo;
            b.ts_hi = thi;
            b.vmax = vm;
            b.pad = 0.0;
            gb[g] = b;
        }
    }
}

void soa_group_bounds(Soa &s, cudaStream_t st) {
    if (s.n == 0) return;
    const int64_t ngb = (s.n + GB_SIZE - 1) / GB_SIZE;
    int grid = (int)std::min<int64_t>((ngb + 7) / 8, 148 * 16);
    k_group_bounds<<<grid, 256, 0, st>>>(s.n, s.ts, s.sx, s.sy, s.sz, s.vx, s.vy, s.vz, s.gb);
    TSK_CUDA(cudaGetLastError());
}

// max |coordinate| over the six position columns (filter margin of K1)
__global__ void k_cmax(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                       const double *__restrict__ c, const double *__restrict__ d,
                       const double *__restrict__ e, const double *__restrict__ f,
                       unsigned long long *out) {
    double cm = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        cm = fmax(cm, fmax(fmax(fabs(a[i]), fabs(b[i])), fmax(fmax(fabs(c[i]), fabs(d[i])),
                                                              fmax(fabs(e[i]), fabs(f[i])))));
    for (int o = 16; o; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(cm));
}

double soa_cmax(const Soa &s, cudaStream_t st) {
    if (s.n == 0) return 0.0;
    unsigned long long *d;
    TSK_CUDA(cudaMallocAsync(&d, 8, st));
    TSK_CUDA(cudaMemsetAsync(d, 0, 8, st));
    int grid = (int)std::min<int64_t>((s.n + 255) / 256, 148 * 16);
    k_cmax<<<grid, 256, 0, st>>>(s.n, s.sx, s.sy, s.sz, s.ex, s.ey, s.ez, d);
    TSK_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    TSK_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
    TSK_CUDA(cudaFreeAsync(d, st));
    TSK_CUDA(cudaStreamSynchronize(st));
    double v;
    memcpy(&v, &h, 8);
    return v;
}

// 1 when every entry id (traj, seg) fits in int32: results then cross PCIe
// with 4-byte entry ids, widened on the host (search.cu)
__global__ void k_ids32(int64_t n, const int64_t *__restrict__ traj, const int64_t *__restrict__ seg, int *ok) {
    bool fit = true;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        fit = fit && traj[i] == (int64_t)(int32_t)traj[i] && seg[i] == (int64_t)(int32_t)seg[i];
    if (!__all_sync(0xffffffffu, fit) && (threadIdx.x & 31) == 0) atomicAnd(ok, 0);
}

int soa_ids32(const Soa &s, cudaStream_t st) {
    if (s.n == 0) return 1;
    int *d;
    TSK_CUDA(cudaMallocAsync(&d, 4, st));
    const int one = 1;
    TSK_CUDA(cudaMemcpyAsync(d, &one, 4, cudaMemcpyHostToDevice, st));
    int grid = (int)std::min<int64_t>((s.n + 255) / 256, 148 * 16);
    k_ids32<<<grid, 256, 0, st>>>(s.n, s.traj, s.seg, d);
    TSK_CUDA(cudaGetLastError());
    int h = 0;
    TSK_CUDA(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, st));
    TSK_CUDA(cudaFreeAsync(d, st));
    TSK_CUDA(cudaStreamSynchronize(st));
    return h;
}

// ── queries → shared-memory records ────────────────────────────────────────

// Queries: hoisted invariants straight into the shared-memory records (one
// pass, no host sync); flags[0] |= 1 when the start times are not sorted
// (the pair kernel then disables its windows).
__global__ void k_qprep(int64_t n, const double *__restrict__ ts, const double *__restrict__ te,
                        const double *__restrict__ sx, const double *__restrict__ sy,
                        const double *__restrict__ sz, const double *__restrict__ ex,
                        const double *__restrict__ ey, const double *__restrict__ ez,
                        QRec *__restrict__ out, int *flags, unsigned long long *cmax_bits) {
    double cm = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        QRec r;
        r.ts = ts[i];
        r.te = te[i];
        r.sx = sx[i];
        r.sy = sy[i];
        r.sz = sz[i];
        r.ex = ex[i];
        r.ey = ey[i];
        r.ez = ez[i];
        const double s[3] = {r.sx, r.sy, r.sz}, e[3] = {r.ex, r.ey, r.ez};
        const SegHoist h = seg_hoist(r.ts, r.te, s, e);
        r.ext = h.ext;
        r.dx = h.d[0]; r.dy = h.d[1]; r.dz = h.d[2];
        r.vx = h.v[0]; r.vy = h.v[1]; r.vz = h.v[2];
        r.flag = h.unsafe ? 1.0 : 0.0;
        out[i] = r;
        if (i + 1 < n && ts[i + 1] < r.ts) atomicOr(&flags[0], 1);
        if (i + 1 < n && te[i + 1] < r.te) atomicOr(&flags[0], 2);
        cm = fmax(cm, fmax(fmax(fabs(r.sx), fabs(r.sy)), fmax(fabs(r.sz), fmax(fabs(r.ex), fmax(fabs(r.ey), fabs(r.ez))))));
    }
    for (int o = 16; o; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    // non-negative doubles order like their bit patterns
    if ((threadIdx.x & 31) == 0) atomicMax(cmax_bits, (unsigned long long)__double_as_longlong(cm));
}

// Pinned (device-mapped) query columns: read them straight from host memory
// over PCIe in one kernel — the H2D transfer and the record build fused —
// writing the device copies of ts/te/traj/seg that K3 and K4 read.
__global__ void k_qprep_mapped(int64_t n, tsk_columns c, double *__restrict__ ts_out, double *__restrict__ te_out,
                               int64_t *__restrict__ traj_out, int64_t *__restrict__ seg_out,
                               QRec *__restrict__ out, int *flags, unsigned long long *cmax_bits) {
    double cm = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        QRec r;
        r.ts = c.ts[i];
        r.te = c.te[i];
        r.sx = c.xs[i];
        r.sy = c.ys[i];
        r.sz = c.zs[i];
        r.ex = c.xe[i];
        r.ey = c.ye[i];
        r.ez = c.ze[i];
        ts_out[i] = r.ts;
        te_out[i] = r.te;
        traj_out[i] = c.traj[i];
        seg_out[i] = c.seg[i];
        const double s[3] = {r.sx, r.sy, r.sz}, e[3] = {r.ex, r.ey, r.ez};
        const SegHoist h = seg_hoist(r.ts, r.te, s, e);
        r.ext = h.ext;
        r.dx = h.d[0]; r.dy = h.d[1]; r.dz = h.d[2];
        r.vx = h.v[0]; r.vy = h.v[1]; r.vz = h.v[2];
        r.flag = h.unsafe ? 1.0 : 0.0;
        out[i] = r;
        // the next query's times from the neighbouring lane (only the last
        // lane re-reads host memory: every column crosses PCIe once)
        const unsigned act = __activemask();
        const int lane = threadIdx.x & 31;
        double nts = __shfl_down_sync(act, r.ts, 1), nte = __shfl_down_sync(act, r.te, 1);
        const bool last = lane == 31 || !((act >> (lane + 1)) & 1u);
        if (last && i + 1 < n) {
            nts = c.ts[i + 1];
            nte = c.te[i + 1];
        }
        if (i + 1 < n && nts < r.ts) atomicOr(&flags[0], 1);
        if (i + 1 < n && nte < r.te) atomicOr(&flags[0], 2);
        cm = fmax(cm, fmax(fmax(fabs(r.sx), fabs(r.sy)), fmax(fabs(r.sz), fmax(fabs(r.ex), fmax(fabs(r.ey), fabs(r.ez))))));
    }
    for (int o = 16; o; o >>= 1) cm = fmax(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    if ((threadIdx.x & 31) == 0) atomicMax(cmax_bits, (unsigned long long)__double_as_longlong(cm));
}

// The device pointers of ten query columns when every one is pinned and
// mapped into the device address space; false otherwise.
bool mapped_columns(const tsk_columns *c, tsk_columns *dev) {
    const void *src[10] = {c->traj, c->seg, c->xs, c->ys, c->zs, c->ts, c->xe, c->ye, c->ze, c->te};
    const void *dst[10];
    for (int k = 0; k < 10; ++k) {
        cudaPointerAttributes a;
        if (!src[k] || cudaPointerGetAttributes(&a, src[k]) != cudaSuccess || a.type != cudaMemoryTypeHost ||
            !a.devicePointer) {
            cudaGetLastError();
            return false;
        }
        dst[k] = a.devicePointer;
    }
    *dev = *c;
    dev->traj = (const int64_t *)dst[0];
    dev->seg = (const int64_t *)dst[1];
    dev->xs = (const double *)dst[2];
    dev->ys = (const double *)dst[3];
    dev->zs = (const double *)dst[4];
    dev->ts = (const double *)dst[5];
    dev->xe = (const double *)dst[6];
    dev->ye = (const double *)dst[7];
    dev->ze = (const double *)dst[8];
    dev->te = (const double *)dst[9];
    return true;
}

void launch_qprep_mapped(const tsk_columns &dev_cols, Soa &q, QRec *out, int *flags, unsigned long long *cmax_bits,
                         cudaStream_t st) {
    TSK_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), st));
    TSK_CUDA(cudaMemsetAsync(cmax_bits, 0, sizeof(unsigned long long), st));
    if (q.n == 0) return;
    int grid = (int)std::min<int64_t>((q.n + 255) / 256, 148 * 8);
    k_qprep_mapped<<<grid, 256, 0, st>>>(q.n, dev_cols, q.ts, q.te, q.traj, q.seg, out, flags, cmax_bits);
    TSK_CUDA(cudaGetLastError());
}

void launch_qprep(const Soa &q, QRec *out, int *flags, unsigned long long *cmax_bits, cudaStream_t st) {
    TSK_CUDA(cudaMemsetAsync(flags, 0, sizeof(int), st));
    TSK_CUDA(cudaMemsetAsync(cmax_bits, 0, sizeof(unsigned long long), st));
    if (q.n == 0) return;
    int grid = (int)std::min<int64_t>((q.n + 255) / 256, 148 * 8);
    k_qprep<<<grid, 256, 0, st>>>(q.n, q.ts, q.te, q.sx, q.sy, q.sz, q.ex, q.ey, q.ez, out, flags,
                                  cmax_bits);
    TSK_CUDA(cudaGetLastError());
}

// ── stable sort by start time ──────────────────────────────────────────────

// Order-preserving map of a double onto uint64 (+0.0 and -0.0 share a key,
// as they compare equal in numpy's stable argsort).
__global__ void k_sortkey(int64_t n, const double *__restrict__ ts, uint64_t *__restrict__ key,
                          int64_t *__restrict__ iota) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v = ts[i];
        if (v == 0.0) v = 0.0;
        uint64_t b = (uint64_t)__double_as_longlong(v);
        key[i] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
        iota[i] = i;
    }
}

}  // namespace tsk

using namespace tsk;

// ── index build (K2) ───────────────────────────────────────────────────────

namespace tsk {


// Runs of equal bin id are contiguous because ts is sorted; record the
// first/last ordinal of each run (the searchsorted pair of index.py:116-118).
__global__ void k_bin_bounds(int64_t n, const double *__restrict__ ts, double t0, double width,
                             int64_t m, int64_t *__restrict__ first, int64_t *__restrict__ last) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t b = bin_of(ts[i], t0, width, m);
        if (i == 0 || bin_of(ts[i - 1], t0, width, m) != b) first[b] = i;
        if (i == n - 1 || bin_of(ts[i + 1], t0, width, m) != b) last[b] = i;
    }
}

__global__ void k_bin_flags(int64_t m, const int64_t *__restrict__ first, int64_t *__restrict__ flag) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x)
        flag[j] = first[j] >= 0 ? 1 : 0;
}

__global__ void k_bin_compact(int64_t m, const int64_t *__restrict__ first,
                              const int64_t *__restrict__ last, const int64_t *__restrict__ pos,
                              const double *__restrict__ ts, int rule, double t0, double width,
                              double *__restrict__ ne_start, int64_t *__restrict__ ne_first,
                              int64_t *__restrict__ ne_last, int64_t *__restrict__ ne_bin) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
         j += (int64_t)gridDim.x * blockDim.x) {
        int64_t f = first[j];
        if (f < 0) continue;
        int64_t k = pos[j];
        ne_first[k] = f;
        ne_last[k] = last[j];
        ne_bin[k] = j;
        // member_extents: ts[first]; grid_start: t0 + j * width (index.py:123-126)
        ne_start[k] = rule == TSK_EXTENT_MEMBER ? ts[f] : __dadd_rn(t0, __dmul_rn((double)j, width));
    }
}

// ne_end = max te over the bin's members (maximum.reduceat, index.py:127); one warp per bin.
__global__ void k_bin_end(int64_t n_ne, const int64_t *__restrict__ ne_first,
                          const int64_t *__restrict__ ne_last, const double *__restrict__ te,
                          double *__restrict__ ne_end) {
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = warp; k < n_ne; k += nw) {
        double mx = -INFINITY;
        for (int64_t i = ne_first[k] + lane; i <= ne_last[k]; i += 32) mx = fmax(mx, te[i]);
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) ne_end[k] = mx;
    }
}

struct MaxOp {
    __device__ __forceinline__ double operator()(double a, double b) const { return a > b ? a : b; }
};

// ── candidate ranges (K3) ──────────────────────────────────────────────────

// For [begin, end]: hi = searchsorted(ne_start, end, "right"); the lowest
// reaching bin is the first k < hi whose running max of ne_end reaches
// begin; the highest is found by a backward warp scan (index.py:160-173).
__device__ void range_lookup(double begin, double end, int64_t n_ne, const double *ne_start,
                             const double *ne_end, const double *ne_endmax, const int64_t *ne_first,
                             const int64_t *ne_last, int64_t *out_first, int64_t *out_last) {
    int lane = threadIdx.x & 31;
    int64_t lo = 0, hi = n_ne;  // upper_bound on ne_start
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ne_start[mid] <= end) lo = mid + 1;
        else hi = mid;
    }
    int64_t h = lo;
    int64_t rf = -1, rl = -1;
    if (h > 0) {
        int64_t a = 0, b = h;  // lower_bound on the running max
        while (a < b) {
            int64_t mid = (a + b) >> 1;
            if (ne_endmax[mid] >= begin) b = mid;
            else a = mid + 1;
        }
        int64_t klo = a;
        if (klo < h) {
            int64_t khi = -1;
            for (int64_t base = h - 1; base >= klo && khi < 0; base -= 32) {
                int64_t k = base - lane;
                bool reach = k >= klo && ne_end[k] >= begin;
                unsigned m = __ballot_sync(0xffffffffu, reach);
                if (m) khi = base - (__ffs(m) - 1);
            }
            rf = ne_first[klo];
            rl = ne_last[khi];
        }
    }
    if (lane == 0) {
        *out_first = rf;
        *out_last = rl;
    }
}

__global__ void k_ranges_given(int64_t k, const double *__restrict__ begin,
                               const double *__restrict__ end, Index ix, int64_t *first,
                               int64_t *last) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = warp; i < k; i += nw)
        range_lookup(begin[i], end[i], ix.n_ne, ix.ne_start, ix.ne_end, ix.ne_endmax, ix.ne_first,
                     ix.ne_last, first + i, last + i);
}

// One warp per batch: extent [ts[lo], max te[lo..hi]] then the range lookup.
__global__ void k_batch_ranges(int64_t nb, const int64_t *__restrict__ lo, const int64_t *__restrict__ hi,
                               const double *__restrict__ qts, const double *__restrict__ qte,
                               Index ix, int64_t *first, int64_t *last) {
    int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = warp; b < nb; b += nw) {
        double mx = -INFINITY;
        for (int64_t i = lo[b] + lane; i <= hi[b]; i += 32) mx = fmax(mx, qte[i]);
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (ix.n_ne == 0) {
            if (lane == 0) first[b] = last[b] = -1;
            continue;
        }
        range_lookup(qts[lo[b]], mx, ix.n_ne, ix.ne_start, ix.ne_end, ix.ne_endmax, ix.ne_first,
                     ix.ne_last, first + b, last + b);
    }
}

void launch_ranges(tsk_db *db, const Soa &q, SearchPlanDev &p, bool spans_given, cudaStream_t st) {
    if (spans_given || p.nb == 0) return;
    TSK_REQUIRE(db->ix.built, "run_search needs an index: call build_index first");
    int grid = (int)std::min<int64_t>((p.nb * 32 + 255) / 256, 148 * 8);
    k_batch_ranges<<<grid, 256, 0, st>>>(p.nb, p.lo, p.hi, q.ts, q.te, db->ix, p.first, p.last);
    TSK_CUDA(cudaGetLastError());
}

// ── work items of a plan ───────────────────────────────────────────────────

// Single block: choose the query tile and the candidate sub-tile count so
// the grid gets at least ~4 waves of items, then count items per work unit
// (plan_unit: batch pairs sharing candidates, and the rest) and scan them.
__global__ void __launch_bounds__(1024, 1) k_plan_items(SearchPlanDev p, int64_t slots, int stride, int pair,
                                                         int align, int tq_max, const int *q_flags) {
    typedef cub::BlockReduce<long long, 1024> BR;
    typedef cub::BlockScan<long long, 1024> BS;
    __shared__ union {
        typename BR::TempStorage r;
        typename BS::TempStorage s;
    } tmp;
    __shared__ long long carry, tiles_sh;
    __shared__ int sub_sh;
    const int64_t nb = p.nb;
    // query tile: tq_max (the kernel's), halved (down to 32) while the grid would get fewer
    // than 4 waves of single-batch items — small plans otherwise under-fill
    // 148 SMs
    const long long want = 4 * slots;
    int tqs = tq_max;
    for (;;) {  // pair == 2 / 5 / 9 (testing): full tiles, always pairs / quads / octets
        long long acc = 0;
        for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
            long long c = p.first[b] >= 0 ? p.last[b] - p.first[b] + 1 : 0;
            long long tq = (p.hi[b] - p.lo[b] + 1 + tqs - 1) / tqs;
            acc += ((c + stride - 1) / stride) * tq;
        }
        long long tiles = BR(tmp.r).Sum(acc);
        if (threadIdx.x == 0) tiles_sh = tiles;
        __syncthreads();
        tiles = tiles_sh;
        __syncthreads();
        if (tiles >= want || tqs <= 32 || pair == 2 || pair == 5 || pair == 9) break;
        tqs >>= 1;
    }
    if (threadIdx.x == 0) {
        // candidate sub-tiles per item: as many as keep >= 8 items per slot
        // (fewer, longer items amortise the per-item set-up; the last items
        // bound the tail)
        int sub = (int)(tiles_sh / (2 * want > 0 ? 2 * want : 1));
        sub_sh = sub < 1 ? 1 : (sub > K1_MAX_SUB ? K1_MAX_SUB : sub);
        carry = 0;
    }
    __syncthreads();
    // sharing only when the plan is big enough to fill the grid with full
    // tiles: quads (pair == 4) when the kernel's box-cull fast path takes
    // every item — query start and end times both sorted (q_flags bits 0, 1
    // from the query kernel) — else pairs
    // (pair == 8 / 9: octets, the 1,024-query kernel; 9 forces them)
    const bool sorted_q = q_flags && (*q_flags & 3) == 0;
    const int group = pair >= 8 ? K1_SHARE_OCTETS : K1_SHARE_QUADS;
    int mode = K1_SHARE_NONE;
    if (pair == 2) mode = K1_SHARE_PAIRS;  // testing: forced, full tiles
    else if (pair == 5 || pair == 9) mode = sorted_q ? group : K1_SHARE_PAIRS;
    else if (pair && tqs == tq_max)
        mode = ((pair == 4 || pair == 8) && sorted_q) ? group : K1_SHARE_PAIRS;
    const int pr = mode;
    const long long ct = (long long)stride * sub_sh;
    const int64_t nu = plan_units_mode(nb, mode);
    for (int64_t base = 0; base < nu; base += blockDim.x) {
        int64_t u = base + threadIdx.x;
        long long v = 0;
        if (u < nu) {
            const UnitT<K1_UNIT_GMAX> U = plan_unit<K1_UNIT_GMAX, false>(p, u, tqs, pr);
            if (U.f <= U.l) {
                // candidate tiles start at a multiple of `align` (K1 layout:
                // warps then coincide with the box groups; the head is masked)
                const long long c = U.l - (U.f / align) * align + 1;
                const long long tq = U.b1 >= 0 ? 1 : (U.s + tqs - 1) / tqs;
                v = ((c + ct - 1) / ct) * tq;
            }
        }
        long long ex, agg;
        BS(tmp.s).ExclusiveSum(v, ex, agg);
        if (u < nu) p.item_off[u] = carry + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry += agg;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        p.item_off[nu] = carry;
        p.meta[0] = carry;
        p.meta[1] = sub_sh;
        p.meta[2] = tqs;
        p.meta[3] = pr;
    }
}

void launch_plan_items(SearchPlanDev &p, int slots, int stride, int pair, int align, int tq_max, const int *q_flags,
                       cudaStream_t st) {
    k_plan_items<<<1, 1024, 0, st>>>(p, slots, stride, pair, align, tq_max, q_flags);
    TSK_CUDA(cudaGetLastError());
}

}  // namespace tsk

// ── C-ABI: db / sort / index / ranges ──────────────────────────────────────

// The work units of a plan in a sharing mode (host code: the same
// plan_unit the item planner and K1 decode run on the device; tests check
// that every (batch, candidate) pair lies in exactly one unit).  Per unit 13
// int64: b, b1, lo_q, s, js, jx[0..5], f, l.  Returns the unit count, or -1
// when `cap` units do not fit.
extern "C" int64_t tsk_plan_units(int64_t nb, const int64_t *lo, const int64_t *hi, const int64_t *first,
                                  const int64_t *last, int mode, int64_t tqs, int64_t *out, int64_t cap) {
    using namespace tsk;
    const int64_t nu = plan_units_mode(nb, mode);
    if (nb < 1 || !out || nu > cap) return -1;
    SearchPlanDev p{};
    p.nb = nb;
    p.lo = lo;
    p.hi = hi;
    p.first = const_cast<int64_t *>(first);
    p.last = const_cast<int64_t *>(last);
    for (int64_t u = 0; u < nu; ++u) {
        const UnitT<K1_UNIT_GMAX> U = plan_unit<K1_UNIT_GMAX, false>(p, u, tqs, mode);
        int64_t *o = out + 13 * u;
        o[0] = U.b;
        o[1] = U.b1;
        o[2] = U.lo_q;
        o[3] = U.s;
        o[4] = U.js;
        for (int i = 0; i < K1_UNIT_GMAX - 2; ++i) o[5 + i] = U.jx[i];
        o[11] = U.f;
        o[12] = U.l;
    }
    return nu;
}

extern "C" int tsk_db_create(int device, const tsk_columns *cols, tsk_db **out) {
    tsk_db *db = nullptr;
    try {
        TSK_REQUIRE(cols && out, "null argument");
        TSK_REQUIRE(cols->n >= 0, "negative store size");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error{TSK_ENODEV, "no CUDA device visible"};
        TSK_REQUIRE(device >= 0 && device < ndev, "device ordinal out of range");
        TSK_CUDA(cudaSetDevice(device));
        db = new tsk_db();
        db->device = device;
        TSK_CUDA(cudaStreamCreateWithFlags(&db->stream, cudaStreamNonBlocking));
        TSK_CUDA(cudaEventCreate(&db->ev0));
        TSK_CUDA(cudaEventCreate(&db->ev1));
        TSK_CUDA(cudaEventCreate(&db->ev_k0));
        TSK_CUDA(cudaEventCreate(&db->ev_k1));
        soa_alloc(db->s, cols->n, true, db->stream);
        soa_upload(db->s, cols, db->stream);
        soa_hoist(db->s, db->stream);
        soa_group_bounds(db->s, db->stream);
        db->cmax = soa_cmax(db->s, db->stream);
        db->ids32 = soa_ids32(db->s, db->stream);
        *out = db;
        return TSK_OK;
    } catch (const Error &e) {
        if (db) tsk_db_free(db);
        return fail(e.code, e.msg);
    }
}

// Replica of a device store on another GPU (or another handle on the same
// one): the SoA block (columns, hoisted invariants, group bounds) is copied
// device to device — over NVLink when the GPUs are peers — instead of being
// re-uploaded from the host and re-hoisted.  The index is not copied; it is
// rebuilt on the replica by tsk_index_build (K2, milliseconds).
extern "C" int tsk_db_replicate(const tsk_db *src, int device, tsk_db **out) {
    tsk_db *db = nullptr;
    try {
        TSK_REQUIRE(src && out, "null argument");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error{TSK_ENODEV, "no CUDA device visible"};
        TSK_REQUIRE(device >= 0 && device < ndev, "device ordinal out of range");
        TSK_CUDA(cudaSetDevice(src->device));
        TSK_CUDA(cudaStreamSynchronize(src->stream));  // src fully built
        TSK_CUDA(cudaSetDevice(device));
        db = new tsk_db();
        db->device = device;
        TSK_CUDA(cudaStreamCreateWithFlags(&db->stream, cudaStreamNonBlocking));
        TSK_CUDA(cudaEventCreate(&db->ev0));
        TSK_CUDA(cudaEventCreate(&db->ev1));
        TSK_CUDA(cudaEventCreate(&db->ev_k0));
        TSK_CUDA(cudaEventCreate(&db->ev_k1));
        soa_alloc(db->s, src->s.n, true, db->stream);  // same layout as the source block
        if (src->s.n > 0) {
            const char *end = reinterpret_cast<const char *>(src->s.gb + (src->s.n + GB_SIZE - 1) / GB_SIZE);
            const size_t bytes = (size_t)(end - src->s.storage.as<char>());
            int can = 0;
            if (device != src->device && cudaDeviceCanAccessPeer(&can, device, src->device) == cudaSuccess && can) {
                const cudaError_t e = cudaDeviceEnablePeerAccess(src->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TSK_CUDA(e);
                cudaGetLastError();
            }
            TSK_CUDA(cudaMemcpyPeerAsync(db->s.storage.p, device, src->s.storage.p, src->device, bytes, db->stream));
        }
        db->s.any_unsafe = src->s.any_unsafe;
        db->s.sorted = src->s.sorted;
        db->s.te_sorted = src->s.te_sorted;
        db->cmax = src->cmax;
        db->ids32 = src->ids32;
        db->host_etraj = src->host_etraj;  // host ids are shared with the source
        db->host_eseg = src->host_eseg;
        TSK_CUDA(cudaStreamSynchronize(db->stream));
        *out = db;
        return TSK_OK;
    } catch (const Error &e) {
        if (db) tsk_db_free(db);
        return fail(e.code, e.msg);
    }
}

extern "C" void tsk_db_free(tsk_db *db) {
    if (!db) return;
    cudaSetDevice(db->device);
    if (db->stream) cudaStreamSynchronize(db->stream);
    db->s.storage.release(db->stream);
    db->ix.storage.release(db->stream);
    free_k1_layout(db);
    db->q.storage.release(db->stream);
    for (DBuf *b : {&db->q_rec, &db->batches, &db->counters, &db->recs, &db->sorted, &db->cub_tmp,
                    &db->out_cols, &db->canon_cols, &db->canon_tmp})
        b->release(db->stream);
    for (cudaEvent_t ev : {db->ev0, db->ev1, db->ev_k0, db->ev_k1})
        if (ev) cudaEventDestroy(ev);
    if (db->stream2) {
        cudaStreamSynchronize(db->stream2);
        cudaStreamDestroy(db->stream2);
    }
    if (db->stream) cudaStreamDestroy(db->stream);
    delete db;
}

extern "C" int64_t tsk_db_size(const tsk_db *db) { return db ? db->s.n : -1; }

extern "C" int tsk_sort_by_start(int device, int64_t n, const double *ts, int64_t *perm) {
    try {
        TSK_REQUIRE(n >= 0 && (n == 0 || (ts && perm)), "bad arguments");
        if (n == 0) return TSK_OK;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error{TSK_ENODEV, "no CUDA device visible"};
        TSK_CUDA(cudaSetDevice(device));
        cudaStream_t st;
        TSK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        double *dts;
        uint64_t *k0, *k1;
        int64_t *v0, *v1;
        size_t nb = (size_t)n * 8;
        TSK_CUDA(cudaMallocAsync(&dts, nb, st));
        TSK_CUDA(cudaMallocAsync(&k0, nb, st));
        TSK_CUDA(cudaMallocAsync(&k1, nb, st));
        TSK_CUDA(cudaMallocAsync(&v0, nb, st));
        TSK_CUDA(cudaMallocAsync(&v1, nb, st));
        TSK_CUDA(cudaMemcpyAsync(dts, ts, nb, cudaMemcpyHostToDevice, st));
        int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        k_sortkey<<<grid, 256, 0, st>>>(n, dts, k0, v0);
        TSK_CUDA(cudaGetLastError());
        size_t tb = 0;
        TSK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, n, 0, 64, st));
        void *tmp;
        TSK_CUDA(cudaMallocAsync(&tmp, tb, st));
        TSK_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, 64, st));
        TSK_CUDA(cudaMemcpyAsync(perm, v1, nb, cudaMemcpyDeviceToHost, st));
        for (void *p : {(void *)dts, (void *)k0, (void *)k1, (void *)v0, (void *)v1, tmp})
            TSK_CUDA(cudaFreeAsync(p, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        TSK_CUDA(cudaStreamDestroy(st));
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_index_build(tsk_db *db, int64_t m, int extent_rule, int64_t *n_nonempty,
                               double *hdr) {
    try {
        TSK_REQUIRE(db, "null db");
        TSK_REQUIRE(m >= 1, "bin count m must be >= 1");
        TSK_REQUIRE(extent_rule == TSK_EXTENT_MEMBER || extent_rule == TSK_EXTENT_GRID,
                    "unknown extent rule");
        TSK_REQUIRE(db->s.n > 0, "cannot index an empty store");
        TSK_REQUIRE(db->s.sorted, "store is not sorted by start time");
        TSK_CUDA(cudaSetDevice(db->device));
        cudaStream_t st = db->stream;
        Soa &s = db->s;
        Index &ix = db->ix;
        const int64_t n = s.n;
        // t0 = ts[0] (sorted), t_max = max te (core.py:213-225)
        double t0, tmax;
        {
            double *dmax;
            TSK_CUDA(cudaMallocAsync(&dmax, sizeof(double), st));
            size_t tb = 0;
            TSK_CUDA(cub::DeviceReduce::Max(nullptr, tb, s.te, dmax, n, st));
            void *tmp;
            TSK_CUDA(cudaMallocAsync(&tmp, tb, st));
            TSK_CUDA(cub::DeviceReduce::Max(tmp, tb, s.te, dmax, n, st));
            TSK_CUDA(cudaMemcpyAsync(&tmax, dmax, sizeof(double), cudaMemcpyDeviceToHost, st));
            TSK_CUDA(cudaMemcpyAsync(&t0, s.ts, sizeof(double), cudaMemcpyDeviceToHost, st));
            TSK_CUDA(cudaFreeAsync(tmp, st));
            TSK_CUDA(cudaFreeAsync(dmax, st));
            TSK_CUDA(cudaStreamSynchronize(st));
        }
        volatile double vm = (double)m;
        double width = (tmax - t0) / vm;  // index.py:107
        // scratch: first[m], last[m], flag[m], pos[m]
        size_t mb = (size_t)m * 8;
        int64_t *first, *last, *flag, *pos, *dn;
        TSK_CUDA(cudaMallocAsync(&first, mb, st));
        TSK_CUDA(cudaMallocAsync(&last, mb, st));
        TSK_CUDA(cudaMallocAsync(&flag, mb, st));
        TSK_CUDA(cudaMallocAsync(&pos, mb, st));
        TSK_CUDA(cudaMallocAsync(&dn, 8, st));
        TSK_CUDA(cudaMemsetAsync(first, 0xff, mb, st));
        TSK_CUDA(cudaMemsetAsync(last, 0xff, mb, st));
        int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
        k_bin_bounds<<<grid, 256, 0, st>>>(n, s.ts, t0, width, m, first, last);
        int gm = (int)std::min<int64_t>((m + 255) / 256, 148 * 8);
        k_bin_flags<<<gm, 256, 0, st>>>(m, first, flag);
        TSK_CUDA(cudaGetLastError());
        size_t tb = 0;
        TSK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, m, st));
        void *tmp;
        TSK_CUDA(cudaMallocAsync(&tmp, tb, st));
        TSK_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, flag, pos, m, st));
        TSK_CUDA(cudaFreeAsync(tmp, st));
        int64_t h_last_pos, h_last_flag;
        TSK_CUDA(cudaMemcpyAsync(&h_last_pos, pos + (m - 1), 8, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaMemcpyAsync(&h_last_flag, flag + (m - 1), 8, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        int64_t n_ne = h_last_pos + h_last_flag;
        size_t nn = (size_t)(n_ne > 0 ? n_ne : 1);
        ix.storage.reserve(nn * (3 * 8 + 3 * 8) + 64, st);
        char *base = ix.storage.as<char>();
        ix.ne_start = (double *)base; base += nn * 8;
        ix.ne_end = (double *)base; base += nn * 8;
        ix.ne_endmax = (double *)base; base += nn * 8;
        ix.ne_first = (int64_t *)base; base += nn * 8;
        ix.ne_last = (int64_t *)base; base += nn * 8;
        ix.ne_bin = (int64_t *)base;
        k_bin_compact<<<gm, 256, 0, st>>>(m, first, last, pos, s.ts, extent_rule, t0, width,
                                          ix.ne_start, ix.ne_first, ix.ne_last, ix.ne_bin);
        TSK_CUDA(cudaGetLastError());
        if (n_ne > 0) {
            int gw = (int)std::min<int64_t>((n_ne * 32 + 255) / 256, 148 * 16);
            k_bin_end<<<gw, 256, 0, st>>>(n_ne, ix.ne_first, ix.ne_last, s.te, ix.ne_end);
            TSK_CUDA(cudaGetLastError());
            tb = 0;
            TSK_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, ix.ne_end, ix.ne_endmax, MaxOp(),
                                                    n_ne, st));
            TSK_CUDA(cudaMallocAsync(&tmp, tb, st));
            TSK_CUDA(cub::DeviceScan::InclusiveScan(tmp, tb, ix.ne_end, ix.ne_endmax, MaxOp(), n_ne,
                                                    st));
            TSK_CUDA(cudaFreeAsync(tmp, st));
        }
        for (void *p : {(void *)first, (void *)last, (void *)flag, (void *)pos, (void *)dn})
            TSK_CUDA(cudaFreeAsync(p, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        ix.m = m;
        ix.n_ne = n_ne;
        ix.rule = extent_rule;
        ix.width = width;
        ix.t0 = t0;
        ix.t_max = tmax;
        ix.built = true;
        // K1's spatially ordered copy for this index's bins (layout.cu); when
        // it cannot be built (device memory) K1 reads the start-sorted store
        try {
            build_k1_layout(db, st);
        } catch (const Error &) {
            cudaGetLastError();
            cudaStreamSynchronize(st);
            free_k1_layout(db);
        }
        if (n_nonempty) *n_nonempty = n_ne;
        if (hdr) {
            hdr[0] = width;
            hdr[1] = t0;
            hdr[2] = tmax;
        }
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_index_copy(const tsk_db *db, double *ne_start, double *ne_end, int64_t *ne_first,
                              int64_t *ne_last, int64_t *bin_id) {
    try {
        TSK_REQUIRE(db && db->ix.built, "index not built");
        TSK_CUDA(cudaSetDevice(db->device));
        const Index &ix = db->ix;
        size_t b = (size_t)ix.n_ne * 8;
        if (b) {
            if (ne_start) TSK_CUDA(cudaMemcpyAsync(ne_start, ix.ne_start, b, cudaMemcpyDeviceToHost, db->stream));
            if (ne_end) TSK_CUDA(cudaMemcpyAsync(ne_end, ix.ne_end, b, cudaMemcpyDeviceToHost, db->stream));
            if (ne_first) TSK_CUDA(cudaMemcpyAsync(ne_first, ix.ne_first, b, cudaMemcpyDeviceToHost, db->stream));
            if (ne_last) TSK_CUDA(cudaMemcpyAsync(ne_last, ix.ne_last, b, cudaMemcpyDeviceToHost, db->stream));
            if (bin_id) TSK_CUDA(cudaMemcpyAsync(bin_id, ix.ne_bin, b, cudaMemcpyDeviceToHost, db->stream));
        }
        TSK_CUDA(cudaStreamSynchronize(db->stream));
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_candidate_ranges(tsk_db *db, int64_t k, const double *begin, const double *end,
                                    int64_t *first, int64_t *last) {
    try {
        TSK_REQUIRE(db && db->ix.built, "index not built");
        TSK_REQUIRE(k >= 0, "negative count");
        if (k == 0) return TSK_OK;
        TSK_CUDA(cudaSetDevice(db->device));
        cudaStream_t st = db->stream;
        double *d_b, *d_e;
        int64_t *d_f, *d_l;
        size_t b = (size_t)k * 8;
        TSK_CUDA(cudaMallocAsync(&d_b, b, st));
        TSK_CUDA(cudaMallocAsync(&d_e, b, st));
        TSK_CUDA(cudaMallocAsync(&d_f, b, st));
        TSK_CUDA(cudaMallocAsync(&d_l, b, st));
        TSK_CUDA(cudaMemcpyAsync(d_b, begin, b, cudaMemcpyHostToDevice, st));
        TSK_CUDA(cudaMemcpyAsync(d_e, end, b, cudaMemcpyHostToDevice, st));
        if (db->ix.n_ne == 0) {
            TSK_CUDA(cudaMemsetAsync(d_f, 0xff, b, st));
            TSK_CUDA(cudaMemsetAsync(d_l, 0xff, b, st));
        } else {
            int grid = (int)std::min<int64_t>((k * 32 + 255) / 256, 148 * 8);
            k_ranges_given<<<grid, 256, 0, st>>>(k, d_b, d_e, db->ix, d_f, d_l);
            TSK_CUDA(cudaGetLastError());
        }
        TSK_CUDA(cudaMemcpyAsync(first, d_f, b, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaMemcpyAsync(last, d_l, b, cudaMemcpyDeviceToHost, st));
        for (void *p : {(void *)d_b, (void *)d_e, (void *)d_f, (void *)d_l}) TSK_CUDA(cudaFreeAsync(p, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}
