// canonical.cu — device canonical ordering of result sets.
//
// ResultSet.canonical_order (/root/reference/pkg/src/trajseek/core.py:290-294)
// is a numpy lexsort by (query_traj, query_seg, entry_traj, entry_seg,
// t_begin, t_end).  Here: least-significant-key-first stable radix sorts of
// order-preserving 64-bit keys — t_end, t_begin, then the four ids packed
// into as few composite keys as their value ranges allow — carrying a
// permutation.  Floats map ±0 to one key (numpy compares them equal; the
// sorts are stable like lexsort).
#include <cub/cub.cuh>

#include "tsk_internal.cuh"

namespace tsk {

__device__ __forceinline__ uint64_t mono_f64(double v) {
    if (v == 0.0) v = 0.0;
    uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_minmax4(int64_t n, const int64_t *__restrict__ a, const int64_t *__restrict__ b,
                          const int64_t *__restrict__ c, const int64_t *__restrict__ d,
                          unsigned long long *mm) {
    // mm[2k] = min (as order-flipped u64), mm[2k+1] = max
    const int64_t *cols[4] = {a, b, c, d};
    uint64_t lo[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { lo[k] = ~0ull; hi[k] = 0ull; }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            uint64_t v = (uint64_t)cols[k][i] ^ 0x8000000000000000ull;
            lo[k] = v < lo[k] ? v : lo[k];
            hi[k] = v > hi[k] ? v : hi[k];
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        for (int o = 16; o; o >>= 1) {
            uint64_t l2 = __shfl_xor_sync(0xffffffffu, lo[k], o), h2 = __shfl_xor_sync(0xffffffffu, hi[k], o);
            lo[k] = l2 < lo[k] ? l2 : lo[k];
            hi[k] = h2 > hi[k] ? h2 : hi[k];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&mm[2 * k], (unsigned long long)lo[k]);
            atomicMax(&mm[2 * k + 1], (unsigned long long)hi[k]);
        }
    }
}

__global__ void k_key_f64(int64_t n, const double *__restrict__ v, const uint32_t *__restrict__ perm,
                          uint64_t *__restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        key[i] = mono_f64(v[perm[i]]);
}

struct IdPack {
    const int64_t *col[4];
    uint64_t base[4];  // order-flipped minimum
    int shift[4];      // bit offset of each field in the composite key (-1: not in this key)
};

__global__ void k_key_ids(int64_t n, IdPack p, const uint32_t *__restrict__ perm,
                          uint64_t *__restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = perm[i];
        uint64_t k = 0;
#pragma unroll
        for (int f = 0; f < 4; ++f)
            if (p.shift[f] >= 0) k |= (((uint64_t)p.col[f][j] ^ 0x8000000000000000ull) - p.base[f]) << p.shift[f];
        key[i] = k;
    }
}

__global__ void k_iota32(int64_t n, uint32_t *v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

static int bits_of(uint64_t range) {  // bits for values 0..range
    int b = 0;
    while (b < 64 && (range >> b) != 0) ++b;
    return b;
}

// Stable canonical permutation of n result rows already in device memory.
// scratch is grown as needed; perm receives the final order.
void canonical_perm(int64_t n, const int64_t *qt, const int64_t *qs, const int64_t *et,
                    const int64_t *es, const double *tb, const double *te, uint32_t *perm,
                    DBuf &scratch, cudaStream_t st) {
    if (n == 0) return;
    const size_t nn = (size_t)n;
    // scratch: key_in, key_out (u64), perm_tmp (u32), mm (8 u64), cub temp
    size_t cub_bytes = 0;
    TSK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                             (uint32_t *)nullptr, (uint32_t *)nullptr, n, 0, 64, st));
    const size_t need = nn * 16 + nn * 4 + 64 + cub_bytes + 256;
    scratch.reserve(need, st);
    char *base = scratch.as<char>();
    uint64_t *k_in = reinterpret_cast<uint64_t *>(base);
    uint64_t *k_out = k_in + nn;
    uint32_t *p_tmp = reinterpret_cast<uint32_t *>(k_out + nn);
    unsigned long long *mm = reinterpret_cast<unsigned long long *>(
        (reinterpret_cast<uintptr_t>(p_tmp + nn) + 15) & ~uintptr_t(15));
    void *cub_tmp = reinterpret_cast<void *>((reinterpret_cast<uintptr_t>(mm + 8) + 255) & ~uintptr_t(255));

    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    // id ranges → composite key layout
    unsigned long long init[8];
    for (int k = 0; k < 4; ++k) { init[2 * k] = ~0ull; init[2 * k + 1] = 0ull; }
    TSK_CUDA(cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, st));
    k_minmax4<<<grid, 256, 0, st>>>(n, qt, qs, et, es, mm);
    TSK_CUDA(cudaGetLastError());
    unsigned long long h[8];
    TSK_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, st));
    TSK_CUDA(cudaStreamSynchronize(st));
    int width[4];
    for (int k = 0; k < 4; ++k) width[k] = bits_of(h[2 * k + 1] - h[2 * k]);

    k_iota32<<<grid, 256, 0, st>>>(n, perm);
    TSK_CUDA(cudaGetLastError());
    uint32_t *cur = perm, *alt = p_tmp;
    auto sort_pass = [&](int end_bit) {
        if (end_bit <= 0) end_bit = 1;
        size_t tb = cub_bytes;
        TSK_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, tb, k_in, k_out, cur, alt, n, 0, end_bit, st));
        std::swap(cur, alt);
    };
    // least significant first: t_end, t_begin
    k_key_f64<<<grid, 256, 0, st>>>(n, te, cur, k_in);
    sort_pass(64);
    k_key_f64<<<grid, 256, 0, st>>>(n, tb, cur, k_in);
    sort_pass(64);
    // ids, packed from the least significant field (entry_seg) upwards into
    // as few 64-bit keys as fit; each key is one stable pass
    const int64_t *cols[4] = {qt, qs, et, es};
    int f = 3;
    while (f >= 0) {
        IdPack p;
        for (int k = 0; k < 4; ++k) {
            p.col[k] = cols[k];
            p.base[k] = h[2 * k];
            p.shift[k] = -1;
        }
        int used = 0;
        while (f >= 0 && used + width[f] <= 64) {
            p.shift[f] = used;
            used += width[f];
            --f;
        }
        if (used == 0) {  // a single field wider than 64 bits cannot happen; guard anyway
            p.shift[f] = 0;
            used = 64;
            --f;
        }
        k_key_ids<<<grid, 256, 0, st>>>(n, p, cur, k_in);
        sort_pass(used);
    }
    TSK_CUDA(cudaGetLastError());
    if (cur != perm) TSK_CUDA(cudaMemcpyAsync(perm, cur, nn * 4, cudaMemcpyDeviceToDevice, st));
}

__global__ void k_permute6(int64_t n, const uint32_t *__restrict__ perm, const int64_t *__restrict__ a,
                           const int64_t *__restrict__ b, const int64_t *__restrict__ c,
                           const int64_t *__restrict__ d, const double *__restrict__ e,
                           const double *__restrict__ f, int64_t *__restrict__ oa,
                           int64_t *__restrict__ ob, int64_t *__restrict__ oc, int64_t *__restrict__ od,
                           double *__restrict__ oe, double *__restrict__ of) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t j = perm[i];
        oa[i] = a[j];
        ob[i] = b[j];
        oc[i] = c[j];
        od[i] = d[j];
        oe[i] = e[j];
        of[i] = f[j];
    }
}

void permute6(int64_t n, const uint32_t *perm, const int64_t *const in_i[4], const double *const in_f[2],
              int64_t *const out_i[4], double *const out_f[2], cudaStream_t st) {
    if (n == 0) return;
    const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_permute6<<<grid, 256, 0, st>>>(n, perm, in_i[0], in_i[1], in_i[2], in_i[3], in_f[0], in_f[1],
                                     out_i[0], out_i[1], out_i[2], out_i[3], out_f[0], out_f[1]);
    TSK_CUDA(cudaGetLastError());
}

}  // namespace tsk

using namespace tsk;

extern "C" int tsk_canonical_order(int device, int64_t n, const int64_t *qt, const int64_t *qs,
                                   const int64_t *et, const int64_t *es, const double *tb,
                                   const double *te, int64_t *o_qt, int64_t *o_qs, int64_t *o_et,
                                   int64_t *o_es, double *o_tb, double *o_te) {
    try {
        TSK_REQUIRE(n >= 0, "negative count");
        TSK_REQUIRE(n < (int64_t(1) << 32), "more than 2^32 rows");
        if (n == 0) return TSK_OK;
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error{TSK_ENODEV, "no CUDA device visible"};
        TSK_CUDA(cudaSetDevice(device));
        cudaStream_t st;
        TSK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const size_t nn = (size_t)n, cb = nn * 8;
        DBuf cols, scratch;
        cols.reserve(cb * 12 + nn * 4, st);
        char *b = cols.as<char>();
        int64_t *din_i[4], *dout_i[4];
        double *din_f[2], *dout_f[2];
        for (int k = 0; k < 4; ++k) din_i[k] = reinterpret_cast<int64_t *>(b + k * cb);
        for (int k = 0; k < 2; ++k) din_f[k] = reinterpret_cast<double *>(b + (4 + k) * cb);
        for (int k = 0; k < 4; ++k) dout_i[k] = reinterpret_cast<int64_t *>(b + (6 + k) * cb);
        for (int k = 0; k < 2; ++k) dout_f[k] = reinterpret_cast<double *>(b + (10 + k) * cb);
        uint32_t *perm = reinterpret_cast<uint32_t *>(b + 12 * cb);
        const int64_t *hi[4] = {qt, qs, et, es};
        const double *hf[2] = {tb, te};
        for (int k = 0; k < 4; ++k) TSK_CUDA(cudaMemcpyAsync(din_i[k], hi[k], cb, cudaMemcpyHostToDevice, st));
        for (int k = 0; k < 2; ++k) TSK_CUDA(cudaMemcpyAsync(din_f[k], hf[k], cb, cudaMemcpyHostToDevice, st));
        canonical_perm(n, din_i[0], din_i[1], din_i[2], din_i[3], din_f[0], din_f[1], perm, scratch, st);
        const int64_t *ci[4] = {din_i[0], din_i[1], din_i[2], din_i[3]};
        const double *cf[2] = {din_f[0], din_f[1]};
        permute6(n, perm, ci, cf, dout_i, dout_f, st);
        int64_t *ho_i[4] = {o_qt, o_qs, o_et, o_es};
        double *ho_f[2] = {o_tb, o_te};
        for (int k = 0; k < 4; ++k) TSK_CUDA(cudaMemcpyAsync(ho_i[k], dout_i[k], cb, cudaMemcpyDeviceToHost, st));
        for (int k = 0; k < 2; ++k) TSK_CUDA(cudaMemcpyAsync(ho_f[k], dout_f[k], cb, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        cols.release(st);
        scratch.release(st);
        TSK_CUDA(cudaStreamDestroy(st));
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}
