// probe.cu — FP64 and FP32 pipe-rate microbenchmarks (K1's roofline denominators).
//
// K1 is bound by binary64 DADD/DMUL/DFMA issue; the
// measured peaks file carries only HBM and bf16 numbers, so the library
// measures the FP64 op rate itself: 8 independent dependency chains per
// thread, a full persistent grid, CUDA-event timing.
#include "tsk_internal.cuh"

namespace tsk {

template <int OP>
__global__ void k_fp64_probe(int iters, double seed, double *sink) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
    const double m = 1.0000000001, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (OP == 0) a[k] = __dadd_rn(a[k], c);
            else if (OP == 1) a[k] = __dmul_rn(a[k], m);
            else a[k] = __fma_rn(a[k], m, c);
        }
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) sink[threadIdx.x] = s;  // keeps the chains alive
}

// FP32 FFMA throughput: 8 independent chains per thread.
__global__ void k_fp32_probe(int iters, float seed, float *sink) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-6f + k;
    const float m = 1.0000001f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = __fmaf_rn(a[k], m, c);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678f) sink[threadIdx.x] = s;
}

}  // namespace tsk

using namespace tsk;

extern "C" int tsk_probe_fp32(int device, double *ffma_per_s) {
    try {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error{TSK_ENODEV, "no CUDA device visible"};
        TSK_CUDA(cudaSetDevice(device));
        int sms = 0;
        TSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        float *sink;
        TSK_CUDA(cudaMalloc(&sink, 1024 * sizeof(float)));
        cudaEvent_t e0, e1;
        TSK_CUDA(cudaEventCreate(&e0));
        TSK_CUDA(cudaEventCreate(&e1));
        const int threads = 256, blocks = sms * 8, iters = 8192;
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            TSK_CUDA(cudaEventRecord(e0));
            k_fp32_probe<<<blocks, threads>>>(iters, 1.0f, sink);
            TSK_CUDA(cudaGetLastError());
            TSK_CUDA(cudaEventRecord(e1));
            TSK_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            TSK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0 && ms < best) best = ms;  // rep 0 warms clocks
        }
        if (ffma_per_s) *ffma_per_s = (double)blocks * threads * iters * 8 / (best * 1e-3);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(sink);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_probe_fp64(int device, double *dadd_per_s, double *dmul_per_s,
                              double *dfma_per_s) {
    try {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw Error{TSK_ENODEV, "no CUDA device visible"};
        TSK_CUDA(cudaSetDevice(device));
        int sms = 0;
        TSK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        double *sink;
        TSK_CUDA(cudaMalloc(&sink, 1024 * sizeof(double)));
        cudaEvent_t e0, e1;
        TSK_CUDA(cudaEventCreate(&e0));
        TSK_CUDA(cudaEventCreate(&e1));
        const int threads = 256, blocks = sms * 8, iters = 4096;
        double *outs[3] = {dadd_per_s, dmul_per_s, dfma_per_s};
        for (int op = 0; op < 3; ++op) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {
                TSK_CUDA(cudaEventRecord(e0));
                if (op == 0) k_fp64_probe<0><<<blocks, threads>>>(iters, 1.0, sink);
                else if (op == 1) k_fp64_probe<1><<<blocks, threads>>>(iters, 1.0, sink);
                else k_fp64_probe<2><<<blocks, threads>>>(iters, 1.0, sink);
                TSK_CUDA(cudaGetLastError());
                TSK_CUDA(cudaEventRecord(e1));
                TSK_CUDA(cudaEventSynchronize(e1));
                float ms = 0;
                TSK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (rep > 0 && ms < best) best = ms;  // rep 0 warms clocks
            }
            double ops = (double)blocks * threads * iters * 8;
            if (outs[op]) *outs[op] = ops / (best * 1e-3);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        cudaFree(sink);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}
