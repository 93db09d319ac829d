// Dev microbenchmark: dependent-chain latency of DADD/DMUL/DFMA and LDS.128 on one warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void lat(int n, double seed, double *out, long long *cyc) {
    double a = seed + threadIdx.x;
    const double m = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (OP == 0) a = __dadd_rn(a, c);
        else if (OP == 1) a = __dmul_rn(a, m);
        else a = __fma_rn(a, m, c);
    }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double *o; long long *c, h;
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 8);
    const char *nm[3] = {"DADD", "DMUL", "DFMA"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            if (op == 0) lat<0><<<1, 32>>>(1 << 16, 1.0, o, c);
            if (op == 1) lat<1><<<1, 32>>>(1 << 16, 1.0, o, c);
            if (op == 2) lat<2><<<1, 32>>>(1 << 16, 1.0, o, c);
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("%s dependent latency: %.2f cycles\n", nm[op], (double)h / (1 << 16));
    }
    return 0;
}
