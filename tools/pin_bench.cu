// Dev microbenchmark: cost of getting a 4 GiB result to the host.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <sys/mman.h>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    const size_t B = size_t(4) << 30;
    void *d; cudaMalloc(&d, B); cudaMemset(d, 1, B); cudaDeviceSynchronize();
    double t;
    // 1. cudaHostAlloc + D2H
    void *h; t = now(); cudaHostAlloc(&h, B, 0); double ta = now() - t;
    t = now(); cudaMemcpy(h, d, B, cudaMemcpyDeviceToHost); double tc = now() - t;
    printf("cudaHostAlloc %.3f s, D2H %.3f s (%.1f GB/s)\n", ta, tc, B / tc / 1e9);
    t = now(); cudaMemcpy(h, d, B, cudaMemcpyDeviceToHost); tc = now() - t;
    printf("  D2H again %.3f s (%.1f GB/s)\n", tc, B / tc / 1e9);
    cudaFreeHost(h);
    // 2. malloc + pageable D2H
    void *p = malloc(B); t = now(); cudaMemcpy(p, d, B, cudaMemcpyDeviceToHost); tc = now() - t;
    printf("pageable fresh D2H %.3f s (%.1f GB/s)\n", tc, B / tc / 1e9);
    t = now(); cudaMemcpy(p, d, B, cudaMemcpyDeviceToHost); tc = now() - t;
    printf("pageable warm D2H %.3f s (%.1f GB/s)\n", tc, B / tc / 1e9);
    free(p);
    // 3. mmap + THP + register
    t = now();
    void *m = mmap(nullptr, B, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(m, B, MADV_HUGEPAGE);
    cudaError_t e = cudaHostRegister(m, B, cudaHostRegisterDefault);
    ta = now() - t;
    t = now(); cudaMemcpy(m, d, B, cudaMemcpyDeviceToHost); tc = now() - t;
    printf("mmap+THP+register %.3f s (%s), D2H %.3f s (%.1f GB/s)\n", ta, cudaGetErrorString(e), tc, B / tc / 1e9);
    cudaHostUnregister(m); munmap(m, B);
    // 4. mmap + MAP_POPULATE + THP + register
    t = now();
    m = mmap(nullptr, B, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_POPULATE, -1, 0);
    e = cudaHostRegister(m, B, cudaHostRegisterDefault);
    ta = now() - t;
    t = now(); cudaMemcpy(m, d, B, cudaMemcpyDeviceToHost); tc = now() - t;
    printf("mmap populate+register %.3f s (%s), D2H %.3f s (%.1f GB/s)\n", ta, cudaGetErrorString(e), tc, B / tc / 1e9);
    return 0;
}
