// Host-side id gather vs PCIe D2H on the GPU box (design probe for the
// compact result path): 16 threads expand (entry ordinal, query ordinal)
// u32 pairs into four int64 id columns, alone and concurrently with a
// device-to-host copy; plus D2H alone.  nvcc -O3 -o /tmp/hgb tools/host_gather_bench.cu -lpthread
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <chrono>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main(int argc, char **argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 85000000;  // hits (c3 d=30)
    const int T = argc > 2 ? atoi(argv[2]) : 16;
    const int64_t ne = 10000000, nq = 40000;
    std::vector<int64_t> etraj(ne), eseg(ne), qtraj(nq), qseg(nq);
    for (int64_t i = 0; i < ne; ++i) { etraj[i] = i / 400; eseg[i] = i % 400; }
    for (int64_t i = 0; i < nq; ++i) { qtraj[i] = i / 400; qseg[i] = i % 400; }
    uint32_t *ord;  // pinned compact input: (e, q) pairs
    int64_t *out;   // pinned result columns (4 id columns)
    cudaHostAlloc((void **)&ord, n * 8, 0);
    cudaHostAlloc((void **)&out, n * 32, 0);
    // batch-like order: entries ascending in runs, queries within a batch of 120
    for (int64_t i = 0; i < n; ++i) {
        int64_t b = i / 250000;
        ord[2 * i] = (uint32_t)((b * 30000 + (i % 250000) / 8) % ne);
        ord[2 * i + 1] = (uint32_t)((b * 120 + (i * 7) % 120) % nq);
    }
    memset(out, 0, n * 32);
    auto gather = [&](int nt) {
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                int64_t a = n * t / nt, z = n * (t + 1) / nt;
                int64_t *o0 = out, *o1 = out + n, *o2 = out + 2 * n, *o3 = out + 3 * n;
                for (int64_t i = a; i < z; ++i) {
                    uint32_t e = ord[2 * i], q = ord[2 * i + 1];
                    o0[i] = qtraj[q]; o1[i] = qseg[q]; o2[i] = etraj[e]; o3[i] = eseg[e];
                }
            });
        for (auto &x : th) x.join();
    };
    for (int r = 0; r < 2; ++r) {
        double t0 = now();
        gather(T);
        double t1 = now();
        printf("gather %lld rows, %d threads: %.1f ms (%.1f GB/s written)\n", (long long)n, T, (t1 - t0) * 1e3,
               n * 32 / (t1 - t0) / 1e9);
    }
    // D2H alone: 24 B/hit and 48 B/hit
    void *dbuf;
    cudaMalloc(&dbuf, n * 48);
    char *h48;
    cudaHostAlloc((void **)&h48, n * 48, 0);
    memset(h48, 0, n * 48);
    for (int bytes : {24, 48}) {
        cudaMemcpy(h48, dbuf, n * bytes, cudaMemcpyDeviceToHost);
        double t0 = now();
        cudaMemcpy(h48, dbuf, n * bytes, cudaMemcpyDeviceToHost);
        double t1 = now();
        printf("D2H %d B/hit: %.1f ms (%.1f GB/s)\n", bytes, (t1 - t0) * 1e3, n * bytes / (t1 - t0) / 1e9);
    }
    // concurrent: D2H of 24 B/hit while gathering
    cudaStream_t s;
    cudaStreamCreate(&s);
    double t0 = now();
    cudaMemcpyAsync(h48, dbuf, n * 24, cudaMemcpyDeviceToHost, s);
    gather(T);
    double tg = now();
    cudaStreamSynchronize(s);
    double t1 = now();
    printf("concurrent D2H 24 B/hit + gather: gather done %.1f ms, both %.1f ms\n", (tg - t0) * 1e3, (t1 - t0) * 1e3);
    for (int nt : {4, 8, 32}) {
        double a = now();
        gather(nt);
        printf("gather %d threads: %.1f ms\n", nt, (now() - a) * 1e3);
    }
    return 0;
}
