// search.cu — plan execution pipeline, K4 result finalisation and the C-ABI
// entry points tsk_search / tsk_pair_intervals / tsk_result_*.
//
//   run_search ........ /root/reference/pkg/src/trajseek/engine.py:151-204
//   execute_batch ..... engine.py:97-148
//   pair_intervals .... core.py:464-565
//   result assembly ... engine.py:133-146 (id gather), core.py:249-303 (ResultSet)
//
// Pipeline on the db's stream (one host sync for the hit count, one at the end):
//   H2D queries → hoist + 112-B records → K3 batch ranges → item scan →
//   K1 (persistent, atomic work queue) → [grow + rerun on overflow] →
//   K4 radix sort of 64-bit (batch, entry, query) keys → id gather → D2H
//   into a pinned block owned by the tsk_result.
#include <cub/cub.cuh>

#include <chrono>
#include <condition_variable>
#include <functional>
#include <thread>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <sys/mman.h>
#include <unistd.h>
#include <algorithm>
#include <mutex>
#include <vector>

#include "hostpool.h"
#include "tsk_internal.cuh"

namespace tsk {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    set_error(msg);
    return code;
}

// ── pinned host pool ───────────────────────────────────────────────────────

// Result columns live in page-locked host blocks kept in a pool: pinning
// costs ~0.2-0.5 s/GB, so steady-state calls reuse blocks.  Large blocks are
// anonymous mmaps advised onto transparent huge pages and registered with
// cudaHostRegister (measured 3x cheaper to pin than cudaHostAlloc on the
// B200 hosts, same 57 GB/s D2H); small ones come from cudaHostAlloc.
static std::mutex g_pin_mu;
static std::multimap<size_t, void *> g_pin_free;
static std::map<void *, int> g_pin_kind;  // 0: cudaHostAlloc, 1: mmap + register
static size_t g_pin_cached = 0;
static const size_t kMmapAbove = size_t(32) << 20;

static size_t pin_cache_max() {
    static size_t cap = [] {
        long pages = sysconf(_SC_PHYS_PAGES), psize = sysconf(_SC_PAGE_SIZE);
        size_t ram = (pages > 0 && psize > 0) ? (size_t)pages * (size_t)psize : (size_t(64) << 30);
        return std::max<size_t>(size_t(8) << 30, ram / 4);
    }();
    return cap;
}

static void pin_release(void *p, size_t bytes) {
    int kind;
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        kind = g_pin_kind[p];
        g_pin_kind.erase(p);
    }
    if (kind == 1) {
        cudaHostUnregister(p);
        munmap(p, bytes);
    } else {
        cudaFreeHost(p);
    }
}

// Size classes for large blocks (2^k x {1, 1.25, 1.5, 1.75}): the
// pipelined and single-launch result paths ask for slightly different sizes
// of the same result, and both then reuse each other's cached blocks.
static size_t pin_size_class(size_t bytes) {
    if (bytes < kMmapAbove) return bytes;
    size_t p = size_t(1) << (63 - __builtin_clzll((unsigned long long)bytes));
    for (int q = 4; q <= 8; ++q)
        if (p / 4 * q >= bytes) return p / 4 * q;
    return 2 * p;
}

static void *pin_alloc(size_t bytes, size_t *got) {
    if (bytes == 0) bytes = 64;
    bytes = pin_size_class(bytes);
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        auto it = g_pin_free.lower_bound(bytes);
        if (it != g_pin_free.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
            void *p = it->second;
            *got = it->first;
            g_pin_cached -= it->first;
            g_pin_free.erase(it);
            return p;
        }
    }
    void *p = nullptr;
    int kind = 0;
    if (bytes >= kMmapAbove) {
        bytes = (bytes + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
        void *m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (m != MAP_FAILED) {
            madvise(m, bytes, MADV_HUGEPAGE);
            if (cudaHostRegister(m, bytes, cudaHostRegisterPortable) == cudaSuccess) {
                p = m;
                kind = 1;
            } else {
                cudaGetLastError();
                munmap(m, bytes);
            }
        }
    }
    if (!p) TSK_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocPortable));
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        g_pin_kind[p] = kind;
    }
    *got = bytes;
    return p;
}

static void pin_free(void *p, size_t bytes) {
    if (!p) return;
    {
        std::lock_guard<std::mutex> g(g_pin_mu);
        if (g_pin_cached + bytes <= pin_cache_max()) {
            g_pin_free.emplace(bytes, p);
            g_pin_cached += bytes;
            return;
        }
    }
    pin_release(p, bytes);
}

static int bits_for(int64_t count) {  // bits to hold 0..count-1
    int b = 0;
    while (b < 63 && (int64_t(1) << b) < count) ++b;
    return b;
}

// ── K4: id gather in the requested order ───────────────────────────────────

struct GatherArgs {
    int64_t n;
    const uint64_t *keys;
    const uint32_t *perm;  // nullptr: identity
    const double *tb_in, *te_in;
    const int64_t *lo, *first;
    const int64_t *qtraj, *qseg, *etraj, *eseg;
    int64_t *o_qtraj, *o_qseg, *o_etraj, *o_eseg, *o_qord, *o_eord;
    double *o_tb, *o_te;
    int major_bits, minor_bits, query_major;
};

__global__ void k_gather(GatherArgs a) {
    const uint64_t mmask = a.major_bits ? ((~0ull) >> (64 - a.major_bits)) : 0ull;
    const uint64_t nmask = a.minor_bits ? ((~0ull) >> (64 - a.minor_bits)) : 0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = a.keys[i];
        int64_t b = (int64_t)(a.major_bits + a.minor_bits < 64 ? (k >> (a.major_bits + a.minor_bits)) : 0);
        int64_t major = (int64_t)((k >> a.minor_bits) & mmask);
        int64_t minor = (int64_t)(k & nmask);
        int64_t q_off = a.query_major ? major : minor;
        int64_t e_off = a.query_major ? minor : major;
        int64_t q = a.lo[b] + q_off, e = a.first[b] + e_off;
        int64_t j = a.perm ? (int64_t)a.perm[i] : i;
        a.o_qtraj[i] = a.qtraj[q];
        a.o_qseg[i] = a.qseg[q];
        a.o_etraj[i] = a.etraj[e];
        a.o_eseg[i] = a.eseg[e];
        a.o_tb[i] = a.tb_in[j];
        a.o_te[i] = a.te_in[j];
        if (a.o_qord) a.o_qord[i] = q;
        if (a.o_eord) a.o_eord[i] = e;
    }
}

// K4, compact form: per sorted hit row the start-sorted entry ordinal and the
// query ordinal (u32 each) and the interval, 24 B instead of 48; the host
// expands the four id columns from the ordinals (search.cu: compact_rows).
__global__ void k_compact(int64_t r0, int64_t r1, const uint64_t *__restrict__ keys, const uint32_t *__restrict__ perm,
                          const double *__restrict__ tb_in, const double *__restrict__ te_in,
                          const int64_t *__restrict__ lo, const int64_t *__restrict__ first, int major_bits,
                          int minor_bits, const int64_t *__restrict__ etraj, const int64_t *__restrict__ eseg,
                          double *__restrict__ o_tb, double *__restrict__ o_te, int64_t *__restrict__ o_et,
                          int64_t *__restrict__ o_es, uint32_t *__restrict__ o_qo, int ids32) {
    const uint64_t mmask = major_bits ? ((~0ull) >> (64 - major_bits)) : 0ull;
    const uint64_t nmask = minor_bits ? ((~0ull) >> (64 - minor_bits)) : 0ull;
    for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const int64_t b = (int64_t)(major_bits + minor_bits < 64 ? (k >> (major_bits + minor_bits)) : 0);
        const int64_t e = first[b] + (int64_t)((k >> minor_bits) & mmask);
        const int64_t q = lo[b] + (int64_t)(k & nmask);
        const int64_t j = perm ? (int64_t)perm[i] : i;
        if (ids32) {  // ids known to fit: 4 bytes each over PCIe
            reinterpret_cast<int32_t *>(o_et)[i] = (int32_t)etraj[e];
            reinterpret_cast<int32_t *>(o_es)[i] = (int32_t)eseg[e];
        } else {
            o_et[i] = etraj[e];
            o_es[i] = eseg[e];
        }
        o_qo[i] = (uint32_t)q;
        o_tb[i] = tb_in[j];
        o_te[i] = te_in[j];
    }
}

__global__ void k_iota(int64_t n, uint32_t *v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

// K4 for small hit counts: one CTA sorts up to K4_SMALL (key, append index)
// pairs in shared memory with a bitonic network — one launch instead of
// the radix sort's several.  Keys are unique (one hit per pair), so the
// order equals the stable radix sort's.
constexpr int K4_SMALL = 4096;

__global__ void __launch_bounds__(1024) k_small_sort(int n, const uint64_t *__restrict__ keys_in,
                                                     uint64_t *__restrict__ keys_out,
                                                     uint32_t *__restrict__ perm_out) {
    __shared__ uint64_t k[K4_SMALL];
    __shared__ uint32_t v[K4_SMALL];
    int m = 1;
    while (m < n) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        k[i] = i < n ? keys_in[i] : ~0ull;  // padding sorts last
        v[i] = (uint32_t)i;
    }
    __syncthreads();
    for (int size = 2; size <= m; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (m >> 1); t += blockDim.x) {
                const int i = 2 * t - (t & (stride - 1));  // lower index of the pair
                const int j = i + stride;
                const bool up = (i & size) == 0;
                const uint64_t a = k[i], b = k[j];
                const uint32_t va = v[i], vb = v[j];
                // (key, index) order: padding stays behind a real all-ones key
                if ((a > b || (a == b && va > vb)) == up) {
                    k[i] = b; k[j] = a;
                    v[i] = vb; v[j] = va;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        keys_out[i] = k[i];
        perm_out[i] = v[i];
    }
}

// Opt-in phase trace (TSK_TRACE=1): CUDA events at phase boundaries on the
// db stream, printed to stderr when the call completes.
struct Trace {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<std::pair<const char *, cudaEvent_t>> marks;
    explicit Trace(cudaStream_t s) : st(s) {
        const char *v = getenv("TSK_TRACE");
        on = v && *v && *v != '0';
    }
    void mark(const char *name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        marks.emplace_back(name, e);
    }
    ~Trace() {
        if (!on || marks.empty()) return;
        cudaEventSynchronize(marks.back().second);
        fprintf(stderr, "[tsk trace]");
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
            fprintf(stderr, " %s=%.3f", marks[i].first, ms);
        }
        fprintf(stderr, " (ms)\n");
        for (auto &m : marks) cudaEventDestroy(m.second);
    }
};

static int sm_count(int device) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n > 0 ? n : 148;
}

// Results of at least this many rows take the compact path (below it the
// 48-byte device gather and one copy are cheaper than the pipeline).
static const int64_t kCompactMin = int64_t(1) << 21;  // below ~2M rows one 48 B/row copy is faster (c3: 0.44 vs 0.82 ms)
static const int64_t kCompactChunk = int64_t(1) << 21;  // rows per pipeline chunk

// Compact result assembly, pipelined: for each chunk of sorted rows K4
// writes t_begin, t_end and the entry ids (gathered on the device) plus the
// query ordinal on the db stream; a copy stream moves the first four
// straight into the result's pinned columns and the ordinals into a pinned
// staging block (36 B/row over PCIe instead of 48); host threads expand the
// query id columns of chunk c (a small, cache-resident table) while chunk
// c+1 is in flight.  Result bytes are identical to the device gather's.
static void compact_rows(tsk_db *db, tsk_result *res, const tsk_columns *qc, int64_t nh, const uint64_t *keys,
                         const uint32_t *perm, const double *tbin, const double *tein, const int64_t *d_lo,
                         const int64_t *d_first, int major_bits, int minor_bits, cudaStream_t st,
                         int64_t &launches) {
    const size_t cb = (size_t)nh * 8;
    db->out_cols.reserve((size_t)nh * 36 + 64, st);
    double *d_tb = db->out_cols.as<double>();
    double *d_te = d_tb + nh;
    int64_t *d_et = reinterpret_cast<int64_t *>(d_te + nh);
    int64_t *d_es = d_et + nh;
    uint32_t *d_qo = reinterpret_cast<uint32_t *>(d_es + nh);
    size_t got = 0;
    res->host = pin_alloc(cb * 6, &got);
    res->host_bytes = got;
    char *hb = static_cast<char *>(res->host);
    res->qtraj = (int64_t *)(hb + 0 * cb);
    res->qseg = (int64_t *)(hb + 1 * cb);
    res->etraj = (int64_t *)(hb + 2 * cb);
    res->eseg = (int64_t *)(hb + 3 * cb);
    res->tbeg = (double *)(hb + 4 * cb);
    res->tend = (double *)(hb + 5 * cb);
    size_t ogot = 0;
    uint32_t *h_qo = static_cast<uint32_t *>(pin_alloc((size_t)nh * 4, &ogot));
    if (!db->stream2) TSK_CUDA(cudaStreamCreateWithFlags(&db->stream2, cudaStreamNonBlocking));
    cudaStream_t st2 = db->stream2;
    int64_t chunk = kCompactChunk;
    if (const char *e = getenv("TSK_COMPACT_CHUNK")) chunk = std::max<int64_t>(1, atoll(e));  // testing
    const int64_t nc = (nh + chunk - 1) / chunk;
    std::vector<cudaEvent_t> evg((size_t)nc), evd((size_t)nc);
    for (int64_t c = 0; c < nc; ++c) {
        TSK_CUDA(cudaEventCreateWithFlags(&evg[c], cudaEventDisableTiming));
        TSK_CUDA(cudaEventCreateWithFlags(&evd[c], cudaEventDisableTiming));  // spin: a blocking wait wakes ~0.5 ms late
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t r0 = c * chunk, r1 = std::min<int64_t>(nh, r0 + chunk), m = r1 - r0;
        const int grid = (int)std::min<int64_t>((m + 255) / 256, 148 * 8);
        k_compact<<<grid, 256, 0, st>>>(r0, r1, keys, perm, tbin, tein, d_lo, d_first, major_bits, minor_bits,
                                        db->s.traj, db->s.seg, d_tb, d_te, d_et, d_es, d_qo, 0);
        TSK_CUDA(cudaGetLastError());
        ++launches;
        TSK_CUDA(cudaEventRecord(evg[c], st));
        TSK_CUDA(cudaStreamWaitEvent(st2, evg[c], 0));
        TSK_CUDA(cudaMemcpyAsync(res->tbeg + r0, d_tb + r0, (size_t)m * 8, cudaMemcpyDeviceToHost, st2));
        TSK_CUDA(cudaMemcpyAsync(res->tend + r0, d_te + r0, (size_t)m * 8, cudaMemcpyDeviceToHost, st2));
        TSK_CUDA(cudaMemcpyAsync(res->etraj + r0, d_et + r0, (size_t)m * 8, cudaMemcpyDeviceToHost, st2));
        TSK_CUDA(cudaMemcpyAsync(res->eseg + r0, d_es + r0, (size_t)m * 8, cudaMemcpyDeviceToHost, st2));
        TSK_CUDA(cudaMemcpyAsync(h_qo + r0, d_qo + r0, (size_t)m * 4, cudaMemcpyDeviceToHost, st2));
        TSK_CUDA(cudaEventRecord(evd[c], st2));
    }
    // the db stream waits for the copies (the caller's end event covers them)
    TSK_CUDA(cudaStreamWaitEvent(st, evd[nc - 1], 0));
    const int64_t *qt = qc->traj, *qs = qc->seg;
    HostPool &pool = HostPool::get();
    const bool trace = getenv("TSK_TRACE") != nullptr;
    double t_wait = 0.0, t_exp = 0.0;
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t r0 = c * chunk, r1 = std::min<int64_t>(nh, r0 + chunk);
        const auto h0 = std::chrono::steady_clock::now();
        TSK_CUDA(cudaEventSynchronize(evd[c]));
        const auto h1 = std::chrono::steady_clock::now();
        t_wait += std::chrono::duration<double>(h1 - h0).count();
        pool.run([&](int part, int parts) {
            const int64_t a = r0 + (r1 - r0) * part / parts, z = r0 + (r1 - r0) * (part + 1) / parts;
            for (int64_t i = a; i < z; ++i) {
                const uint32_t q = h_qo[i];
                res->qtraj[i] = qt[q];
                res->qseg[i] = qs[q];
            }
        });
        t_exp += std::chrono::duration<double>(std::chrono::steady_clock::now() - h1).count();
    }
    if (trace)
        fprintf(stderr, "[tsk trace] compact %lld rows in %lld chunks: host wait %.3f ms, expansion %.3f ms (%d threads)\n",
                (long long)nh, (long long)nc, t_wait * 1e3, t_exp * 1e3, pool.size());
    for (int64_t c = 0; c < nc; ++c) {
        cudaEventDestroy(evg[c]);
        cudaEventDestroy(evd[c]);
    }
    pin_free(h_qo, ogot);
}

// ── pipelined search (north star (d): H2D / compute / D2H overlap) ───────────
//
// Reference-ordered results through the compact path (28 B/row over PCIe
// when entry ids fit in int32, else 36).  The plan is cut into
// chunks of consecutive batches (even boundaries keep K1's batch pairs);
// chunk c's K1 appends to the shared result buffer behind chunk c-1's hits,
// and the host learns each chunk's row range from a counter snapshot.  The
// db stream runs K1(0) S(0) K1(1) S(1) ... where S(c) sorts chunk c's keys
// (K4) and gathers its rows (t_begin, t_end, entry ids, query ordinal); the
// host enqueues S(c) and K1(c+1) as soon as K1(c)'s count arrives (a gap of
// one host round trip per chunk), the copy stream moves chunk c's rows over
// PCIe while K1(c+1) computes, and host threads expand the query ids of
// finished chunks.
// The rows land in their final place in one pinned block sized by the
// buffer capacity; the result equals the single-launch path's (batch order
// is chunk order, engine.py:176-195).  On overflow of the buffer it returns
// nullptr and the caller falls back to the exact-sizing path.
static const int64_t kPipeMinRows = int64_t(1) << 20;
// Plans of at least this many batches run K1 in its wide build (octets).
// Measured K1 time, wide against 512-query tiles: c5 (3,334 batches) -6.5%,
// its N = 2 / 4 shards (1,667 / 834) -4% / -1%, c4 (575) -6%; N = 8 shards
// (417) +3%, c3 (334) +3%, c2 (334) +26%.
static const int64_t kWideMinBatches = 512;
static const int kPipeMinChunks = 4, kPipeMaxChunks = 16;

// Counter snapshot straight into mapped host memory: a copy-engine read
// would queue behind the chunk copies already crossing PCIe.
__global__ void k_snap(const unsigned long long *__restrict__ ctr, unsigned long long *host) {
    host[0] = ctr[1];
    host[1] = ctr[2];
    __threadfence_system();
}

// Rows one call returns: 2^32 (TSK_MAX_HITS lowers it for testing).
static unsigned long long max_hits_per_call() {
    unsigned long long m = 1ull << 32;
    if (const char *e = getenv("TSK_MAX_HITS")) m = std::min<unsigned long long>(m, strtoull(e, nullptr, 10));
    return m;
}

static void sort_rows(tsk_db *db, const uint64_t *keys, uint64_t *ko, uint32_t *v0, uint32_t *v1, int64_t n,
                      int end_bit, cudaStream_t st, int64_t &launches) {
    if (n <= K4_SMALL) {
        k_small_sort<<<1, 1024, 0, st>>>((int)n, keys, ko, v1);
        TSK_CUDA(cudaGetLastError());
        ++launches;
        return;
    }
    const int gi = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_iota<<<gi, 256, 0, st>>>(n, v0);
    TSK_CUDA(cudaGetLastError());
    ++launches;
    if (end_bit == 0) end_bit = 1;
    size_t tb = 0;
    TSK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, ko, v0, v1, n, 0, end_bit, st));
    db->cub_tmp.reserve(tb, st);
    TSK_CUDA(cub::DeviceRadixSort::SortPairs(db->cub_tmp.p, tb, keys, ko, v0, v1, n, 0, end_bit, st));
}

static tsk_result *run_pipelined(tsk_db *db, const tsk_columns *qc, const SearchPlanDev &plan, K1Launch L,
                                 int slots, int stride, int pair, int align, int tq_max, int major_bits, int minor_bits, int bb,
                                 uint64_t cap, Trace &tr, int64_t &launches) {
    const int64_t nb = plan.nb;
    // chunks: worth it once the rows' PCIe time is noticeable (the previous
    // call's hit count predicts this one's); ~2^20 rows per chunk, 4..16
    // (Mid-size results go through one 48 B/row copy instead: at c5, 8.8e5
    // rows behind 24 ms of K1, 3 chunks measured 26.3 ms against 26.0.)
    int C = 0;
    if (db->last_hits >= kPipeMinRows)
        C = (int)std::min<int64_t>(kPipeMaxChunks, std::max<int64_t>(kPipeMinChunks, db->last_hits >> 20));
    if (const char *e = getenv("TSK_PIPE_CHUNKS")) C = std::max(0, atoi(e));  // testing: 0 = off
    if (C == 0) return nullptr;
    C = (int)std::max<int64_t>(1, std::min<int64_t>(C, nb / 2));
    // the host block holds `cap` rows: not when cap is far above recent results
    if ((double)cap > 8.0 * (double)std::max<int64_t>(db->last_hits, int64_t(1) << 20)) return nullptr;
    cudaStream_t st = db->stream;
    if (!db->stream2) TSK_CUDA(cudaStreamCreateWithFlags(&db->stream2, cudaStreamNonBlocking));
    cudaStream_t st2 = db->stream2;

    // boundaries at even batch ordinals with about equal interactions each,
    // from the batches' candidate spans (K3 has run: one small read-back)
    std::vector<int64_t> B((size_t)C + 1);
    {
        size_t sg = 0;
        int64_t *h_fl = static_cast<int64_t *>(pin_alloc((size_t)nb * 16, &sg));
        TSK_CUDA(cudaMemcpyAsync(h_fl, plan.first, (size_t)nb * 16, cudaMemcpyDeviceToHost, st));  // first[], last[]
        std::vector<int64_t> blo((size_t)nb), bhi((size_t)nb);
        TSK_CUDA(cudaMemcpyAsync(blo.data(), plan.lo, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaMemcpyAsync(bhi.data(), plan.hi, (size_t)nb * 8, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        std::vector<double> pre((size_t)nb + 1, 0.0);
        for (int64_t b = 0; b < nb; ++b) {
            const int64_t f = h_fl[b], l = h_fl[nb + b];
            const double w = f >= 0 ? (double)(l - f + 1) * (double)(bhi[b] - blo[b] + 1) : 0.0;
            pre[b + 1] = pre[b] + w;
        }
        pin_free(h_fl, sg);
        B[0] = 0;
        for (int c = 1; c < C; ++c) {
            const double target = pre[nb] * c / C;
            int64_t b = std::lower_bound(pre.begin(), pre.end(), target) - pre.begin();
            b &= ~int64_t(1);
            B[c] = std::max(B[c - 1], std::min(b, nb));
        }
        B[C] = nb;
    }
    std::vector<SearchPlanDev> pc((size_t)C);
    size_t words = 0;
    for (int c = 0; c < C; ++c) words += (size_t)plan_units(B[c + 1] - B[c]) + 5;
    db->pipe.reserve(words * 8, st);
    int64_t *pp = db->pipe.as<int64_t>();
    for (int c = 0; c < C; ++c) {
        const int64_t b0 = B[c], nbc = B[c + 1] - b0, nu = plan_units(nbc);
        pc[c] = SearchPlanDev{nbc, plan.lo + b0, plan.hi + b0, plan.first + b0, plan.last + b0, pp, pp + nu + 1,
                              plan.ovl + b0, plan.hits + b0};
        pp += nu + 5;
    }
    // device buffers sized by the capacity
    L.cap = cap;
    L.keys = db->recs.as<uint64_t>();
    L.tbeg = reinterpret_cast<double *>(L.keys + cap);
    L.tend = L.tbeg + cap;
    db->sorted.reserve((size_t)cap * 24 + 64, st);
    uint64_t *ko = db->sorted.as<uint64_t>();
    uint32_t *v0 = reinterpret_cast<uint32_t *>(ko + cap), *v1 = v0 + cap;
    db->out_cols.reserve((size_t)cap * 36 + 64, st);
    double *d_tb = db->out_cols.as<double>(), *d_te = d_tb + cap;
    int64_t *d_et = reinterpret_cast<int64_t *>(d_te + cap), *d_es = d_et + cap;
    uint32_t *d_qo = reinterpret_cast<uint32_t *>(d_es + cap);
    unsigned long long *d_ctr = L.item_counter;  // [0] items, [1] hits, [2] evaluated pairs
    TSK_CUDA(cudaMemsetAsync(d_ctr, 0, 24, st));
    TSK_CUDA(cudaMemsetAsync(plan.ovl, 0, (size_t)nb * 16, st));  // ovl[nb] then hits[nb]
    // pinned: counter snapshots, the result block (cap rows), query ordinals
    size_t sgot = 0, hgot = 0, qgot = 0;
    unsigned long long *snap = static_cast<unsigned long long *>(pin_alloc((size_t)C * 16, &sgot));
    unsigned long long *snap_dev = nullptr;
    TSK_CUDA(cudaHostGetDevicePointer((void **)&snap_dev, snap, 0));
    char *hb = static_cast<char *>(pin_alloc((size_t)cap * 48, &hgot));
    // query ordinals (and 32-bit entry ids when they fit), widened on the
    // host.  Beyond ~2^23 rows the host's memory bandwidth, not PCIe, bounds
    // the call (the widening adds 20 B/row of host traffic to save 8 B/row
    // of PCIe): c3 d = 30, 8.4e7 rows, 68 ms at 36 B/row vs 73 ms at 28
    const int ids32 = db->ids32 && db->last_hits < (int64_t(1) << 23);
    uint32_t *h_qo = static_cast<uint32_t *>(pin_alloc((size_t)cap * (ids32 ? 12 : 4), &qgot));
    int32_t *h_et32 = reinterpret_cast<int32_t *>(h_qo + cap), *h_es32 = h_et32 + cap;
    const size_t cs = (size_t)cap * 8;
    int64_t *o_qt = (int64_t *)(hb + 0 * cs), *o_qs = (int64_t *)(hb + 1 * cs);
    int64_t *o_et = (int64_t *)(hb + 2 * cs), *o_es = (int64_t *)(hb + 3 * cs);
    double *o_tb = (double *)(hb + 4 * cs), *o_te = (double *)(hb + 5 * cs);

    std::vector<cudaEvent_t> ek0((size_t)C), ek1((size_t)C), eks((size_t)C), evd((size_t)C), evq((size_t)C);
    for (int c = 0; c < C; ++c) {
        TSK_CUDA(cudaEventCreate(&ek0[c]));
        TSK_CUDA(cudaEventCreate(&ek1[c]));
        // spin on the count (a blocking wait adds ~0.2 ms of wake-up per chunk)
        TSK_CUDA(cudaEventCreateWithFlags(&eks[c], cudaEventDisableTiming));
        TSK_CUDA(cudaEventCreate(&evd[c]));  // spin wait (see compact_rows)
        TSK_CUDA(cudaEventCreateWithFlags(&evq[c], cudaEventDisableTiming));
    }
    const bool trace = getenv("TSK_TRACE") != nullptr;
    std::vector<cudaEvent_t> esd((size_t)C, nullptr);  // (trace) end of S(c)
    std::vector<double> h_seen((size_t)C, 0.0);          // (trace) host saw K1(c)'s count, ms after start
    const auto h_start = std::chrono::steady_clock::now();
    auto cleanup = [&]() {
        for (int c = 0; c < C; ++c) {
            cudaEventDestroy(ek0[c]);
            cudaEventDestroy(ek1[c]);
            cudaEventDestroy(eks[c]);
            cudaEventDestroy(evd[c]);
            cudaEventDestroy(evq[c]);
            if (esd[c]) cudaEventDestroy(esd[c]);
        }
        pin_free(snap, sgot);
        pin_free(h_qo, qgot);
    };
    // a chunk below the wide kernel's plan size runs the 512-query kernel
    // (quads) even when the whole plan chose the wide one
    const char *we = getenv("TSK_K1_WIDE");
    const bool force_wide = we && !strcmp(we, "force");
    auto enqueue_k1 = [&](int c) {
        K1Launch Lc = L;
        Lc.plan = pc[c];
        int c_slots = slots, c_stride = stride, c_pair = pair, c_tq = tq_max;
        if (L.wide && !force_wide && pc[c].nb < kWideMinBatches) {
            Lc.wide = 0;
            c_slots = sm_count(db->device) * k1_blocks_per_sm(true);
            c_stride = K1_THREADS * k1_candidates_per_thread(true);
            c_pair = pair == 9 ? 5 : 4;
            c_tq = K1_TQ;
        }
        launch_plan_items(pc[c], c_slots, c_stride, c_pair, align, c_tq, L.q_unsorted, st);
        ++launches;
        TSK_CUDA(cudaMemsetAsync(d_ctr, 0, 8, st));  // the item counter
        TSK_CUDA(cudaEventRecord(ek0[c], st));
        launch_k1(Lc, c_slots, st);
        ++launches;
        TSK_CUDA(cudaEventRecord(ek1[c], st));
        k_snap<<<1, 1, 0, st>>>(d_ctr, snap_dev + 2 * c);
        TSK_CUDA(cudaGetLastError());
        TSK_CUDA(cudaEventRecord(eks[c], st));
    };
    tr.mark("ranges");
    std::vector<int64_t> start((size_t)C + 1, 0);
    std::vector<char> copied((size_t)C, 0);
    const int64_t *qt = qc->traj, *qs = qc->seg;
    HostPool &pool = HostPool::get();
    // the query-id expansion runs on its own thread (with the host pool) so
    // the driving thread answers each chunk's count at once
    std::mutex xmu;
    std::condition_variable xcv;
    int x_ready = 0;  // chunks handed to the expander
    bool x_stop = false;
    std::thread expander([&] {
        int c = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(xmu);
                xcv.wait(lk, [&] { return c < x_ready || x_stop; });
                if (c >= x_ready) return;
            }
            if (copied[c]) {
                cudaEventSynchronize(evq[c]);
                const int64_t r0 = start[c], r1 = start[c + 1];
                pool.run([&](int part, int parts) {
                    const int64_t a = r0 + (r1 - r0) * part / parts, z = r0 + (r1 - r0) * (part + 1) / parts;
                    for (int64_t i = a; i < z; ++i) {
                        const uint32_t q = h_qo[i];
                        o_qt[i] = qt[q];
                        o_qs[i] = qs[q];
                    }
                });
                if (ids32) {
                    cudaEventSynchronize(evd[c]);
                    pool.run([&](int part, int parts) {
                        const int64_t a = r0 + (r1 - r0) * part / parts, z = r0 + (r1 - r0) * (part + 1) / parts;
                        for (int64_t i = a; i < z; ++i) {
                            o_et[i] = h_et32[i];
                            o_es[i] = h_es32[i];
                        }
                    });
                }
            }
            ++c;
        }
    });
    auto hand_over = [&](int upto) {
        std::lock_guard<std::mutex> g(xmu);
        x_ready = upto;
        xcv.notify_one();
    };
    auto finish_expander = [&]() {
        {
            std::lock_guard<std::mutex> g(xmu);
            x_stop = true;
            xcv.notify_one();
        }
        if (expander.joinable()) expander.join();
    };
    // a CUDA error thrown below must not leave the thread joinable
    // (std::thread's destructor would terminate the process)
    struct JoinGuard {
        const std::function<void()> fn;
        ~JoinGuard() { fn(); }
    } join_guard{[&] {
        if (!expander.joinable()) return;
        {
            std::lock_guard<std::mutex> g(xmu);
            x_ready = 0;  // skip chunks not expanded yet: the call is failing
            x_stop = true;
            xcv.notify_one();
        }
        expander.join();
    }};
    const int end_bit = bb + major_bits + minor_bits;
    enqueue_k1(0);
    bool overflow = false;
    for (int c = 0; c < C; ++c) {
        TSK_CUDA(cudaEventSynchronize(eks[c]));
        h_seen[c] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h_start).count();
        const unsigned long long end = snap[2 * c];
        if (end > cap || end >= max_hits_per_call()) {
            overflow = true;
            break;
        }
        start[c + 1] = (int64_t)end;
        const int64_t s0 = start[c], n = (int64_t)end - s0;
        if (n > 0) {
            sort_rows(db, L.keys + s0, ko + s0, v0 + s0, v1 + s0, n, end_bit, st, launches);
            const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
            k_compact<<<grid, 256, 0, st>>>(0, n, ko + s0, v1 + s0, L.tbeg + s0, L.tend + s0, plan.lo + B[c],
                                            plan.first + B[c], major_bits, minor_bits, db->s.traj, db->s.seg,
                                            d_tb + s0, d_te + s0,
                                            // 32-bit ids: int32 arrays at the same element offset
                                            ids32 ? reinterpret_cast<int64_t *>(reinterpret_cast<int32_t *>(d_et) + s0)
                                                  : d_et + s0,
                                            ids32 ? reinterpret_cast<int64_t *>(reinterpret_cast<int32_t *>(d_es) + s0)
                                                  : d_es + s0,
                                            d_qo + s0, ids32);
            TSK_CUDA(cudaGetLastError());
            ++launches;
            cudaEvent_t eg;
            TSK_CUDA(cudaEventCreateWithFlags(&eg, cudaEventDisableTiming));
            TSK_CUDA(cudaEventRecord(eg, st));
            if (trace) {
                TSK_CUDA(cudaEventCreate(&esd[c]));
                TSK_CUDA(cudaEventRecord(esd[c], st));
            }
            TSK_CUDA(cudaStreamWaitEvent(st2, eg, 0));
            TSK_CUDA(cudaEventDestroy(eg));  // destruction is deferred until the event completes
            // the query ordinals first: the expander gathers the query ids
            // while the chunk's other columns cross PCIe
            TSK_CUDA(cudaMemcpyAsync(h_qo + s0, d_qo + s0, (size_t)n * 4, cudaMemcpyDeviceToHost, st2));
            TSK_CUDA(cudaEventRecord(evq[c], st2));
            TSK_CUDA(cudaMemcpyAsync(o_tb + s0, d_tb + s0, (size_t)n * 8, cudaMemcpyDeviceToHost, st2));
            TSK_CUDA(cudaMemcpyAsync(o_te + s0, d_te + s0, (size_t)n * 8, cudaMemcpyDeviceToHost, st2));
            if (ids32) {
                TSK_CUDA(cudaMemcpyAsync(h_et32 + s0, reinterpret_cast<int32_t *>(d_et) + s0, (size_t)n * 4,
                                         cudaMemcpyDeviceToHost, st2));
                TSK_CUDA(cudaMemcpyAsync(h_es32 + s0, reinterpret_cast<int32_t *>(d_es) + s0, (size_t)n * 4,
                                         cudaMemcpyDeviceToHost, st2));
            } else {
                TSK_CUDA(cudaMemcpyAsync(o_et + s0, d_et + s0, (size_t)n * 8, cudaMemcpyDeviceToHost, st2));
                TSK_CUDA(cudaMemcpyAsync(o_es + s0, d_es + s0, (size_t)n * 8, cudaMemcpyDeviceToHost, st2));
            }
            TSK_CUDA(cudaEventRecord(evd[c], st2));
            copied[c] = 1;
        }
        if (c + 1 < C) enqueue_k1(c + 1);
        hand_over(c + 1);
    }
    if (overflow) {
        hand_over(0);
        finish_expander();
        TSK_CUDA(cudaStreamSynchronize(st));
        TSK_CUDA(cudaStreamSynchronize(st2));
        cleanup();
        pin_free(hb, hgot);
        return nullptr;
    }
    // the overlap counts (statistics only) once for the whole plan, behind
    // the last chunk's copy instead of on the K1 chain of every chunk
    if (L.ext_count) {
        launch_count_overlaps_ext(plan, db->q, db->s, L.q_unsorted, L.q_cmax_bits, L.db_cmax, L.d2, st);
        ++launches;
    }
    tr.mark("pipeline");
    finish_expander();
    const int64_t nh = start[C];
    tsk_result *res = new tsk_result();
    res->n = nh;
    res->nb = nb;
    res->k1_evals = (int64_t)snap[2 * (C - 1) + 1];
    float k1_ms = 0.f;
    for (int c = 0; c < C; ++c) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ek0[c], ek1[c]);
        k1_ms += ms;
    }
    res->k1_ms = k1_ms;
    size_t pb_got = 0;
    const size_t nbz = (size_t)nb;
    res->pb_host = static_cast<int64_t *>(pin_alloc(nbz * 4 * 8, &pb_got));
    res->pb_bytes = pb_got;
    TSK_CUDA(cudaMemcpyAsync(res->pb_host, plan.first, nbz * 16, cudaMemcpyDeviceToHost, st));
    TSK_CUDA(cudaMemcpyAsync(res->pb_host + 2 * nbz, plan.ovl, nbz * 16, cudaMemcpyDeviceToHost, st));
    res->host = hb;
    res->host_bytes = hgot;
    res->qtraj = o_qt;
    res->qseg = o_qs;
    res->etraj = o_et;
    res->eseg = o_es;
    res->tbeg = o_tb;
    res->tend = o_te;
    for (int c = C - 1; c >= 0; --c)
        if (copied[c]) {
            TSK_CUDA(cudaStreamWaitEvent(st, evd[c], 0));
            break;
        }
    TSK_CUDA(cudaEventRecord(db->ev1, st));
    TSK_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, db->ev0, db->ev1);
    res->device_ms = ms;
    res->launches = launches;
    db->last_hits = nh;
    db->last_k1_ms = k1_ms;
    if (trace) {
        auto at = [&](cudaEvent_t e) {
            float t = -1.f;
            if (e) cudaEventElapsedTime(&t, db->ev0, e);
            return t;
        };
        fprintf(stderr, "[tsk trace] pipeline %d chunks, %lld rows (ms from start: K1 begin-end / host saw / S end / D2H end):", C,
                (long long)nh);
        for (int c = 0; c < C; ++c)
            fprintf(stderr, " [%.2f-%.2f / %.2f / %.2f / %.2f]", at(ek0[c]), at(ek1[c]), h_seen[c], at(esd[c]),
                    copied[c] ? at(evd[c]) : -1.f);
        fprintf(stderr, "\n");
    }
    cleanup();
    return res;
}

static tsk_result *run(tsk_db *db, const tsk_columns *qc, int64_t nb, const int64_t *b_lo,
                       const int64_t *b_hi, const int64_t *b_first, const int64_t *b_last, double d,
                       uint32_t flags) {
    TSK_REQUIRE(std::isfinite(d) && d >= 0.0, "threshold d must be finite and non-negative");
    TSK_REQUIRE(qc && qc->n > 0, "query set is empty");
    TSK_REQUIRE(nb >= 1 && b_lo && b_hi, "a plan needs at least one batch");
    const bool spans_given = flags & TSK_SPANS_GIVEN;
    const int64_t nq = qc->n, n = db->s.n;
    int64_t max_s = 1;
    for (int64_t b = 0; b < nb; ++b) {
        TSK_REQUIRE(b_lo[b] >= 0 && b_lo[b] <= b_hi[b] && b_hi[b] < nq, "batch outside the query set");
        max_s = std::max<int64_t>(max_s, b_hi[b] - b_lo[b] + 1);
        if (spans_given) {
            TSK_REQUIRE(b_first && b_last, "spans missing");
            if (b_first[b] >= 0 || b_last[b] >= 0)
                TSK_REQUIRE(0 <= b_first[b] && b_first[b] <= b_last[b] && b_last[b] < n,
                            "candidate span outside store");
        }
    }
    TSK_CUDA(cudaSetDevice(db->device));
    cudaStream_t st = db->stream;
    const bool query_major = flags & TSK_ORDER_QUERY_MAJOR;
    const bool canonical = flags & TSK_ORDER_CANONICAL;
    TSK_REQUIRE(!(canonical && (flags & TSK_WANT_ORDINALS)), "canonical order does not carry ordinals");
    const bool ordered = query_major || (flags & TSK_ORDER_REFERENCE);
    const int bb = bits_for(nb);
    const int eb = bits_for(std::max<int64_t>(n, 1)), qb = bits_for(max_s);
    const int major_bits = query_major ? qb : eb, minor_bits = query_major ? eb : qb;
    TSK_REQUIRE(bb + major_bits + minor_bits <= 64, "result key wider than 64 bits");

    int64_t launches = 0;
    // pinned staging of pageable query columns, returned to the pool when the
    // call returns (every return path has synchronised the stream)
    struct Stage {
        void *p = nullptr;
        size_t bytes = 0;
        ~Stage() { pin_free(p, bytes); }
    } stage;
    Trace tr(st);
    tr.mark("start");
    TSK_CUDA(cudaEventRecord(db->ev0, st));
    if (flags & TSK_QUERIES_RESIDENT) {
        TSK_REQUIRE(db->q.n == nq && db->q_rec.p, "no resident query set of this size");
    } else {
        // queries → device SoA → shared-memory records with hoisted invariants
        soa_alloc(db->q, nq, true, st);
        db->q_rec.reserve((size_t)nq * sizeof(QRec), st);
        db->counters.reserve(64, st);
        tsk_columns mapped;
        if (mapped_columns(qc, &mapped)) {  // pinned inputs: one kernel reads them over PCIe
            launch_qprep_mapped(mapped, db->q, db->q_rec.as<QRec>(), db->counters.as<int>() + 8,
                                db->counters.as<unsigned long long>() + 5, st);
        } else {
            // pageable inputs (plain numpy): host threads copy the columns
            // into a pooled pinned block, which the kernel then reads over
            // PCIe like pinned inputs (a pageable cudaMemcpy runs at a
            // fraction of the bus rate through the driver's bounce buffer)
            const size_t cb = (size_t)nq * 8;
            stage.p = pin_alloc(cb * 10, &stage.bytes);
            char *sb = static_cast<char *>(stage.p);
            const void *src[10] = {qc->traj, qc->seg, qc->xs, qc->ys, qc->zs, qc->ts, qc->xe, qc->ye, qc->ze, qc->te};
            HostPool::get().run([&](int part, int parts) {
                const size_t a = cb * part / parts & ~size_t(63), z = part + 1 == parts ? cb : cb * (part + 1) / parts & ~size_t(63);
                for (int k = 0; k < 10; ++k)
                    if (src[k] && z > a) memcpy(sb + k * cb + a, static_cast<const char *>(src[k]) + a, z - a);
            });
            tsk_columns staged = *qc;
            staged.traj = qc->traj ? (const int64_t *)(sb + 0 * cb) : nullptr;
            staged.seg = qc->seg ? (const int64_t *)(sb + 1 * cb) : nullptr;
            staged.xs = (const double *)(sb + 2 * cb);
            staged.ys = (const double *)(sb + 3 * cb);
            staged.zs = (const double *)(sb + 4 * cb);
            staged.ts = (const double *)(sb + 5 * cb);
            staged.xe = (const double *)(sb + 6 * cb);
            staged.ye = (const double *)(sb + 7 * cb);
            staged.ze = (const double *)(sb + 8 * cb);
            staged.te = (const double *)(sb + 9 * cb);
            if (qc->traj && mapped_columns(&staged, &mapped)) {
                launch_qprep_mapped(mapped, db->q, db->q_rec.as<QRec>(), db->counters.as<int>() + 8,
                                    db->counters.as<unsigned long long>() + 5, st);
            } else {
                soa_upload(db->q, &staged, st);
                launch_qprep(db->q, db->q_rec.as<QRec>(), db->counters.as<int>() + 8,
                             db->counters.as<unsigned long long>() + 5, st);
            }
        }
        launches += 1;
    }
    tr.mark("queries");

    // batch table: lo hi first last item_off(units+1) meta(4) ovl hits
    size_t nbz = (size_t)nb;
    const size_t nuz = (size_t)plan_units(nb);
    db->batches.reserve((nbz * 6 + nuz + 8) * 8, st);
    int64_t *d_lo = db->batches.as<int64_t>();
    int64_t *d_hi = d_lo + nbz, *d_first = d_hi + nbz, *d_last = d_first + nbz;
    int64_t *d_off = d_last + nbz, *d_meta = d_off + nuz + 1;
    unsigned long long *d_ovl = (unsigned long long *)(d_meta + 4);
    unsigned long long *d_hits = d_ovl + nbz;
    TSK_CUDA(cudaMemcpyAsync(d_lo, b_lo, nbz * 8, cudaMemcpyHostToDevice, st));
    TSK_CUDA(cudaMemcpyAsync(d_hi, b_hi, nbz * 8, cudaMemcpyHostToDevice, st));
    if (spans_given) {
        TSK_CUDA(cudaMemcpyAsync(d_first, b_first, nbz * 8, cudaMemcpyHostToDevice, st));
        TSK_CUDA(cudaMemcpyAsync(d_last, b_last, nbz * 8, cudaMemcpyHostToDevice, st));
    }
    SearchPlanDev plan{nb, d_lo, d_hi, d_first, d_last, d_off, d_meta, d_ovl, d_hits};
    launch_ranges(db, db->q, plan, spans_given, st);
    const bool k1_f32 = k1_use_f32(d * d, db->cmax);
    const int bps = k1_blocks_per_sm(k1_f32);
    int slots = sm_count(db->device) * bps;
    // batch pairs share candidate tiles in the FP32 kernel (not in the
    // FP64 fallback kernel or for brute force's query-major keys)
    // TSK_K1_PAIR=off|force (testing) disables pairing or forces it on
    // small plans (full query tiles)
    int pair = (k1_f32 && !query_major) ? 1 : 0;
    if (const char *e = getenv("TSK_K1_PAIR")) {
        if (!strcmp(e, "off")) pair = 0;
        else if (!strcmp(e, "force") && pair) pair = 2;
    }
    // indexed searches read K1's spatially ordered copy of the store (its
    // candidate ranges are unions of whole bins, so the same ordinal ranges)
    // and cull (query, warp) pairs by box; spans given by the caller are
    // arbitrary and use the start-sorted store.  TSK_SPATIAL=nocull keeps the
    // layout without the cull (testing).
    const char *sp_env = getenv("TSK_SPATIAL");
    const bool use_k = !spans_given && db->k.built;
    const int cull = (use_k && !(sp_env && !strcmp(sp_env, "nocull"))) ? 1 : 0;
    int k1_stride = K1_THREADS * k1_candidates_per_thread(k1_f32);
    const int k1_align = cull ? BOX_GROUP : 1;
    int k1_tq_max = k1_f32 ? K1_TQ : K1P_TQ;
    launches += spans_given ? 0 : 1;

    db->counters.reserve(64, st);
    unsigned long long *d_ctr = db->counters.as<unsigned long long>();  // [0] items [1] hits; int[8] = q unsorted
    uint64_t cap = db->recs.bytes / 24;
    if (cap < (uint64_t(1) << 20)) {
        db->recs.reserve((size_t(1) << 20) * 24, st);
        cap = db->recs.bytes / 24;
    }
    K1Launch L;
    L.e = use_k ? db->k.s : db->s;
    L.orig = use_k ? db->k.orig : nullptr;
    L.gbox = use_k ? db->k.box : nullptr;
    L.gtime = use_k ? db->k.gtime : nullptr;
    L.frec = use_k && !getenv("TSK_NO_FREC") ? db->k.frec : nullptr;  // TSK_NO_FREC: testing
    L.gorig = use_k ? db->k.gorig : nullptr;
    L.cull = cull;
    // overlap counts outside K1 (count_overlaps_ext) when the store's end
    // times are sorted too; the kernel itself checks the query flags
    L.ext_count = (L.cull && k1_f32 && db->s.te_sorted && !(flags & (TSK_OVERLAPS_ONLY | TSK_NOOP)) &&
                   !(sp_env && !strcmp(sp_env, "noext")))
                      ? 1
                      : 0;
    L.q = db->q_rec.as<QRec>();
    L.plan = plan;
    L.item_counter = d_ctr;
    L.hit_count = d_ctr + 1;
    L.eval_count = d_ctr + 2;
    L.d2 = d * d;  // core.py:527
    // filter margin scale: entry max |coordinate| here, the query one is
    // reduced on the device by qprep and folded in by K1
    L.db_cmax = db->cmax;
    L.filter_km = 0x1p-35 - 1.0;
    L.q_cmax_bits = db->counters.as<unsigned long long>() + 5;
    L.major_bits = major_bits;
    L.minor_bits = minor_bits;
    L.query_major = query_major;
    L.noop = (flags & TSK_NOOP) ? 1 : 0;
    L.overlaps_only = (flags & TSK_OVERLAPS_ONLY) ? 1 : 0;
    // counts only: no hit rows are written (cap 0), so no regrow and no K4
    const bool count_only = flags & (TSK_COUNT_ONLY | TSK_OVERLAPS_ONLY);
    L.q_unsorted = db->counters.as<int>() + 8;
    // quads of batches per tile when every item takes the box-cull fast path
    // (k_plan_items confirms the query order on the device); TSK_K1_QUADS=off
    // (testing) keeps pairs
    {
        const char *qe = getenv("TSK_K1_QUADS");
        if (pair == 1 && L.cull && L.ext_count && k1_tq_max >= 512 && !(qe && !strcmp(qe, "off")))
            pair = (qe && !strcmp(qe, "force")) ? 5 : 4;  // force: quads on small plans too (testing)
        // octets in the wide kernel (1,024-query tiles, one CTA per SM) for
        // plans with enough groups of 8 to fill the grid; TSK_K1_WIDE=off|force
        // (testing: force takes it on any plan quads would take)
        const char *we = getenv("TSK_K1_WIDE");
        bool wide = (pair == 4 || pair == 5) && nb >= kWideMinBatches;
        if (we && !strcmp(we, "off")) wide = false;
        if (we && !strcmp(we, "force") && (pair == 4 || pair == 5)) wide = true;
        if (wide) {
            L.wide = 1;
            pair = pair == 5 ? 9 : 8;
            slots = sm_count(db->device) * k1f_blocks_per_sm_wide();
            k1_stride = K1W_THREADS * k1_candidates_per_thread(true);
            k1_tq_max = K1W_TQ;
        }
    }
    // reference-ordered results through the compact path: K1 chunk by chunk,
    // each chunk's rows sorted, gathered and copied while later chunks run
    const bool on_device_early = flags & TSK_RESULTS_ON_DEVICE;
    if (!count_only && !L.noop && ordered && !query_major && !canonical && !(flags & TSK_WANT_ORDINALS) &&
        !on_device_early && qc->traj && qc->seg && nq <= 0xffffffffll) {
        tsk_result *pres = run_pipelined(db, qc, plan, L, slots, k1_stride, pair, k1_align, k1_tq_max, major_bits, minor_bits,
                                         bb, cap, tr, launches);
        if (pres) return pres;
        // a chunk overflowed the result buffer: the plain path below sizes it
        // exactly (and the next call's pipeline fits)
    }
    launch_plan_items(plan, slots, k1_stride, pair, k1_align, k1_tq_max, L.q_unsorted, st);
    ++launches;
    tr.mark("ranges+items");
    unsigned long long h_ctr[2] = {0, 0};  // hits, evaluated pairs
    unsigned long long &h_hits = h_ctr[0];
    float k1_ms = 0.f;
    for (int attempt = 0;; ++attempt) {
        L.cap = count_only ? 0 : cap;
        L.keys = db->recs.as<uint64_t>();
        L.tbeg = reinterpret_cast<double *>(L.keys + cap);
        L.tend = L.tbeg + cap;
        TSK_CUDA(cudaMemsetAsync(d_ctr, 0, 24, st));
        TSK_CUDA(cudaMemsetAsync(d_ovl, 0, nbz * 16, st));
        if (L.ext_count) {
            launch_count_overlaps_ext(plan, db->q, db->s, L.q_unsorted, L.q_cmax_bits, L.db_cmax, L.d2, st);
            ++launches;
        }
        TSK_CUDA(cudaEventRecord(db->ev_k0, st));
        launch_k1(L, slots, st);
        ++launches;
        TSK_CUDA(cudaEventRecord(db->ev_k1, st));
        TSK_CUDA(cudaMemcpyAsync(h_ctr, d_ctr + 1, 16, cudaMemcpyDeviceToHost, st));
        TSK_CUDA(cudaStreamSynchronize(st));
        tr.mark("k1");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, db->ev_k0, db->ev_k1);
        k1_ms += ms;
        if (count_only || h_hits <= cap) break;
        TSK_REQUIRE(attempt < 3, "result buffer kept overflowing");
        // overflow-safe sizing: grow to the exact count and rerun K1
        db->recs.reserve((size_t)h_hits * 24 + 24 * 1024, st);
        cap = db->recs.bytes / 24;
    }
    if (!count_only && h_hits >= max_hits_per_call())
        throw Error{TSK_ETOOMANY, "more than " + std::to_string(max_hits_per_call()) +
                                      " hits in one call (the row permutation is 32-bit): split the plan"};
    const int64_t nh = count_only ? 0 : (int64_t)h_hits;
    if (!count_only) {
        db->last_hits = nh;
        db->last_k1_ms = k1_ms;
    }

    tsk_result *res = new tsk_result();
    res->n = nh;
    res->nb = nb;
    res->k1_ms = k1_ms;
    res->k1_evals = (int64_t)h_ctr[1];
    // per-batch first/last/ovl/hits are contiguous on the device (d_first .. d_hits
    // are laid out first,last,item_off,meta,ovl,hits): copy first/last and ovl/hits
    size_t pb_got = 0;
    res->pb_host = static_cast<int64_t *>(pin_alloc(nbz * 4 * 8, &pb_got));
    res->pb_bytes = pb_got;
    TSK_CUDA(cudaMemcpyAsync(res->pb_host, d_first, nbz * 16, cudaMemcpyDeviceToHost, st));
    TSK_CUDA(cudaMemcpyAsync(res->pb_host + 2 * nbz, d_ovl, nbz * 16, cudaMemcpyDeviceToHost, st));
    const bool want_ord = flags & TSK_WANT_ORDINALS;
    const bool on_device = flags & TSK_RESULTS_ON_DEVICE;
    const int ncols = want_ord ? 8 : 6;
    size_t cb = (size_t)nh * 8;
    // the pinned host block is taken after K4 is enqueued, so a fresh
    // registration (large results) overlaps the device's sort and gather
    auto host_block = [&]() {
        size_t got = 0;
        res->host = on_device ? nullptr : pin_alloc((size_t)(nh > 0 ? nh : 1) * 8 * ncols, &got);
        res->host_bytes = got;
        char *hb = static_cast<char *>(res->host);
        if (hb) {
            res->qtraj = (int64_t *)(hb + 0 * cb);
            res->qseg = (int64_t *)(hb + 1 * cb);
            res->etraj = (int64_t *)(hb + 2 * cb);
            res->eseg = (int64_t *)(hb + 3 * cb);
            res->tbeg = (double *)(hb + 4 * cb);
            res->tend = (double *)(hb + 5 * cb);
        }
        if (hb && want_ord) {
            res->qord = (int64_t *)(hb + 6 * cb);
            res->eord = (int64_t *)(hb + 7 * cb);
        }
    };
    if (nh == 0) host_block();
    if (nh > 0) {
        const uint64_t *keys = db->recs.as<uint64_t>();
        const double *tbin = reinterpret_cast<const double *>(keys + cap);
        const double *tein = tbin + cap;
        const uint32_t *perm = nullptr;
        if (ordered) {
            // K4: radix sort (batch, major, minor) keys; values = append index
            db->sorted.reserve((size_t)nh * (8 + 8 + 4 + 4), st);
            uint64_t *ks = db->sorted.as<uint64_t>();
            uint64_t *ko = ks + nh;
            uint32_t *v0 = reinterpret_cast<uint32_t *>(ko + nh);
            uint32_t *v1 = v0 + nh;
            if (nh <= K4_SMALL) {
                k_small_sort<<<1, 1024, 0, st>>>((int)nh, keys, ko, v1);
                TSK_CUDA(cudaGetLastError());
                ++launches;
            } else {
                int gi = (int)std::min<int64_t>((nh + 255) / 256, 148 * 8);
                k_iota<<<gi, 256, 0, st>>>(nh, v0);
                TSK_CUDA(cudaGetLastError());
                ++launches;
                TSK_CUDA(cudaMemcpyAsync(ks, keys, cb, cudaMemcpyDeviceToDevice, st));
                int end_bit = bb + major_bits + minor_bits;
                if (end_bit == 0) end_bit = 1;
                size_t tb = 0;
                TSK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ks, ko, v0, v1, nh, 0, end_bit, st));
                db->cub_tmp.reserve(tb, st);
                TSK_CUDA(cub::DeviceRadixSort::SortPairs(db->cub_tmp.p, tb, ks, ko, v0, v1, nh, 0, end_bit, st));
            }
            keys = ko;
            perm = v1;
        }
        // compact rows + host expansion of the ids, pipelined in chunks over
        // a second stream (large reference-ordered results of indexed and
        // span searches; the caller registered the store's host id columns)
        const char *cpenv = getenv("TSK_COMPACT");
        const bool compact = !on_device && !canonical && !want_ord && ordered && !query_major &&
                             qc->traj && qc->seg && n <= 0xffffffffll &&
                             nq <= 0xffffffffll &&
                             (cpenv ? strcmp(cpenv, "off") != 0 : nh >= kCompactMin) &&
                             !(cpenv && !strcmp(cpenv, "off"));
        if (compact) {
            tr.mark("sort");
            compact_rows(db, res, qc, nh, keys, perm, tbin, tein, d_lo, d_first, major_bits, minor_bits, st,
                         launches);
            tr.mark("d2h");
            TSK_CUDA(cudaEventRecord(db->ev1, st));
            TSK_CUDA(cudaStreamSynchronize(st));
            float ms = 0.f;
            cudaEventElapsedTime(&ms, db->ev0, db->ev1);
            res->device_ms = ms;
            res->launches = launches;
            return res;
        }
        db->out_cols.reserve(cb * ncols, st);
        char *ob = db->out_cols.as<char>();
        GatherArgs g;
        g.n = nh;
        g.keys = keys;
        g.perm = perm;
        g.tb_in = tbin;
        g.te_in = tein;
        g.lo = d_lo;
        g.first = d_first;
        g.qtraj = db->q.traj;
        g.qseg = db->q.seg;
        g.etraj = db->s.traj;
        g.eseg = db->s.seg;
        g.o_qtraj = (int64_t *)(ob + 0 * cb);
        g.o_qseg = (int64_t *)(ob + 1 * cb);
        g.o_etraj = (int64_t *)(ob + 2 * cb);
        g.o_eseg = (int64_t *)(ob + 3 * cb);
        g.o_tb = (double *)(ob + 4 * cb);
        g.o_te = (double *)(ob + 5 * cb);
        g.o_qord = want_ord ? (int64_t *)(ob + 6 * cb) : nullptr;
        g.o_eord = want_ord ? (int64_t *)(ob + 7 * cb) : nullptr;
        g.major_bits = major_bits;
        g.minor_bits = minor_bits;
        g.query_major = query_major;
        int gg = (int)std::min<int64_t>((nh + 255) / 256, 148 * 8);
        tr.mark("sort");
        k_gather<<<gg, 256, 0, st>>>(g);
        TSK_CUDA(cudaGetLastError());
        ++launches;
        tr.mark("gather");
        if (canonical) {
            // ResultSet.canonical_order on the device (core.py:290-294)
            db->canon_cols.reserve(cb * 6 + (size_t)nh * 4 + 64, st);
            char *cbuf = db->canon_cols.as<char>();
            uint32_t *perm = reinterpret_cast<uint32_t *>(cbuf + 6 * cb);
            canonical_perm(nh, g.o_qtraj, g.o_qseg, g.o_etraj, g.o_eseg, g.o_tb, g.o_te, perm,
                           db->canon_tmp, st);
            const int64_t *in_i[4] = {g.o_qtraj, g.o_qseg, g.o_etraj, g.o_eseg};
            const double *in_f[2] = {g.o_tb, g.o_te};
            int64_t *out_i[4] = {(int64_t *)(cbuf + 0 * cb), (int64_t *)(cbuf + 1 * cb),
                                 (int64_t *)(cbuf + 2 * cb), (int64_t *)(cbuf + 3 * cb)};
            double *out_f[2] = {(double *)(cbuf + 4 * cb), (double *)(cbuf + 5 * cb)};
            permute6(nh, perm, in_i, in_f, out_i, out_f, st);
            ob = cbuf;
            tr.mark("canonical");
        }
        host_block();
        if (!on_device) TSK_CUDA(cudaMemcpyAsync(res->host, ob, cb * ncols, cudaMemcpyDeviceToHost, st));
        tr.mark("d2h");
    }
    TSK_CUDA(cudaEventRecord(db->ev1, st));
    TSK_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, db->ev0, db->ev1);
    res->device_ms = ms;
    res->launches = launches;
    return res;
}

}  // namespace tsk

using namespace tsk;

extern "C" int tsk_abi_version(void) { return TSK_ABI_VERSION; }

extern "C" int tsk_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" const char *tsk_last_error(void) { return g_last_error.c_str(); }

extern "C" int tsk_search(tsk_db *db, const tsk_columns *queries, int64_t nb, const int64_t *b_lo,
                          const int64_t *b_hi, const int64_t *b_first, const int64_t *b_last,
                          double d, uint32_t flags, tsk_result **out) {
    try {
        TSK_REQUIRE(db && out, "null argument");
        *out = run(db, queries, nb, b_lo, b_hi, b_first, b_last, d, flags);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_pair_intervals(int device, const tsk_columns *rows, const tsk_columns *cols,
                                  double d, tsk_result **out) {
    tsk_db *db = nullptr;
    try {
        TSK_REQUIRE(rows && cols && out, "null argument");
        TSK_REQUIRE(std::isfinite(d) && d >= 0.0, "threshold d must be finite and non-negative");
        TSK_REQUIRE(rows->n > 0 && cols->n > 0, "pair_intervals needs non-empty stores");
        int rc = tsk_db_create(device, rows, &db);
        if (rc != TSK_OK) return rc;
        int64_t lo = 0, hi = cols->n - 1, first = 0, last = rows->n - 1;
        *out = run(db, cols, 1, &lo, &hi, &first, &last, d,
                   TSK_SPANS_GIVEN | TSK_ORDER_REFERENCE | TSK_WANT_ORDINALS);
        tsk_db_free(db);
        return TSK_OK;
    } catch (const Error &e) {
        if (db) tsk_db_free(db);
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_db_set_host_ids(tsk_db *db, const int64_t *traj, const int64_t *seg) {
    if (!db) return fail(TSK_EINVAL, "null db");
    if ((traj == nullptr) != (seg == nullptr)) return fail(TSK_EINVAL, "traj and seg go together");
    db->host_etraj = traj;
    db->host_eseg = seg;
    return TSK_OK;
}

extern "C" int tsk_result_info(const tsk_result *r, int64_t *n_hits, int64_t *nb, double *device_ms) {
    if (!r) return fail(TSK_EINVAL, "null result");
    if (n_hits) *n_hits = r->n;
    if (nb) *nb = r->nb;
    if (device_ms) *device_ms = r->device_ms;
    return TSK_OK;
}

extern "C" int tsk_result_k1_evals(const tsk_result *r, int64_t *evals) {
    if (!r || !evals) return fail(TSK_EINVAL, "null argument");
    *evals = r->k1_evals;
    return TSK_OK;
}

extern "C" int tsk_result_timing(const tsk_result *r, double *device_ms, double *k1_ms,
                                 int64_t *launches) {
    if (!r) return fail(TSK_EINVAL, "null result");
    if (device_ms) *device_ms = r->device_ms;
    if (k1_ms) *k1_ms = r->k1_ms;
    if (launches) *launches = r->launches;
    return TSK_OK;
}

extern "C" int tsk_result_per_batch(const tsk_result *r, int64_t *per_batch) {
    if (!r || !per_batch) return fail(TSK_EINVAL, "null argument");
    // stored column-wise (first[], last[], ovl[], hits[]); returned row-wise
    const int64_t nb = r->nb;
    for (int64_t b = 0; b < nb; ++b)
        for (int k = 0; k < 4; ++k) per_batch[b * 4 + k] = r->pb_host[k * nb + b];
    return TSK_OK;
}

extern "C" int tsk_result_columns(const tsk_result *r, const int64_t **query_traj,
                                  const int64_t **query_seg, const int64_t **entry_traj,
                                  const int64_t **entry_seg, const double **t_begin,
                                  const double **t_end, const int64_t **query_ord,
                                  const int64_t **entry_ord) {
    if (!r) return fail(TSK_EINVAL, "null result");
    if (query_traj) *query_traj = r->qtraj;
    if (query_seg) *query_seg = r->qseg;
    if (entry_traj) *entry_traj = r->etraj;
    if (entry_seg) *entry_seg = r->eseg;
    if (t_begin) *t_begin = r->tbeg;
    if (t_end) *t_end = r->tend;
    if (query_ord) *query_ord = r->qord;
    if (entry_ord) *entry_ord = r->eord;
    return TSK_OK;
}

extern "C" void tsk_result_free(tsk_result *r) {
    if (!r) return;
    pin_free(r->host, r->host_bytes);
    pin_free(r->pb_host, r->pb_bytes);
    delete r;
}

extern "C" void *tsk_pinned_alloc(int64_t bytes) {
    void *p = nullptr;
    if (bytes <= 0) bytes = 64;
    if (cudaHostAlloc(&p, (size_t)bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaHostAlloc failed");
        return nullptr;
    }
    return p;
}

extern "C" void tsk_pinned_free(void *p) {
    if (p) cudaFreeHost(p);
}
