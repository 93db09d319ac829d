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

static void *pin_alloc(size_t bytes, size_t *got) {
    if (bytes == 0) bytes = 64;
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
                          int64_t *__restrict__ o_es, uint32_t *__restrict__ o_qo) {
    const uint64_t mmask = major_bits ? ((~0ull) >> (64 - major_bits)) : 0ull;
    const uint64_t nmask = minor_bits ? ((~0ull) >> (64 - minor_bits)) : 0ull;
    for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const int64_t b = (int64_t)(major_bits + minor_bits < 64 ? (k >> (major_bits + minor_bits)) : 0);
        const int64_t e = first[b] + (int64_t)((k >> minor_bits) & mmask);
        const int64_t q = lo[b] + (int64_t)(k & nmask);
        const int64_t j = perm ? (int64_t)perm[i] : i;
        o_et[i] = etraj[e];
        o_es[i] = eseg[e];
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
static const int64_t kCompactMin = int64_t(1) << 18;
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
        TSK_CUDA(cudaEventCreateWithFlags(&evd[c], cudaEventDisableTiming | cudaEventBlockingSync));
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t r0 = c * chunk, r1 = std::min<int64_t>(nh, r0 + chunk), m = r1 - r0;
        const int grid = (int)std::min<int64_t>((m + 255) / 256, 148 * 8);
        k_compact<<<grid, 256, 0, st>>>(r0, r1, keys, perm, tbin, tein, d_lo, d_first, major_bits, minor_bits,
                                        db->s.traj, db->s.seg, d_tb, d_te, d_et, d_es, d_qo);
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
            soa_upload(db->q, qc, st);
            launch_qprep(db->q, db->q_rec.as<QRec>(), db->counters.as<int>() + 8,
                         db->counters.as<unsigned long long>() + 5, st);
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
    const int slots = sm_count(db->device) * bps;
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
    launch_plan_items(plan, slots, K1_THREADS * k1_candidates_per_thread(k1_f32), pair, cull ? BOX_GROUP : 1, st);
    launches += spans_given ? 1 : 2;
    tr.mark("ranges+items");

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
    TSK_REQUIRE(count_only || h_hits < (1ull << 32), "more than 2^32 hits in one call");
    const int64_t nh = count_only ? 0 : (int64_t)h_hits;

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
