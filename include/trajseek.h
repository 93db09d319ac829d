/*
 * trajseek.h — C-ABI of libtrajseek.so, the B200 (sm_100a) engine behind the
 * distance-threshold search path of arXiv 1405.7461 (GPUTrajDistSearch).
 *
 * The reference (`trajseek`, pure Python + numpy) has no native boundary;
 * each entry point below replaces one reference Python function on the hot
 * path (paths relative to /root/reference/pkg/src/trajseek/):
 *
 *   tsk_db_create / tsk_db_free   SegmentStore residency (core.py:121-243);
 *                                 the device SoA + hoisted per-segment invariants
 *   tsk_sort_by_start             SegmentStore stable sort (core.py:162-166)
 *   tsk_index_build / _copy       build_index (index.py:85-146)            [K2]
 *   tsk_candidate_ranges          candidate_range (index.py:149-173)       [K3]
 *   tsk_search                    run_search (engine.py:151-204) and
 *                                 execute_batch (engine.py:97-148)        [K1+K4]
 *   tsk_pair_intervals            pair_intervals (core.py:464-565)          [K1]
 *
 * Conventions: plain pointers and sizes only; host arrays are owned by the
 * caller (numpy); every function returns TSK_OK or an error code and the
 * thread-local message is available from tsk_last_error().  A handle is
 * thread-compatible (one host thread at a time per handle).
 */
#ifndef TRAJSEEK_H
#define TRAJSEEK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSK_ABI_VERSION 1

enum {
    TSK_OK = 0,
    TSK_EINVAL = 1,  /* precondition violated → DomainError (core.py:25-26) */
    TSK_ECUDA = 2,   /* CUDA runtime failure → RuntimeError              */
    TSK_ENOMEM = 3,  /* allocation failure → MemoryError                 */
    TSK_ENODEV = 4,  /* no CUDA device                                   */
    TSK_EFORMAT = 5, /* unparsable / invalid CSV → FormatError (core.py:29-30) */
    TSK_ETOOMANY = 6 /* more hits than one call returns (2^32): split the plan and call again */
};

/* tsk_search flags */
enum {
    TSK_NOOP = 1u << 0,          /* launch with pair arithmetic elided (engine.py:86-88,207-224) */
    TSK_ORDER_REFERENCE = 1u << 1,/* items in the reference order: (batch, entry, query)          */
    TSK_ORDER_QUERY_MAJOR = 1u << 2,/* items ordered (query, entry) as brute_force (oracle.py:26) */
    TSK_SPANS_GIVEN = 1u << 3,   /* b_first/b_last supplied by the caller (execute_batch)        */
    TSK_WANT_ORDINALS = 1u << 4, /* also return query/entry ordinals (pair_intervals)            */
    TSK_QUERIES_RESIDENT = 1u << 5,/* reuse the query set uploaded by the previous call on this db */
    TSK_RESULTS_ON_DEVICE = 1u << 6,/* leave hit columns in HBM (no D2H): device-throughput runs */
    TSK_ORDER_CANONICAL = 1u << 7,/* items in ResultSet.canonical_order (core.py:290-294)        */
    TSK_COUNT_ONLY = 1u << 8,    /* per-batch overlap/hit counts only; no result rows (perfmodel) */
    TSK_OVERLAPS_ONLY = 1u << 9  /* per-batch temporal overlaps only (perfmodel.py:327-343)      */
};

/* Index extent rules (index.py:26) */
enum { TSK_EXTENT_MEMBER = 0, TSK_EXTENT_GRID = 1 };

/* One segment store in SoA form: 2 int64 id columns + 8 float64 columns,
 * sorted by non-decreasing ts (SegmentStore, core.py:121-166). */
typedef struct tsk_columns {
    int64_t n;
    const int64_t *traj, *seg;
    const double *xs, *ys, *zs, *ts, *xe, *ye, *ze, *te;
} tsk_columns;

typedef struct tsk_db tsk_db;         /* device-resident entry store (+ index) */
typedef struct tsk_result tsk_result; /* search output (pinned host columns)   */

int tsk_abi_version(void);
int tsk_device_count(void);
const char *tsk_last_error(void);

/* Upload a sorted store to `device` and hoist per-segment invariants. */
int tsk_db_create(int device, const tsk_columns *cols, tsk_db **out);
void tsk_db_free(tsk_db *db);
/* Replica of `src` on `device` (device-to-device copy, NVLink peer copy
 * between GPUs); build its index with tsk_index_build. */
int tsk_db_replicate(const tsk_db *src, int device, tsk_db **out);
int64_t tsk_db_size(const tsk_db *db);
/* Register caller-owned host copies of the store's traj/seg id columns
 * (start-sorted order, n each; NULL, NULL clears).  With them, large
 * reference-ordered results cross PCIe as 24-byte (ordinals, interval)
 * rows and the ids are expanded on host threads, pipelined with the copy
 * (engine.py:136-141's id gather).  The arrays must outlive the handle or
 * be cleared first. */
int tsk_db_set_host_ids(tsk_db *db, const int64_t *traj, const int64_t *seg);

/* Stable device sort of n start times: perm[i] = input row of sorted row i
 * (numpy argsort kind="stable", core.py:163). */
int tsk_sort_by_start(int device, int64_t n, const double *ts, int64_t *perm);

/* [K2] Build the m-bin temporal index on the device (index.py:85-146).
 * hdr receives {bin_width, t0, t_max}; *n_nonempty the non-empty bin count.
 * The index stays on the db handle and serves tsk_candidate_ranges/tsk_search. */
int tsk_index_build(tsk_db *db, int64_t m, int extent_rule, int64_t *n_nonempty, double *hdr);
/* Copy the non-empty-bin arrays (each n_nonempty long); bin_id = bin number j. */
int tsk_index_copy(const tsk_db *db, double *ne_start, double *ne_end, int64_t *ne_first,
                   int64_t *ne_last, int64_t *bin_id);

/* [K3] Candidate ranges of k closed intervals; (-1,-1) where none qualifies. */
int tsk_candidate_ranges(tsk_db *db, int64_t k, const double *begin, const double *end,
                         int64_t *first, int64_t *last);

/* [K1+K3+K4] Evaluate a batch plan.  Batch b holds query ordinals
 * b_lo[b]..b_hi[b] (contiguous, ascending).  Without TSK_SPANS_GIVEN the
 * candidate span of each batch comes from the db's index (K3, engine.py:177-179);
 * with it, b_first/b_last supply the spans.  d must be finite and >= 0. */
int tsk_search(tsk_db *db, const tsk_columns *queries, int64_t nb, const int64_t *b_lo,
               const int64_t *b_hi, const int64_t *b_first, const int64_t *b_last, double d,
               uint32_t flags, tsk_result **out);

/* [K1] pair_intervals(rows, cols, d): the rows×cols mesh, row-major hits. */
int tsk_pair_intervals(int device, const tsk_columns *rows, const tsk_columns *cols, double d,
                       tsk_result **out);

/* Result accessors.  per_batch (nb × 4 int64): first, last, overlaps, hits
 * (first = last = -1 for a batch with no candidates).  Column pointers stay
 * valid until tsk_result_free.  Missing columns come back NULL. */
int tsk_result_info(const tsk_result *r, int64_t *n_hits, int64_t *nb, double *device_ms);
/* Device time of the whole call and of the K1 launches (CUDA events), and
 * the number of kernels this library launched for the call. */
int tsk_result_timing(const tsk_result *r, double *device_ms, double *k1_ms, int64_t *launches);
int tsk_result_per_batch(const tsk_result *r, int64_t *per_batch);
/* (candidate, query) pairs K1's FP32 pre-filter evaluated in the call (its
 * work count for the kernel roofline; 0 where the FP64 kernel ran). */
int tsk_result_k1_evals(const tsk_result *r, int64_t *evals);
int tsk_result_columns(const tsk_result *r, const int64_t **query_traj, const int64_t **query_seg,
                       const int64_t **entry_traj, const int64_t **entry_seg,
                       const double **t_begin, const double **t_end, const int64_t **query_ord,
                       const int64_t **entry_ord);
void tsk_result_free(tsk_result *r);

/* Native batch planners over the host copy of the index (host code, no GPU).
 * Queries are given by their start-sorted ts/te; the index by its non-empty
 * bin arrays (tsk_index_copy).  Outputs hold up to nq batches: lo/hi query
 * ordinals, candidate span first/last (-1 when none) and the batch end time.
 *   tsk_plan_setsplit  mode 0: setsplit_fixed(num_batches)   (planner.py:293-309)
 *                      mode 1: setsplit_minmax(min, max)     (planner.py:312-358)
 *   tsk_plan_greedy    variant 0: greedy_min, 1: greedy_max  (planner.py:384-429) */
int tsk_plan_setsplit(int64_t nq, const double *ts, const double *te, int64_t n_ne,
                      const double *ne_start, const double *ne_end, const int64_t *ne_first,
                      const int64_t *ne_last, int mode, int64_t num_batches, int64_t min_size,
                      int64_t max_size, int64_t *nb_out, int64_t *b_lo, int64_t *b_hi,
                      int64_t *b_first, int64_t *b_last, double *b_end);
int tsk_plan_greedy(int64_t nq, const double *ts, const double *te, int64_t n_ne,
                    const double *ne_start, const double *ne_end, const int64_t *ne_first,
                    const int64_t *ne_last, int variant, int64_t bound, int64_t *nb_out,
                    int64_t *b_lo, int64_t *b_hi, int64_t *b_first, int64_t *b_last, double *b_end);

/* Work units of a plan (host code; the decomposition K1 runs, tsk_internal.cuh):
 * mode 0 none, 1 pairs, 4 quads, 8 octets (staircase groups), tqs the query
 * tile.  Writes 13 int64 per unit (b, b1, lo_q, s, js, jx[6], f, l) and
 * returns the unit count (-1 if it exceeds cap).  No reference counterpart:
 * a test hook for the partition property of the sharing layouts. */
int64_t tsk_plan_units(int64_t nb, const int64_t *lo, const int64_t *hi, const int64_t *first,
                       const int64_t *last, int mode, int64_t tqs, int64_t *out, int64_t cap);

/* Canonical order (core.py:290-294: query ids, entry ids, t_begin, t_end) of
 * n result rows, computed on `device`; outputs may alias nothing. */
int tsk_canonical_order(int device, int64_t n, const int64_t *qt, const int64_t *qs, const int64_t *et,
                        const int64_t *es, const double *tb, const double *te, int64_t *o_qt,
                        int64_t *o_qs, int64_t *o_et, int64_t *o_es, double *o_tb, double *o_te);

/* CSV I/O (host code).  Floats are written exactly as Python repr(float).
 *   tsk_save_store_csv     datagen.save   (datagen.py:273-285)
 *   tsk_write_results_csv  cli._write_results rows (cli.py:62-77)
 *   tsk_load_store_csv     datagen.load   (datagen.py:288-333): rows in file
 *                          order; *bad_line = offending line on TSK_EFORMAT
 *   tsk_format_double      repr(float) of one value (testing) */
typedef struct tsk_csv tsk_csv;
int tsk_format_double(double x, char *out, int cap);
int tsk_save_store_csv(const char *path, int64_t n, const int64_t *traj, const int64_t *seg,
                       const double *xs, const double *ys, const double *zs, const double *ts,
                       const double *xe, const double *ye, const double *ze, const double *te,
                       int nthreads);
int tsk_write_results_csv(const char *path, int64_t n, const int64_t *qt, const int64_t *qs,
                          const int64_t *et, const int64_t *es, const double *tb, const double *te,
                          int nthreads);
int tsk_load_store_csv(const char *path, int strict, tsk_csv **out, int64_t *n_out, int64_t *bad_line);
int tsk_csv_columns(const tsk_csv *c, int64_t *traj, int64_t *seg, double *xs, double *ys, double *zs,
                    double *ts, double *xe, double *ye, double *ze, double *te);
void tsk_csv_free(tsk_csv *c);

/* Page-locked host memory for query/result staging (cudaHostAlloc). */
void *tsk_pinned_alloc(int64_t bytes);
void tsk_pinned_free(void *p);

/* Measured FP64 pipe rate of `device` (DADD/DMUL per second, each counted
 * as one op; DFMA counted as one op too) — the roofline denominator of the
 * FP64-bound pair kernel. */
int tsk_probe_fp64(int device, double *dadd_per_s, double *dmul_per_s, double *dfma_per_s);
/* Measured FP32 FFMA rate of `device` (ops/s, an FFMA counted as one op) —
 * the issue roofline of K1's FP32 pre-filter. */
int tsk_probe_fp32(int device, double *ffma_per_s);
/* K1 development counters of `device` (up to 8: box-cull sub-tiles, box
 * tests, box survivors, sub-tiles with survivors, pre-filter flags,
 * separating-axis survivors, exact-path flushes, items); all zero unless
 * the library was built with -DTSK_K1_STATS.  reset != 0 zeroes them. */
int tsk_k1_stats(int device, unsigned long long *out, int n, int reset);

#ifdef __cplusplus
}
#endif
#endif /* TRAJSEEK_H */
