// planner.cu — native batch planners (host code).
//
// SetSplit (heap-incremental cheapest adjacent merge, planner.py:232-365)
// and GreedySetSplit (free-merge pass + forward size pass, planner.py:371-429)
// over the host copy of the temporal index.  Same semantics as the
// reference, including the heap order (delta, left lo, push sequence) that
// reproduces the earliest-strict-minimum rescan, the floor pass (a missing
// neighbour costs infinity, ties go right) and the greedy bounds.  The
// candidate-range lookup is index.py:149-173.
#include <cstdint>
#include <limits>
#include <queue>
#include <string>
#include <vector>

#include "tsk_internal.cuh"

namespace {

struct IndexView {
    int64_t n_ne;
    const double *start, *end;
    const int64_t *first, *last;
    std::vector<double> endmax;  // running max of end (non-decreasing)

    IndexView(int64_t n, const double *s, const double *e, const int64_t *f, const int64_t *l)
        : n_ne(n), start(s), end(e), first(f), last(l), endmax((size_t)(n > 0 ? n : 0)) {
        double m = -std::numeric_limits<double>::infinity();
        for (int64_t k = 0; k < n; ++k) {
            m = e[k] > m ? e[k] : m;
            endmax[(size_t)k] = m;
        }
    }

    // candidate_range: false when no bin qualifies
    bool range(double b, double e, int64_t &f, int64_t &l) const {
        if (n_ne == 0) return false;
        int64_t lo = 0, hi = n_ne;  // upper_bound(start, e)
        while (lo < hi) {
            int64_t m = (lo + hi) >> 1;
            if (start[m] <= e) lo = m + 1;
            else hi = m;
        }
        const int64_t h = lo;
        if (h == 0) return false;
        int64_t a = 0, z = h;  // lower_bound(endmax[:h], b)
        while (a < z) {
            int64_t m = (a + z) >> 1;
            if (endmax[(size_t)m] >= b) z = m;
            else a = m + 1;
        }
        if (a >= h) return false;
        int64_t k = h - 1;
        while (end[k] < b) --k;
        f = first[a];
        l = last[k];
        return true;
    }
};

struct Runs {
    const IndexView &ix;
    std::vector<int64_t> lo, hi, first, last, ints, prev, next, version;
    std::vector<double> begin, end;
    std::vector<char> dead;

    Runs(const IndexView &index, int64_t n, const double *ts, const double *te) : ix(index) {
        lo.resize(n); hi.resize(n); first.resize(n); last.resize(n); ints.resize(n);
        prev.resize(n); next.resize(n); version.assign(n, 0); dead.assign(n, 0);
        begin.assign(ts, ts + n);
        end.assign(te, te + n);
        for (int64_t i = 0; i < n; ++i) {
            lo[i] = hi[i] = i;
            prev[i] = i - 1;
            next[i] = i + 1 < n ? i + 1 : -1;
            int64_t f, l;
            if (ix.range(ts[i], te[i], f, l)) {
                first[i] = f; last[i] = l; ints[i] = l - f + 1;
            } else {
                first[i] = last[i] = -1; ints[i] = 0;
            }
        }
    }

    int64_t size(int64_t i) const { return hi[i] - lo[i] + 1; }

    // (interactions, first, last) of a and b as one batch
    void merged(int64_t a, int64_t b, int64_t &mi, int64_t &mf, int64_t &ml) const {
        const int64_t s = size(a) + size(b);
        const double e = end[a] > end[b] ? end[a] : end[b];
        if (ix.range(begin[a], e, mf, ml)) mi = s * (ml - mf + 1);
        else { mi = 0; mf = ml = -1; }
    }

    int64_t merge(int64_t a, int64_t b, int64_t mi, int64_t mf, int64_t ml) {
        hi[a] = hi[b];
        end[a] = end[a] > end[b] ? end[a] : end[b];
        first[a] = mf; last[a] = ml; ints[a] = mi;
        const int64_t nb = next[b];
        next[a] = nb;
        if (nb >= 0) prev[nb] = a;
        dead[b] = 1;
        ++version[a];
        return a;
    }

    int64_t head() const {
        int64_t i = 0;
        while (dead[i]) ++i;
        while (prev[i] >= 0) i = prev[i];
        return i;
    }
};

struct Entry {
    int64_t delta, lo, seq, a, b, va, vb, ints, first, last;
    bool operator>(const Entry &o) const {
        if (delta != o.delta) return delta > o.delta;
        if (lo != o.lo) return lo > o.lo;
        return seq > o.seq;
    }
};

void cheapest_merges(Runs &R, int64_t stop_count /* -1: none */, int64_t max_size /* -1: none */) {
    std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
    int64_t seq = 0;
    auto push = [&](int64_t a, int64_t b) {
        if (max_size >= 0 && R.size(a) + R.size(b) > max_size) return;
        Entry e;
        R.merged(a, b, e.ints, e.first, e.last);
        e.delta = e.ints - (R.ints[a] + R.ints[b]);
        e.lo = R.lo[a];
        e.seq = seq++;
        e.a = a; e.b = b; e.va = R.version[a]; e.vb = R.version[b];
        heap.push(e);
    };
    const int64_t n = (int64_t)R.lo.size();
    for (int64_t a = 0; a < n; ++a)
        if (R.next[a] >= 0) push(a, R.next[a]);
    int64_t live = n;
    while (!heap.empty() && (stop_count < 0 || live > stop_count)) {
        Entry e = heap.top();
        heap.pop();
        if (R.dead[e.a] || R.dead[e.b] || R.version[e.a] != e.va || R.version[e.b] != e.vb ||
            R.next[e.a] != e.b)
            continue;
        const int64_t a = R.merge(e.a, e.b, e.ints, e.first, e.last);
        --live;
        if (R.prev[a] >= 0) push(R.prev[a], a);
        if (R.next[a] >= 0) push(a, R.next[a]);
    }
}

int64_t emit(const Runs &R, int64_t *b_lo, int64_t *b_hi, int64_t *b_first, int64_t *b_last,
             double *b_end) {
    int64_t k = 0;
    for (int64_t i = R.head(); i >= 0; i = R.next[i], ++k) {
        b_lo[k] = R.lo[i];
        b_hi[k] = R.hi[i];
        b_first[k] = R.first[i];
        b_last[k] = R.last[i];
        b_end[k] = R.end[i];
    }
    return k;
}

}  // namespace

using namespace tsk;

// mode 0: setsplit_fixed(num_batches); mode 1: setsplit_minmax(min_size, max_size)
extern "C" int tsk_plan_setsplit(int64_t nq, const double *ts, const double *te, int64_t n_ne,
                                 const double *ne_start, const double *ne_end,
                                 const int64_t *ne_first, const int64_t *ne_last, int mode,
                                 int64_t num_batches, int64_t min_size, int64_t max_size,
                                 int64_t *nb_out, int64_t *b_lo, int64_t *b_hi, int64_t *b_first,
                                 int64_t *b_last, double *b_end) {
    try {
        TSK_REQUIRE(nq > 0, "query set is empty");
        TSK_REQUIRE(ts && te && nb_out && b_lo && b_hi && b_first && b_last && b_end, "null argument");
        IndexView ix(n_ne, ne_start, ne_end, ne_first, ne_last);
        Runs R(ix, nq, ts, te);
        if (mode == 0) {
            TSK_REQUIRE(num_batches >= 1, "num_batches must be >= 1");
            cheapest_merges(R, num_batches, -1);
        } else {
            TSK_REQUIRE(min_size >= 1, "min_size must be >= 1");
            TSK_REQUIRE(max_size >= min_size, "max_size must be >= min_size");
            cheapest_merges(R, -1, max_size);
            // floor pass (planner.py:336-357)
            const double inf = std::numeric_limits<double>::infinity();
            int64_t i = R.head();
            while (i >= 0) {
                if (R.size(i) >= min_size) {
                    i = R.next[i];
                    continue;
                }
                const int64_t left = R.prev[i], right = R.next[i];
                if (left < 0 && right < 0) break;
                int64_t li = 0, lf = -1, ll = -1, ri = 0, rf = -1, rl = -1;
                double lc = inf, rc = inf;
                if (left >= 0) {
                    R.merged(left, i, li, lf, ll);
                    lc = (double)li;
                }
                if (right >= 0) {
                    R.merged(i, right, ri, rf, rl);
                    rc = (double)ri;
                }
                if (lc < rc) i = R.merge(left, i, li, lf, ll);
                else i = R.merge(i, right, ri, rf, rl);
            }
        }
        *nb_out = emit(R, b_lo, b_hi, b_first, b_last, b_end);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    } catch (const std::bad_alloc &) {
        return fail(TSK_ENOMEM, "out of host memory in planner");
    }
}

// variant 0: greedy_min(bound); variant 1: greedy_max(bound)
extern "C" int tsk_plan_greedy(int64_t nq, const double *ts, const double *te, int64_t n_ne,
                               const double *ne_start, const double *ne_end,
                               const int64_t *ne_first, const int64_t *ne_last, int variant,
                               int64_t bound, int64_t *nb_out, int64_t *b_lo, int64_t *b_hi,
                               int64_t *b_first, int64_t *b_last, double *b_end) {
    try {
        TSK_REQUIRE(nq > 0, "query set is empty");
        TSK_REQUIRE(bound >= 1, "bound must be >= 1");
        TSK_REQUIRE(ts && te && nb_out && b_lo && b_hi && b_first && b_last && b_end, "null argument");
        IndexView ix(n_ne, ne_start, ne_end, ne_first, ne_last);
        Runs R(ix, nq, ts, te);
        // free-merge pass (planner.py:371-381)
        int64_t i = 0;
        while (i >= 0 && R.next[i] >= 0) {
            const int64_t j = R.next[i];
            int64_t mi, mf, ml;
            R.merged(i, j, mi, mf, ml);
            if (mi == R.ints[i] + R.ints[j]) R.merge(i, j, mi, mf, ml);
            else i = j;
        }
        // size pass (planner.py:384-429)
        i = R.head();
        while (i >= 0 && R.next[i] >= 0) {
            const bool grow = variant == 0 ? R.size(i) < bound : R.size(i) <= bound;
            if (grow) {
                const int64_t j = R.next[i];
                int64_t mi, mf, ml;
                R.merged(i, j, mi, mf, ml);
                R.merge(i, j, mi, mf, ml);
            } else {
                i = R.next[i];
            }
        }
        *nb_out = emit(R, b_lo, b_hi, b_first, b_last, b_end);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    } catch (const std::bad_alloc &) {
        return fail(TSK_ENOMEM, "out of host memory in planner");
    }
}
