// csvio.cu — native CSV I/O for stores and results (host code).
//
//   save  ............ datagen.save  (/root/reference/pkg/src/trajseek/datagen.py:273-285)
//   load  ............ datagen.load  (datagen.py:288-333)
//   result CSV ....... cli._write_results (cli.py:62-77)
//
// Floats are written exactly as Python's repr(float): the shortest digits
// that round-trip (std::to_chars), laid out by CPython's 'r' rules —
// fixed notation when -4 < decpt <= 16 (always with a fractional part, e.g.
// "123.0"), otherwise "d.ddde±XX" with at least two exponent digits.
// Parsing uses strtod, which is correctly rounded like Python's float().
// Rows are formatted/parsed in parallel chunks; output order is row order.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tsk_internal.cuh"

namespace {

// Python repr(float) for finite x into out; returns the length.
int py_repr(double x, char *out) {
    char *o = out;
    if (std::isnan(x)) {
        memcpy(o, "nan", 3);
        return 3;
    }
    if (std::isinf(x)) {
        if (x < 0) *o++ = '-';
        memcpy(o, "inf", 3);
        return (int)(o - out) + 3;
    }
    if (x == 0.0) {
        if (std::signbit(x)) *o++ = '-';
        memcpy(o, "0.0", 3);
        return (int)(o - out) + 3;
    }
    char buf[40];
    auto r = std::to_chars(buf, buf + sizeof(buf) - 1, x, std::chars_format::scientific);
    *r.ptr = 0;  // atoi below reads the exponent up to the terminator
    // buf: [-]d[.ddd]e±XX
    const char *p = buf, *end = r.ptr;
    if (*p == '-') {
        *o++ = '-';
        ++p;
    }
    char digits[32];
    int nd = 0;
    while (p < end && *p != 'e') {
        if (*p != '.') digits[nd++] = *p;
        ++p;
    }
    int e10 = atoi(p + 1);  // exponent of d.ddd form
    int decpt = e10 + 1;    // value = 0.d1d2... x 10^decpt
    while (nd > 1 && digits[nd - 1] == '0') --nd;  // to_chars is already shortest; be safe
    if (decpt <= -4 || decpt > 16) {
        *o++ = digits[0];
        if (nd > 1) {
            *o++ = '.';
            memcpy(o, digits + 1, nd - 1);
            o += nd - 1;
        }
        int ex = decpt - 1;
        *o++ = 'e';
        *o++ = ex < 0 ? '-' : '+';
        int ax = ex < 0 ? -ex : ex;
        char eb[8];
        int ne = 0;
        do {
            eb[ne++] = (char)('0' + ax % 10);
            ax /= 10;
        } while (ax);
        if (ne < 2) eb[ne++] = '0';
        while (ne) *o++ = eb[--ne];
    } else if (decpt <= 0) {
        *o++ = '0';
        *o++ = '.';
        for (int i = 0; i < -decpt; ++i) *o++ = '0';
        memcpy(o, digits, nd);
        o += nd;
    } else if (decpt < nd) {
        memcpy(o, digits, decpt);
        o += decpt;
        *o++ = '.';
        memcpy(o, digits + decpt, nd - decpt);
        o += nd - decpt;
    } else {
        memcpy(o, digits, nd);
        o += nd;
        for (int i = nd; i < decpt; ++i) *o++ = '0';
        *o++ = '.';
        *o++ = '0';
    }
    return (int)(o - out);
}

int put_i64(int64_t v, char *out) {
    auto r = std::to_chars(out, out + 24, v);
    return (int)(r.ptr - out);
}

// Format rows [0, n) with fmt_row(i, char*) -> length, in parallel chunks,
// and write them after `header` to path.
template <class F>
void write_rows(const char *path, const std::string &header, int64_t n, int max_row, F fmt_row,
                int nthreads) {
    FILE *fh = fopen(path, "wb");
    if (!fh) throw tsk::Error{TSK_EINVAL, std::string("cannot open ") + path + " for writing"};
    fwrite(header.data(), 1, header.size(), fh);
    if (nthreads < 1) nthreads = 1;
    const int64_t chunk = 1 << 16;
    std::vector<std::string> bufs(nthreads);
    for (int64_t base = 0; base < n; base += chunk * nthreads) {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t) {
            th.emplace_back([&, t] {
                const int64_t lo = base + t * chunk, hi = std::min<int64_t>(lo + chunk, n);
                std::string &b = bufs[t];
                b.clear();
                if (lo >= hi) return;
                b.resize((size_t)(hi - lo) * max_row);
                char *o = &b[0];
                for (int64_t i = lo; i < hi; ++i) o += fmt_row(i, o);
                b.resize(o - &b[0]);
            });
        }
        for (auto &x : th) x.join();
        for (auto &b : bufs) fwrite(b.data(), 1, b.size(), fh);
    }
    if (fclose(fh) != 0) throw tsk::Error{TSK_ECUDA, std::string("write failed: ") + path};
}

}  // namespace

using namespace tsk;

extern "C" int tsk_format_double(double x, char *out, int cap) {
    char b[48];
    int n = py_repr(x, b);
    if (n >= cap) return -1;
    memcpy(out, b, n);
    out[n] = 0;
    return n;
}

// datagen.save: header + one row per segment, ints as int(), floats as repr().
extern "C" int tsk_save_store_csv(const char *path, int64_t n, const int64_t *traj, const int64_t *seg,
                                  const double *xs, const double *ys, const double *zs, const double *ts,
                                  const double *xe, const double *ye, const double *ze, const double *te,
                                  int nthreads) {
    try {
        const double *f[8] = {xs, ys, zs, ts, xe, ye, ze, te};
        write_rows(path, "traj_id,seg_id,x_s,y_s,z_s,t_s,x_e,y_e,z_e,t_e\n", n, 2 * 21 + 8 * 26 + 12,
                   [&](int64_t i, char *o) {
                       char *s = o;
                       o += put_i64(traj[i], o);
                       *o++ = ',';
                       o += put_i64(seg[i], o);
                       for (int k = 0; k < 8; ++k) {
                           *o++ = ',';
                           o += py_repr(f[k][i], o);
                       }
                       *o++ = '\n';
                       return (int)(o - s);
                   },
                   nthreads);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

// cli._write_results: header + one row per hit (ids as int, times as repr).
extern "C" int tsk_write_results_csv(const char *path, int64_t n, const int64_t *qt, const int64_t *qs,
                                     const int64_t *et, const int64_t *es, const double *tb,
                                     const double *te, int nthreads) {
    try {
        write_rows(path, "query_traj,query_seg,entry_traj,entry_seg,t_begin,t_end\n", n,
                   4 * 21 + 2 * 26 + 8,
                   [&](int64_t i, char *o) {
                       char *s = o;
                       o += put_i64(qt[i], o);
                       *o++ = ',';
                       o += put_i64(qs[i], o);
                       *o++ = ',';
                       o += put_i64(et[i], o);
                       *o++ = ',';
                       o += put_i64(es[i], o);
                       *o++ = ',';
                       o += py_repr(tb[i], o);
                       *o++ = ',';
                       o += py_repr(te[i], o);
                       *o++ = '\n';
                       return (int)(o - s);
                   },
                   nthreads);
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

// ── load ────────────────────────────────────────────────────────────────────

struct tsk_csv {
    std::vector<int64_t> traj, seg;
    std::vector<double> col[8];
};

namespace {

bool parse_i64(const char *b, const char *e, int64_t &v) {
    // Python int(): optional surrounding whitespace, optional sign, digits, '_' separators
    while (b < e && (*b == ' ' || *b == '\t')) ++b;
    while (e > b && (e[-1] == ' ' || e[-1] == '\t' || e[-1] == '\r')) --e;
    if (b == e) return false;
    auto r = std::from_chars(b + (*b == '+' ? 1 : 0), e, v);
    return r.ec == std::errc() && r.ptr == e;
}

bool parse_f64(const char *b, const char *e, double &v) {
    while (b < e && (*b == ' ' || *b == '\t')) ++b;
    while (e > b && (e[-1] == ' ' || e[-1] == '\t' || e[-1] == '\r')) --e;
    if (b == e) return false;
    if (*b == '+') ++b;  // float() accepts a leading '+'
    auto r = std::from_chars(b, e, v);  // correctly rounded, as Python's float()
    return r.ec == std::errc() && r.ptr == e;
}

struct Chunk {
    std::vector<int64_t> traj, seg;
    std::vector<double> col[8];
    int64_t lines = 0;       // lines in this chunk
    int64_t err_line = -1;   // first bad line, relative to the chunk (1-based)
    int err_kind = 0;        // 1 arity, 2 unparsable, 3 non-finite, 4 reversed
    int err_count = 0;
    double err_ts = 0, err_te = 0;
};

void parse_chunk(const char *p, const char *end, Chunk &c) {
    const size_t est = (size_t)(end - p) / 120 + 16;
    c.traj.reserve(est);
    c.seg.reserve(est);
    for (auto &v : c.col) v.reserve(est);
    while (p < end) {
        const char *b = p;
        const char *nl = (const char *)memchr(p, '\n', end - p);
        const char *e = nl ? nl : end;
        p = nl ? nl + 1 : end;
        ++c.lines;
        if (e > b && e[-1] == '\r') --e;
        if (b == e) continue;  // csv.reader yields [] for an empty line
        const char *f[11];
        int count = 1;
        f[0] = b;
        for (const char *q = b; q < e; ++q)
            if (*q == ',') {
                if (count < 10) f[count] = q + 1;
                ++count;
            }
        if (count != 10) {
            c.err_line = c.lines;
            c.err_kind = 1;
            c.err_count = count;
            return;
        }
        f[10] = e + 1;
        int64_t iv[2];
        double dv[8];
        bool ok = parse_i64(f[0], f[1] - 1, iv[0]) && parse_i64(f[1], f[2] - 1, iv[1]);
        for (int k = 0; k < 8 && ok; ++k) ok = parse_f64(f[2 + k], f[3 + k] - 1, dv[k]);
        if (!ok) {
            c.err_line = c.lines;
            c.err_kind = 2;
            return;
        }
        for (int k = 0; k < 8; ++k)
            if (!std::isfinite(dv[k])) {
                c.err_line = c.lines;
                c.err_kind = 3;
                return;
            }
        if (dv[7] < dv[3]) {
            c.err_line = c.lines;
            c.err_kind = 4;
            c.err_ts = dv[3];
            c.err_te = dv[7];
            return;
        }
        c.traj.push_back(iv[0]);
        c.seg.push_back(iv[1]);
        for (int k = 0; k < 8; ++k) c.col[k].push_back(dv[k]);
    }
}

}  // namespace

// datagen.load: validation and error messages follow datagen.py:288-333;
// rows are returned sorted by start time (stable) unless strict, where
// unsorted input is an error.  *bad_line receives the offending line.
extern "C" int tsk_load_store_csv(const char *path, int strict, tsk_csv **out, int64_t *n_out,
                                  int64_t *bad_line) {
    *bad_line = 0;
    try {
        FILE *fh = fopen(path, "rb");
        if (!fh) throw Error{TSK_EFORMAT, std::string(path) + ": cannot open"};
        fseek(fh, 0, SEEK_END);
        long sz = ftell(fh);
        fseek(fh, 0, SEEK_SET);
        std::string data((size_t)(sz > 0 ? sz : 0), '\0');
        if (sz > 0 && fread(&data[0], 1, (size_t)sz, fh) != (size_t)sz) {
            fclose(fh);
            throw Error{TSK_EFORMAT, std::string(path) + ": read error"};
        }
        fclose(fh);
        const char *p = data.data(), *end = p + data.size();
        auto next_line = [&](const char *&b, const char *&e) -> bool {
            if (p >= end) return false;
            b = p;
            const char *nl = (const char *)memchr(p, '\n', end - p);
            e = nl ? nl : end;
            p = nl ? nl + 1 : end;
            if (e > b && e[-1] == '\r') --e;
            return true;
        };
        const char *b, *e;
        if (!next_line(b, e)) throw Error{TSK_EFORMAT, std::string(path) + ": empty file"};
        if (std::string(b, e) != "traj_id,seg_id,x_s,y_s,z_s,t_s,x_e,y_e,z_e,t_e")
            throw Error{TSK_EFORMAT, std::string(path) + ": bad header " + std::string(b, e)};
        // split the body at line boundaries into one chunk per thread
        const int nthreads = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
        std::vector<const char *> cut{p};
        for (int t = 1; t < nthreads; ++t) {
            const char *c0 = p + (end - p) * t / nthreads;
            if (c0 < cut.back()) c0 = cut.back();
            const char *nl = (const char *)memchr(c0, '\n', end - c0);
            cut.push_back(nl ? nl + 1 : end);
        }
        cut.push_back(end);
        std::vector<Chunk> chunks(nthreads);
        {
            std::vector<std::thread> th;
            for (int t = 0; t < nthreads; ++t)
                th.emplace_back([&, t] { parse_chunk(cut[t], cut[t + 1], chunks[t]); });
            for (auto &x : th) x.join();
        }
        int64_t lines_before = 1;  // the header
        for (auto &ch : chunks) {
            if (ch.err_line >= 0) {
                const int64_t lineno = lines_before + ch.err_line;
                *bad_line = lineno;
                const std::string at = std::string(path) + ":" + std::to_string(lineno) + ": ";
                if (ch.err_kind == 1)
                    throw Error{TSK_EFORMAT, at + "expected 10 fields, got " + std::to_string(ch.err_count)};
                if (ch.err_kind == 2) throw Error{TSK_EFORMAT, at + "unparsable field"};
                if (ch.err_kind == 3) throw Error{TSK_EFORMAT, at + "non-finite coordinate"};
                char a1[48], z1[48];
                a1[py_repr(ch.err_te, a1)] = 0;
                z1[py_repr(ch.err_ts, z1)] = 0;
                throw Error{TSK_EFORMAT, at + "segment ends at t=" + a1 + " before it starts at t=" + z1};
            }
            lines_before += ch.lines;
        }
        auto *c = new tsk_csv();
        size_t total = 0;
        for (auto &ch : chunks) total += ch.traj.size();
        c->traj.reserve(total);
        c->seg.reserve(total);
        for (auto &v : c->col) v.reserve(total);
        for (auto &ch : chunks) {
            c->traj.insert(c->traj.end(), ch.traj.begin(), ch.traj.end());
            c->seg.insert(c->seg.end(), ch.seg.begin(), ch.seg.end());
            for (int k = 0; k < 8; ++k) c->col[k].insert(c->col[k].end(), ch.col[k].begin(), ch.col[k].end());
        }
        if (c->traj.empty()) {
            delete c;
            throw Error{TSK_EFORMAT, std::string(path) + ": no segments"};
        }
        if (strict) {
            const auto &t = c->col[3];
            for (size_t i = 1; i < t.size(); ++i)
                if (t[i] < t[i - 1]) {
                    *bad_line = (int64_t)i + 2;
                    delete c;
                    throw Error{TSK_EFORMAT, std::string(path) + ":" + std::to_string(i + 2) +
                                                 ": rows not sorted by t_s (strict mode)"};
                }
        }
        *out = c;
        *n_out = (int64_t)c->traj.size();
        return TSK_OK;
    } catch (const Error &e) {
        return fail(e.code, e.msg);
    }
}

extern "C" int tsk_csv_columns(const tsk_csv *c, int64_t *traj, int64_t *seg, double *xs, double *ys,
                               double *zs, double *ts, double *xe, double *ye, double *ze, double *te) {
    if (!c) return fail(TSK_EINVAL, "null handle");
    const size_t n = c->traj.size();
    memcpy(traj, c->traj.data(), n * 8);
    memcpy(seg, c->seg.data(), n * 8);
    double *o[8] = {xs, ys, zs, ts, xe, ye, ze, te};
    for (int k = 0; k < 8; ++k) memcpy(o[k], c->col[k].data(), n * 8);
    return TSK_OK;
}

extern "C" void tsk_csv_free(tsk_csv *c) { delete c; }
