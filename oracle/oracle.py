"""CPU oracle for the distance-threshold search path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `trajseek` package's
hot path (arXiv 1405.7461, GPUTrajDistSearch, CPU emulation).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline arm may import it, and only as the checker or as the timed
CPU baseline.  The product package (``paper_1405_7461_b200``) never
imports anything from ``oracle/``.

Parity pin: every function here is checked against golden vectors that
were produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.

Arrays are plain dicts of numpy columns (``traj seg xs ys zs ts xe ye ze te``)
so that the oracle shares no types with the product package.

The arithmetic must be *operation-for-operation* identical to the
reference, because results are compared bit-for-bit:

* pair mesh        — /root/reference/pkg/src/trajseek/core.py:464-565
* scalar solver    — /root/reference/pkg/src/trajseek/core.py:309-438
* index build      — /root/reference/pkg/src/trajseek/index.py:85-146
* candidate range  — /root/reference/pkg/src/trajseek/index.py:149-173
* planners         — /root/reference/pkg/src/trajseek/planner.py:202-429
* engine           — /root/reference/pkg/src/trajseek/engine.py:78-204
* brute force      — /root/reference/pkg/src/trajseek/oracle.py:23-41
"""

from __future__ import annotations

import heapq
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

COLS = ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")
FLOAT_COLS = COLS[2:]

# engine.py:29 — pairs per candidate chunk
CHUNK_PAIRS = 1 << 20
# oracle.py:20 — queries per brute-force slab
SLAB = 64


# ── store helpers (core.py:121-243) ────────────────────────────────────────


def make_store(traj, seg, xs, ys, zs, ts, xe, ye, ze, te, presorted=False):
    """Columns → dict, stably sorted by start time (core.py:162-166)."""
    s = {"traj": np.asarray(traj, np.int64), "seg": np.asarray(seg, np.int64)}
    for k, v in zip(FLOAT_COLS, (xs, ys, zs, ts, xe, ye, ze, te)):
        s[k] = np.asarray(v, np.float64)
    n = s["traj"].shape[0]
    if not presorted and n and (np.diff(s["ts"]) < 0).any():
        perm = np.argsort(s["ts"], kind="stable")
        s = {k: v[perm] for k, v in s.items()}
    return s


def store_len(s) -> int:
    return int(s["traj"].shape[0])


def sub(s, lo, hi):
    """Inclusive ordinal slice (core.py:227-237)."""
    return {k: v[lo : hi + 1] for k, v in s.items()}


# ── pair mesh (core.py:464-565) ────────────────────────────────────────────


def _clip_at(s, idx, t):
    """Positions of segments ``idx`` at times ``t`` (core.py:503-521)."""
    t0 = s["ts"][idx]
    t1 = s["te"][idx]
    ext = t1 - t0
    frac = (t - t0) / np.where(ext == 0.0, 1.0, ext)
    verbatim_start = (ext == 0.0) | (t == t0)
    at_end = t == t1
    out = []
    for a, b in (("xs", "xe"), ("ys", "ye"), ("zs", "ze")):
        p0 = s[a][idx]
        p1 = s[b][idx]
        lerp = p0 + frac * (p1 - p0)
        out.append(np.where(verbatim_start, p0, np.where(at_end, p1, lerp)))
    return out


def pair_mesh(rows, cols, d):
    """All (row, col) pairs → (row_idx, col_idx, t_begin, t_end, tmiss, smiss).

    Hits are emitted row-major.  Restates core.py:464-565 exactly.
    """
    if d < 0 or not math.isfinite(d):
        raise ValueError(f"threshold d={d!r} must be finite and non-negative")
    nr, nc = store_len(rows), store_len(cols)
    ei = np.empty(0, np.int64)
    ef = np.empty(0, np.float64)
    if nr == 0 or nc == 0:
        return ei, ei, ef, ef, 0, 0
    t_a = np.maximum(rows["ts"][:, None], cols["ts"][None, :])
    t_b = np.minimum(rows["te"][:, None], cols["te"][None, :])
    ov = t_a <= t_b
    n_ov = int(np.count_nonzero(ov))
    tmiss = nr * nc - n_ov
    if n_ov == 0:
        return ei, ei, ef, ef, tmiss, 0
    ri, ci = np.nonzero(ov)
    t_a = t_a[ri, ci]
    t_b = t_b[ri, ci]
    span = t_b - t_a

    ra = _clip_at(rows, ri, t_a)
    rb = _clip_at(rows, ri, t_b)
    ca = _clip_at(cols, ci, t_a)
    cb = _clip_at(cols, ci, t_b)

    u = [ra[k] - ca[k] for k in range(3)]
    cc = u[0] * u[0] + u[1] * u[1] + u[2] * u[2]
    d2 = d * d
    w = [(rb[k] - ra[k]) - (cb[k] - ca[k]) for k in range(3)]
    aa = w[0] * w[0] + w[1] * w[1] + w[2] * w[2]
    bb = 2.0 * (u[0] * w[0] + u[1] * w[1] + u[2] * w[2])

    flat = aa == 0.0
    disc = bb * bb - 4.0 * aa * (cc - d2)
    real = disc >= 0.0
    root = np.sqrt(np.where(real, disc, 0.0))
    qq = np.where(bb >= 0.0, -0.5 * (bb + root), -0.5 * (bb - root))
    r1 = qq / np.where(flat, 1.0, aa)
    r2 = np.where(qq == 0.0, r1, (cc - d2) / np.where(qq == 0.0, 1.0, qq))
    lo = np.where(flat, 0.0, np.minimum(r1, r2))
    hi = np.where(flat, 1.0, np.maximum(r1, r2))
    hit = np.where(flat, cc <= d2, real & (lo <= 1.0) & (hi >= 0.0))
    t_begin = np.where(lo <= 0.0, t_a, t_a + lo * span)
    t_end = np.where(hi >= 1.0, t_b, t_a + hi * span)

    keep = np.nonzero(hit)[0]
    return ri[keep], ci[keep], t_begin[keep], t_end[keep], tmiss, n_ov - keep.shape[0]


# ── scalar solver (core.py:309-438), pure Python floats ────────────────────


def pair_scalar(a, b, d):
    """One pair, each a tuple (xs, ys, zs, ts, xe, ye, ze, te).

    Returns (begin, end) or None.  Restates temporal_intersection followed
    by threshold_interval (core.py:334-438).
    """
    ta = max(a[3], b[3])
    tb = min(a[7], b[7])
    if ta > tb:
        return None

    def at(s, t):
        t0, t1 = s[3], s[7]
        if t1 == t0 or t == t0:
            return (s[0], s[1], s[2])
        if t == t1:
            return (s[4], s[5], s[6])
        f = (t - t0) / (t1 - t0)
        return (s[0] + f * (s[4] - s[0]), s[1] + f * (s[5] - s[1]), s[2] + f * (s[6] - s[2]))

    def clip(s):
        if s[3] == ta and s[7] == tb:
            return s
        p, q = at(s, ta), at(s, tb)
        return (p[0], p[1], p[2], ta, q[0], q[1], q[2], tb)

    a, b = clip(a), clip(b)
    span = tb - ta
    d2 = d * d
    ux, uy, uz = a[0] - b[0], a[1] - b[1], a[2] - b[2]
    cc = ux * ux + uy * uy + uz * uz
    if span == 0.0:
        return (ta, tb) if cc <= d2 else None
    wx = (a[4] - a[0]) - (b[4] - b[0])
    wy = (a[5] - a[1]) - (b[5] - b[1])
    wz = (a[6] - a[2]) - (b[6] - b[2])
    aa = wx * wx + wy * wy + wz * wz
    bb = 2.0 * (ux * wx + uy * wy + uz * wz)
    if aa == 0.0:
        return (ta, tb) if cc <= d2 else None
    disc = bb * bb - 4.0 * aa * (cc - d2)
    if disc < 0.0:
        return None
    sd = math.sqrt(disc)
    qq = -0.5 * (bb + sd) if bb >= 0.0 else -0.5 * (bb - sd)
    r1 = qq / aa
    r2 = (cc - d2) / qq if qq != 0.0 else r1
    lo, hi = min(r1, r2), max(r1, r2)
    if lo > 1.0 or hi < 0.0:
        return None
    return (ta if lo <= 0.0 else ta + lo * span, tb if hi >= 1.0 else ta + hi * span)


# ── temporal index (index.py:85-188) ───────────────────────────────────────


def index_build(store, m, rule="member_extents"):
    """→ dict(m, width, t0, t_max, nonempty, ne_start, ne_end, ne_first, ne_last).

    ``nonempty`` is the boolean per-bin occupancy (index.py:116-119).
    """
    if m < 1:
        raise ValueError("m must be >= 1")
    ts, te = store["ts"], store["te"]
    n = ts.shape[0]
    if n == 0:
        raise ValueError("empty store")
    t0 = float(ts[0])
    t_max = float(te.max())
    width = (t_max - t0) / m
    if width > 0.0:
        bins = np.minimum((ts - t0) // width, m - 1).astype(np.int64)
    else:
        bins = np.zeros(n, np.int64)
    js = np.arange(m)
    first = np.searchsorted(bins, js, side="left")
    last = np.searchsorted(bins, js, side="right") - 1
    occupied = last >= first
    ne = np.nonzero(occupied)[0]
    ne_first = first[ne].astype(np.int64)
    ne_last = last[ne].astype(np.int64)
    if rule == "member_extents":
        ne_start = ts[ne_first].astype(np.float64)
    elif rule == "grid_start":
        ne_start = t0 + ne * width
    else:
        raise ValueError(rule)
    ne_end = np.maximum.reduceat(te, ne_first) if ne.shape[0] else np.empty(0)
    return dict(m=m, width=float(width), t0=t0, t_max=t_max, nonempty=occupied,
                ne_start=ne_start, ne_end=np.asarray(ne_end, np.float64),
                ne_first=ne_first, ne_last=ne_last)


def cand_range(ix, begin, end):
    """Contiguous candidate span for [begin, end] or None (index.py:149-173)."""
    starts = ix["ne_start"]
    if starts.shape[0] == 0:
        return None
    hi = int(np.searchsorted(starts, end, side="right"))
    if hi == 0:
        return None
    reach = ix["ne_end"][:hi] >= begin
    if not reach.any():
        return None
    k_lo = int(np.argmax(reach))
    k_hi = hi - 1 - int(np.argmax(reach[::-1]))
    return int(ix["ne_first"][k_lo]), int(ix["ne_last"][k_hi])


# ── planners (planner.py:202-429) ──────────────────────────────────────────
# A plan is a list of (lo, hi, begin, end, first, last) tuples.


def plan_periodic(q, s, ix=None):
    n = store_len(q)
    starts = np.arange(0, n, s)
    ends = np.maximum.reduceat(q["te"], starts)
    out = []
    for k, lo in enumerate(starts):
        lo = int(lo)
        hi = min(lo + s, n) - 1
        b, e = float(q["ts"][lo]), float(ends[k])
        fl = cand_range(ix, b, e) if ix is not None else None
        out.append((lo, hi, b, e, None if fl is None else fl[0], None if fl is None else fl[1]))
    return out


class _Run:
    """Mutable batch in a doubly linked list (planner.py:93-125)."""

    def __init__(self, lo, hi, b, e, fl, ints):
        self.lo, self.hi, self.b, self.e = lo, hi, b, e
        self.fl = fl
        self.ints = ints
        self.left = self.right = None
        self.gen = 0
        self.gone = False

    def n(self):
        return self.hi - self.lo + 1


def _lookup(ix, b, e, size):
    fl = cand_range(ix, b, e)
    return (fl, 0) if fl is None else (fl, size * (fl[1] - fl[0] + 1))


def _join_cost(ix, a, b):
    fl, ints = _lookup(ix, a.b, max(a.e, b.e), a.n() + b.n())
    return ints, fl


def _join(a, b, fl, ints):
    a.hi = b.hi
    a.e = max(a.e, b.e)
    a.fl = fl
    a.ints = ints
    a.right = b.right
    if b.right is not None:
        b.right.left = a
    b.gone = True
    a.gen += 1
    return a


def _singletons(q, ix):
    runs = []
    for i in range(store_len(q)):
        b, e = float(q["ts"][i]), float(q["te"][i])
        fl, ints = _lookup(ix, b, e, 1)
        r = _Run(i, i, b, e, fl, ints)
        if runs:
            r.left = runs[-1]
            runs[-1].right = r
        runs.append(r)
    return runs


def _head(runs):
    r = next(x for x in runs if not x.gone)
    while r.left is not None:
        r = r.left
    return r


def _export(runs):
    out = []
    r = _head(runs)
    while r is not None:
        fl = r.fl
        out.append((r.lo, r.hi, r.b, r.e, None if fl is None else fl[0], None if fl is None else fl[1]))
        r = r.right
    return out


def _merge_cheapest(runs, ix, stop, cap):
    """Heap-driven cheapest adjacent merge, ties to the earliest pair
    (planner.py:232-264)."""
    heap = []
    tick = 0

    def push(a, b):
        nonlocal tick
        if cap is not None and a.n() + b.n() > cap:
            return
        ints, fl = _join_cost(ix, a, b)
        heapq.heappush(heap, (ints - (a.ints + b.ints), a.lo, tick, a, b, a.gen, b.gen, ints, fl))
        tick += 1

    for a in runs:
        if a.right is not None:
            push(a, a.right)
    live = len(runs)
    while heap and (stop is None or live > stop):
        _, _, _, a, b, ga, gb, ints, fl = heapq.heappop(heap)
        if a.gone or b.gone or a.gen != ga or b.gen != gb or a.right is not b:
            continue
        a = _join(a, b, fl, ints)
        live -= 1
        if a.left is not None:
            push(a.left, a)
        if a.right is not None:
            push(a, a.right)


def plan_setsplit_fixed(q, ix, k):
    runs = _singletons(q, ix)
    _merge_cheapest(runs, ix, k, None)
    return _export(runs)


def plan_setsplit_minmax(q, ix, lo_size, hi_size):
    runs = _singletons(q, ix)
    _merge_cheapest(runs, ix, None, hi_size)
    r = _head(runs)
    while r is not None:
        if r.n() >= lo_size:
            r = r.right
            continue
        left, right = r.left, r.right
        if left is None and right is None:
            break
        lc = _join_cost(ix, left, r) if left is not None else None
        rc = _join_cost(ix, r, right) if right is not None else None
        li = lc[0] if lc is not None else math.inf
        ri = rc[0] if rc is not None else math.inf
        if li < ri:
            r = _join(left, r, lc[1], lc[0])
        else:
            r = _join(r, right, rc[1], rc[0])
    return _export(runs)


def plan_setsplit_max(q, ix, hi_size):
    return plan_setsplit_minmax(q, ix, 1, hi_size)


def _free_merges(runs, ix):
    r = runs[0]
    while r is not None and r.right is not None:
        nxt = r.right
        ints, fl = _join_cost(ix, r, nxt)
        if ints == r.ints + nxt.ints:
            _join(r, nxt, fl, ints)
        else:
            r = r.right


def plan_greedy(q, ix, bound, variant):
    runs = _singletons(q, ix)
    _free_merges(runs, ix)
    r = _head(runs)
    while r is not None and r.right is not None:
        grow = r.n() < bound if variant == "min" else r.n() <= bound
        if grow:
            ints, fl = _join_cost(ix, r, r.right)
            _join(r, r.right, fl, ints)
        else:
            r = r.right
    return _export(runs)


# ── engine (engine.py:78-204) and brute force (oracle.py:23-41) ────────────


def _chunks(first, last, size):
    per = max(1, CHUNK_PAIRS // max(1, size))
    return [(lo, min(lo + per - 1, last)) for lo in range(first, last + 1, per)]


def run_batch(store, batch, first, last, d, workers=1):
    """One batch → (rows dict of hit columns, tmiss, smiss).

    Hit columns: q_ord (index within ``batch``), e_ord, t_begin, t_end, in
    the reference's candidate-major chunk order (engine.py:97-148).
    """
    chunks = _chunks(first, last, store_len(batch))

    def work(c):
        return pair_mesh(sub(store, c[0], c[1]), batch, d)

    if workers <= 1 or len(chunks) <= 1:
        parts = [work(c) for c in chunks]
    else:
        with ThreadPoolExecutor(max_workers=min(workers, len(chunks))) as ex:
            parts = list(ex.map(work, chunks))
    qo, eo, tb, te = [], [], [], []
    tm = sm = 0
    for (lo, _), (ri, ci, b, e, t, s) in zip(chunks, parts):
        qo.append(ci)
        eo.append(ri + lo)
        tb.append(b)
        te.append(e)
        tm += t
        sm += s
    return (np.concatenate(qo), np.concatenate(eo), np.concatenate(tb), np.concatenate(te)), tm, sm


def search(store, ix, q, plan, d, workers=None, batch_ids=None):
    """Whole-plan search → (result dict, stats dict) in reference order.

    ``batch_ids`` optionally restricts execution to a subset of batches
    (the sampled CPU baseline); their relative order is kept.
    """
    if workers is None:
        workers = max(1, os.cpu_count() or 1)
    sel = range(len(plan)) if batch_ids is None else batch_ids
    cols = {k: [] for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")}
    st = dict(interactions=0, temporal_misses=0, spatial_misses=0, hits=0, per_batch=[])
    for k in sel:
        lo, hi, *_ = plan[k]
        bq = sub(q, lo, hi)
        b = float(q["ts"][lo])
        e = float(q["te"][lo : hi + 1].max())
        fl = cand_range(ix, b, e)
        if fl is None:
            st["per_batch"].append((k, hi - lo + 1, 0, 0, 0))
            continue
        (qo, eo, tbg, ten), tm, sm = run_batch(store, bq, fl[0], fl[1], d, workers)
        cols["query_traj"].append(bq["traj"][qo])
        cols["query_seg"].append(bq["seg"][qo])
        cols["entry_traj"].append(store["traj"][eo])
        cols["entry_seg"].append(store["seg"][eo])
        cols["t_begin"].append(tbg)
        cols["t_end"].append(ten)
        ints = (fl[1] - fl[0] + 1) * (hi - lo + 1)
        st["interactions"] += ints
        st["temporal_misses"] += tm
        st["spatial_misses"] += sm
        st["hits"] += qo.shape[0]
        st["per_batch"].append((k, hi - lo + 1, fl[1] - fl[0] + 1, ints, int(qo.shape[0])))
    out = {}
    for k, v in cols.items():
        dt = np.float64 if k.startswith("t_") else np.int64
        out[k] = np.concatenate(v) if v else np.empty(0, dt)
    return out, st


def brute_force(store, q, d):
    """Every query against every entry, query-major (oracle.py:23-41)."""
    cols = {k: [] for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")}
    n = store_len(q)
    for lo in range(0, n, SLAB):
        hi = min(lo + SLAB, n) - 1
        bq = sub(q, lo, hi)
        ri, ci, b, e, _, _ = pair_mesh(bq, store, d)
        cols["query_traj"].append(bq["traj"][ri])
        cols["query_seg"].append(bq["seg"][ri])
        cols["entry_traj"].append(store["traj"][ci])
        cols["entry_seg"].append(store["seg"][ci])
        cols["t_begin"].append(b)
        cols["t_end"].append(e)
    out = {}
    for k, v in cols.items():
        dt = np.float64 if k.startswith("t_") else np.int64
        out[k] = np.concatenate(v) if v else np.empty(0, dt)
    return out


def canonical_keys(res):
    """(n, 6) canonically ordered key array (core.py:290-303)."""
    order = np.lexsort((res["t_end"], res["t_begin"], res["entry_seg"],
                        res["entry_traj"], res["query_seg"], res["query_traj"]))
    return np.column_stack([
        res["query_traj"][order].astype(np.float64), res["query_seg"][order].astype(np.float64),
        res["entry_traj"][order].astype(np.float64), res["entry_seg"][order].astype(np.float64),
        res["t_begin"][order], res["t_end"][order],
    ])
