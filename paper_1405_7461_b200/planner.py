"""Query-batch planners (host side).

Same names, arguments, results and DomainError behaviour as
/root/reference/pkg/src/trajseek/planner.py:

* ``periodic`` (planner.py:202-226) — fixed size s, short remainder batch.
* ``setsplit_fixed`` / ``setsplit_minmax`` / ``setsplit_max``
  (planner.py:293-365) — cheapest adjacent merge first (ties → earliest
  pair), heap-incremental or, with ``literal=True``, full rescans.
* ``greedy_min`` / ``greedy_max`` (planner.py:371-429) — free-merge pass,
  then a forward size pass.

SetSplit and Greedy run natively by default (C++ in libtrajseek,
csrc/planner.cu, same heap order and tie-breaking); ``literal=True``
(SetSplit) and ``native=False`` (Greedy) select the Python implementations
below, kept as the differential check.  The batches are kept in flat arrays
linked by prev/next indices; merge costs come from the index's candidate
ranges (host lookups on the arrays the GPU index build copied back).  The
batch table a plan produces feeds the GPU search.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass

import numpy as np

from .core import DomainError, SegmentStore, TimeInterval
from .index import TemporalIndex, candidate_range, candidate_ranges


@dataclass(frozen=True)
class QueryBatch:
    """Contiguous query ordinals lo..hi with their cached candidate span."""

    lo: int
    hi: int
    extent: TimeInterval
    first: int | None
    last: int | None

    @property
    def size(self) -> int:
        return self.hi - self.lo + 1

    @property
    def candidates(self) -> int:
        return 0 if self.first is None else self.last - self.first + 1

    @property
    def interactions(self) -> int:
        return self.size * self.candidates


@dataclass(frozen=True)
class BatchPlan:
    """Ordered partition of a query set into batches (planner.py:66-90)."""

    queries: SegmentStore
    batches: tuple[QueryBatch, ...]

    def __post_init__(self) -> None:
        if not self.batches:
            raise DomainError("a plan needs at least one batch")
        n = len(self.queries)
        cursor = 0
        for b in self.batches:
            if b.lo != cursor or b.hi < b.lo:
                raise DomainError(f"batches do not partition 0..{n - 1} contiguously")
            cursor = b.hi + 1
        if cursor != n:
            raise DomainError(f"batches cover 0..{cursor - 1} but the query set has {n} segments")

    @property
    def total_interactions(self) -> int:
        return sum(b.interactions for b in self.batches)

    def sizes(self) -> list[int]:
        return [b.size for b in self.batches]

    def table(self) -> tuple[np.ndarray, np.ndarray]:
        """(lo, hi) int64 arrays — the batch table handed to the GPU (built
        once per plan: the plan and its batches are immutable; read-only)."""
        t = self.__dict__.get("_table")
        if t is None:
            lo = np.fromiter((b.lo for b in self.batches), np.int64, len(self.batches))
            hi = np.fromiter((b.hi for b in self.batches), np.int64, len(self.batches))
            lo.flags.writeable = False
            hi.flags.writeable = False
            t = (lo, hi)
            object.__setattr__(self, "_table", t)
        return t


def num_interactions(batch: QueryBatch, index: TemporalIndex) -> int:
    """Interactions of ``batch`` recomputed against ``index``."""
    span = candidate_range(index, batch.extent)
    return 0 if span is None else batch.size * (span[1] - span[0] + 1)


def _check_queries(queries: SegmentStore) -> None:
    if len(queries) == 0:
        raise DomainError("query set is empty")


# ── periodic ────────────────────────────────────────────────────────────────


def periodic(queries: SegmentStore, s: int, index: TemporalIndex | None = None) -> BatchPlan:
    """Batches of s consecutive queries; the last one keeps the remainder."""
    _check_queries(queries)
    if s < 1:
        raise DomainError(f"batch size s={s} must be >= 1")
    n = len(queries)
    starts = np.arange(0, n, s)
    ends = np.maximum.reduceat(queries.te, starts)
    begins = queries.ts[starts]
    if index is not None:
        first, last = candidate_ranges(index, begins, ends)
    batches = []
    for k, lo in enumerate(starts.tolist()):
        f = l = None
        if index is not None and first[k] >= 0:
            f, l = int(first[k]), int(last[k])
        batches.append(QueryBatch(lo, min(lo + s, n) - 1,
                                  TimeInterval(float(begins[k]), float(ends[k])), f, l))
    return BatchPlan(queries, tuple(batches))


# ── linked batches under construction ──────────────────────────────────────


class _Runs:
    """Batches as parallel lists linked by prev/next (−1 = none)."""

    def __init__(self, queries: SegmentStore, index: TemporalIndex):
        n = len(queries)
        self.index = index
        self.queries = queries
        self.lo = list(range(n))
        self.hi = list(range(n))
        self.begin = queries.ts.tolist()
        self.end = queries.te.tolist()
        f, l = candidate_ranges(index, queries.ts, queries.te)
        self.first = [None if v < 0 else v for v in f.tolist()]
        self.last = [None if v < 0 else v for v in l.tolist()]
        self.ints = [0 if a is None else b - a + 1 for a, b in zip(self.first, self.last)]
        self.prev = list(range(-1, n - 1))
        self.next = list(range(1, n)) + [-1]
        self.version = [0] * n
        self.dead = [False] * n

    def size(self, i: int) -> int:
        return self.hi[i] - self.lo[i] + 1

    def merged(self, a: int, b: int):
        """(interactions, first, last) if a and b were one batch."""
        size = self.size(a) + self.size(b)
        span = candidate_range(self.index, TimeInterval(self.begin[a], max(self.end[a], self.end[b])))
        if span is None:
            return 0, None, None
        return size * (span[1] - span[0] + 1), span[0], span[1]

    def merge(self, a: int, b: int, ints: int, first, last) -> int:
        """Fold b (a's successor) into a; returns a."""
        self.hi[a] = self.hi[b]
        self.end[a] = max(self.end[a], self.end[b])
        self.first[a], self.last[a], self.ints[a] = first, last, ints
        nb = self.next[b]
        self.next[a] = nb
        if nb >= 0:
            self.prev[nb] = a
        self.dead[b] = True
        self.version[a] += 1
        return a

    def head(self) -> int:
        i = next(k for k, d in enumerate(self.dead) if not d)
        while self.prev[i] >= 0:
            i = self.prev[i]
        return i

    def plan(self) -> BatchPlan:
        out = []
        i = self.head()
        while i >= 0:
            out.append(QueryBatch(self.lo[i], self.hi[i], TimeInterval(self.begin[i], self.end[i]),
                                  self.first[i], self.last[i]))
            i = self.next[i]
        return BatchPlan(self.queries, tuple(out))


def _cheapest_heap(R: _Runs, stop_count: int | None, max_size: int | None) -> None:
    """Minimum-cost adjacent merges via a lazily invalidated heap
    (planner.py:241-264); heap order (delta, left lo, push sequence)
    reproduces the earliest-strict-minimum rescan."""
    heap: list = []
    seq = 0

    def push(a: int, b: int) -> None:
        nonlocal seq
        if max_size is not None and R.size(a) + R.size(b) > max_size:
            return
        ints, f, l = R.merged(a, b)
        heapq.heappush(heap, (ints - (R.ints[a] + R.ints[b]), R.lo[a], seq, a, b,
                              R.version[a], R.version[b], ints, f, l))
        seq += 1

    for a in range(len(R.lo)):
        if R.next[a] >= 0:
            push(a, R.next[a])
    live = len(R.lo)
    while heap and (stop_count is None or live > stop_count):
        _, _, _, a, b, va, vb, ints, f, l = heapq.heappop(heap)
        if R.dead[a] or R.dead[b] or R.version[a] != va or R.version[b] != vb or R.next[a] != b:
            continue
        a = R.merge(a, b, ints, f, l)
        live -= 1
        if R.prev[a] >= 0:
            push(R.prev[a], a)
        if R.next[a] >= 0:
            push(a, R.next[a])


def _cheapest_rescan(R: _Runs, stop_count: int | None, max_size: int | None) -> None:
    """Quadratic variant: rescan all adjacent pairs each round and merge the
    first strict minimum (planner.py:267-290)."""
    live = len(R.lo)
    while stop_count is None or live > stop_count:
        best = None
        a = R.head()
        while a >= 0 and R.next[a] >= 0:
            b = R.next[a]
            if max_size is None or R.size(a) + R.size(b) <= max_size:
                ints, f, l = R.merged(a, b)
                delta = ints - (R.ints[a] + R.ints[b])
                if best is None or delta < best[0]:
                    best = (delta, a, b, ints, f, l)
            a = b
        if best is None:
            break
        _, a, b, ints, f, l = best
        R.merge(a, b, ints, f, l)
        live -= 1


def _native_plan(queries: SegmentStore, kind: str, index: TemporalIndex, **kw) -> BatchPlan:
    """The C++ planners of libtrajseek (csrc/planner.cu): same semantics, no Python loop."""
    from . import _native

    lo, hi, first, last, end = _native.plan_native(kind, queries.ts, queries.te, index, **kw)
    ts = queries.ts
    batches = tuple(
        QueryBatch(a, b, TimeInterval(float(ts[a]), e), None if f < 0 else f, None if f < 0 else l)
        for a, b, f, l, e in zip(lo.tolist(), hi.tolist(), first.tolist(), last.tolist(), end.tolist())
    )
    return BatchPlan(queries, batches)


def _native_ok() -> bool:
    from . import _native

    try:
        _native.load()
        return True
    except (RuntimeError, OSError):
        return False


def setsplit_fixed(queries: SegmentStore, index: TemporalIndex, num_batches: int, *,
                   literal: bool = False) -> BatchPlan:
    """Cheapest-first merging from singletons down to num_batches batches."""
    _check_queries(queries)
    if num_batches < 1:
        raise DomainError(f"num_batches={num_batches} must be >= 1")
    if not literal and _native_ok():
        return _native_plan(queries, "fixed", index, num_batches=num_batches)
    R = _Runs(queries, index)
    (_cheapest_rescan if literal else _cheapest_heap)(R, num_batches, None)
    return R.plan()


def setsplit_minmax(queries: SegmentStore, index: TemporalIndex, min_size: int, max_size: int,
                    *, literal: bool = False) -> BatchPlan:
    """Cheapest-first merging under a size ceiling, then a floor pass that
    folds each batch below min_size into its cheaper neighbour (a missing
    neighbour costs infinity; ties go right)."""
    _check_queries(queries)
    if min_size < 1:
        raise DomainError(f"min_size={min_size} must be >= 1")
    if max_size < min_size:
        raise DomainError(f"max_size={max_size} must be >= min_size={min_size}")
    if not literal and _native_ok():
        return _native_plan(queries, "minmax", index, min_size=min_size, max_size=max_size)
    R = _Runs(queries, index)
    (_cheapest_rescan if literal else _cheapest_heap)(R, None, max_size)
    i = R.head()
    while i >= 0:
        if R.size(i) >= min_size:
            i = R.next[i]
            continue
        left, right = R.prev[i], R.next[i]
        if left < 0 and right < 0:
            break
        lm = R.merged(left, i) if left >= 0 else None
        rm = R.merged(i, right) if right >= 0 else None
        lcost = lm[0] if lm is not None else math.inf
        rcost = rm[0] if rm is not None else math.inf
        if lcost < rcost:
            i = R.merge(left, i, *lm)
        else:
            i = R.merge(i, right, *rm)
    return R.plan()


def setsplit_max(queries: SegmentStore, index: TemporalIndex, max_size: int, *,
                 literal: bool = False) -> BatchPlan:
    """setsplit_minmax with the floor at one."""
    return setsplit_minmax(queries, index, 1, max_size, literal=literal)


# ── greedy family ───────────────────────────────────────────────────────────


def _free_pass(R: _Runs) -> None:
    """Merge forward while a merge adds no interactions (planner.py:371-381)."""
    i = 0
    while i >= 0 and R.next[i] >= 0:
        j = R.next[i]
        ints, f, l = R.merged(i, j)
        if ints == R.ints[i] + R.ints[j]:
            R.merge(i, j, ints, f, l)
        else:
            i = j


def _greedy(queries: SegmentStore, index: TemporalIndex, bound: int, grow, kind=None,
            native: bool = True) -> BatchPlan:
    _check_queries(queries)
    if bound < 1:
        raise DomainError(f"bound={bound} must be >= 1")
    if native and kind is not None and _native_ok():
        return _native_plan(queries, kind, index, bound=bound)
    R = _Runs(queries, index)
    _free_pass(R)
    i = R.head()
    while i >= 0 and R.next[i] >= 0:
        if grow(R.size(i), bound):
            j = R.next[i]
            R.merge(i, j, *R.merged(i, j))
        else:
            i = R.next[i]
    return R.plan()


def greedy_min(queries: SegmentStore, index: TemporalIndex, bound: int, *,
               native: bool = True) -> BatchPlan:
    """Free merges, then grow each batch until it holds at least ``bound``."""
    return _greedy(queries, index, bound, lambda size, b: size < b, "greedy_min", native)


def greedy_max(queries: SegmentStore, index: TemporalIndex, bound: int, *,
               native: bool = True) -> BatchPlan:
    """Free merges, then grow each batch until it exceeds ``bound``."""
    return _greedy(queries, index, bound, lambda size, b: size <= b, "greedy_max", native)
